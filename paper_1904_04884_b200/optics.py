"""Geometry types and the GPU propagation operators.

Mirrors the parts of the reference's ``holotrack.optics`` that the solver
path uses (``optics.py:27-95`` types, ``optics.py:146-169`` TransferLadder,
``optics.py:187-230`` forward / adjoint).  The types are host-side records;
every numeric operator runs on the GPU through ``libholo_b200.so``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["ComplexField2D", "VolumeGeometry", "TransferLadder", "forward", "adjoint"]


@dataclass
class ComplexField2D:
    """Complex wavefield on a square-pixel grid (optics.py:27-59)."""

    values: np.ndarray
    pitch: float
    wavelength: float

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.complex128)
        if self.values.ndim != 2 or self.values.shape[0] < 1 or self.values.shape[1] < 1:
            raise ValueError(f"field values must be a 2D array, got shape {self.values.shape}")
        if self.pitch <= 0:
            raise ValueError(f"pitch must be positive, got {self.pitch}")
        if self.wavelength <= 0:
            raise ValueError(f"wavelength must be positive, got {self.wavelength}")
        if not np.all(np.isfinite(self.values)):
            raise ValueError("field values contain NaN or Inf")

    @property
    def height(self) -> int:
        return self.values.shape[0]

    @property
    def width(self) -> int:
        return self.values.shape[1]

    def copy(self) -> "ComplexField2D":
        return ComplexField2D(self.values.copy(), self.pitch, self.wavelength)


@dataclass(frozen=True)
class VolumeGeometry:
    """nx*ny voxels on nz planes; plane k at z0 + k*dz (optics.py:62-95)."""

    nx: int
    ny: int
    nz: int
    pitch: float
    dz: float
    z0: float
    wavelength: float

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1 or self.nz < 1:
            raise ValueError(f"voxel counts must be >= 1, got {(self.nx, self.ny, self.nz)}")
        if self.pitch <= 0 or self.dz <= 0 or self.wavelength <= 0:
            raise ValueError("pitch, dz and wavelength must be positive")
        if self.z0 < 0:
            raise ValueError(f"z0 must be nonnegative, got {self.z0}")

    @property
    def plane_shape(self) -> tuple[int, int]:
        return (self.ny, self.nx)

    def plane_z(self, k: int) -> float:
        return self.z0 + k * self.dz

    @property
    def n_voxels(self) -> int:
        return self.nx * self.ny * self.nz


def _session(geom):
    from .engine import session
    return session(geom)


class TransferLadder:
    """Per-plane transfer functions H(z0 + k dz) evaluated on the GPU
    (optics.py:146-169).  ``stack`` returns complex64 planes; the phase is
    carried as a 64-bit fixed-point cycle count so it is exact mod 1."""

    def __init__(self, geom):
        self.geom = geom

    def stack(self, k0: int, k1: int, conj: bool = False):
        return _session(self.geom).transfer(k0, k1, conj)


def forward(x, geom, chunk: int = 16) -> ComplexField2D:
    """Re{sum_k propagate(x_k, -(z0 + k dz))} on the GPU (optics.py:187-212).
    ``x``: SparseVolume or dense (nz, ny, nx) stack.  ``chunk`` is accepted for
    API compatibility; the GPU processes all planes at once."""
    del chunk
    dense = x.to_dense() if hasattr(x, "planes") else np.asarray(x)
    if dense.shape[0] != geom.nz:
        raise ValueError(f"volume has {dense.shape[0]} planes, geometry expects {geom.nz}")
    out = _session(geom).forward(dense)
    return ComplexField2D(out.astype(np.complex128), geom.pitch, geom.wavelength)


def adjoint(r: ComplexField2D, geom, chunk: int = 16) -> np.ndarray:
    """Plane k = propagate(r, +(z0 + k dz)) on the GPU (optics.py:215-230).
    Only Re(r) enters, as in the solver path (solver.py:274)."""
    del chunk
    vals = r.values if hasattr(r, "values") else np.asarray(r)
    if vals.shape != geom.plane_shape:
        raise ValueError(f"sensor field shape {vals.shape} does not match geometry planes {geom.plane_shape}")
    if np.iscomplexobj(vals) and np.any(vals.imag != 0):
        raise ValueError("the GPU adjoint takes a real sensor field (solver path semantics)")
    return _session(geom).adjoint(np.real(vals), scale=1.0)
