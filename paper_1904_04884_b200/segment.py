"""Particle extraction from a reconstructed volume (segment.py of the reference).

SURVEY 8f row 1 (output side).  The reference labels 26-connected components
with a Python BFS over a dict of voxels (segment.py:106-146), which dominates
once the solve takes milliseconds.  Here the labelling is a GPU union-find
(`holo_label_components`, csrc/segment.cu); thresholding (segment.py:79-94),
the min-volume filter (:149-153), intensity-weighted centroids (:156-167) and
principal axes (:170-193) are vectorised reductions over the labelled voxels.
Emission order matches the reference: components sorted by their smallest
(k, i, j) voxel.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat

__all__ = ["ParticleDetection", "threshold_volume", "label_components", "extract_particles", "principal_axis"]


@dataclass
class ParticleDetection:
    """segment.py:62-76."""

    blob_id: int
    x_vox: float
    y_vox: float
    z_vox: float
    x: float
    y: float
    z: float
    volume: int
    peak_intensity: float
    axis: np.ndarray | None = None
    elongation: float | None = None


def threshold_volume(v, rel_tol: float):
    """Keep entries with |value| >= rel_tol * max|value| (segment.py:79-94)."""
    from .sparsevol import SparsePlane, SparseVolume
    if not 0.0 <= rel_tol < 1.0:
        raise ValueError(f"rel_tol must be in [0, 1), got {rel_tol}")
    if rel_tol == 0.0 or v.nnz == 0:
        return v
    vmax = max(float(np.abs(p.values).max()) for p in v.planes if p.nnz)
    cut = rel_tol * vmax
    planes = []
    for p in v.planes:
        if p.nnz == 0:
            planes.append(p)
            continue
        keep = np.abs(p.values) >= cut
        planes.append(SparsePlane(p.rows[keep], p.cols[keep], p.values[keep], p.shape))
    return SparseVolume(planes, v.geom)


def _voxels(v):
    """(n, 3) int32 (k, i, j) in lexicographic order and |value| weights."""
    ks, rs, cs, ws = [], [], [], []
    for k, p in enumerate(v.planes):
        if p.nnz:
            ks.append(np.full(p.nnz, k, dtype=np.int32))
            rs.append(np.asarray(p.rows, dtype=np.int32))
            cs.append(np.asarray(p.cols, dtype=np.int32))
            ws.append(np.abs(p.values))
    if not ks:
        return np.zeros((0, 3), np.int32), np.zeros(0)
    kij = np.stack([np.concatenate(ks), np.concatenate(rs), np.concatenate(cs)], axis=1)
    return np.ascontiguousarray(kij), np.concatenate(ws)


def label_components(kij: np.ndarray, shape3) -> np.ndarray:
    """Root id (smallest member id) of each voxel's 26-connected component, on the GPU."""
    import torch
    n = len(kij)
    if n == 0:
        return np.zeros(0, np.int32)
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
    lib = nat.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    k = torch.as_tensor(np.ascontiguousarray(kij, dtype=np.int32)).to(dev)
    roots = torch.empty(n, dtype=torch.int32, device=dev)
    nz, ny, nx = shape3
    nat.check(lib.holo_label_components(ctypes.c_void_p(k.data_ptr()), n, int(nz), int(ny), int(nx),
                                        ctypes.c_void_p(roots.data_ptr()),
                                        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
              "holo_label_components")
    return roots.cpu().numpy()


@dataclass
class AxisEstimate:
    axis: np.ndarray
    elongation: float
    reliable: bool


def principal_axis(pos: np.ndarray, w: np.ndarray, degenerate_tol: float = 1e-9) -> AxisEstimate:
    """Leading eigenvector of the weighted (x, y, z) covariance (segment.py:170-193)."""
    if len(w) < 2 or np.count_nonzero(w > 0) < 2:
        raise ValueError("principal axis needs at least 2 voxels with positive intensity")
    tot = w.sum()
    mean = (w[:, None] * pos).sum(axis=0) / tot
    d = pos - mean
    cov = (w[:, None, None] * d[:, :, None] * d[:, None, :]).sum(axis=0) / tot
    evals, evecs = np.linalg.eigh(cov)
    l1, l2 = float(evals[-1]), float(evals[-2])
    axis = evecs[:, -1]
    if axis[int(np.argmax(np.abs(axis)))] < 0:
        axis = -axis
    elong = float(np.sqrt(l1 / l2)) if l2 > 0 else float("inf")
    return AxisEstimate(axis, elong, (l1 - l2) > degenerate_tol * max(l1, degenerate_tol))


def extract_particles(v, rel_tol: float, min_vox: int, with_orientation: bool = False):
    """Threshold, label (GPU), filter and reduce to detections (segment.py:196-225)."""
    if min_vox < 0:
        raise ValueError(f"min_vox must be nonnegative, got {min_vox}")
    g = v.geom
    kij, w = _voxels(threshold_volume(v, rel_tol))
    if len(w) == 0:
        return []
    roots = label_components(kij, (g.nz, g.ny, g.nx))
    uniq, inv = np.unique(roots, return_inverse=True)  # ascending root = smallest-voxel order
    vol = np.bincount(inv)
    keep = np.nonzero(vol > min_vox)[0]
    tot = np.bincount(inv, weights=w)
    sx = np.bincount(inv, weights=w * kij[:, 2])
    sy = np.bincount(inv, weights=w * kij[:, 1])
    sz = np.bincount(inv, weights=w * kij[:, 0])
    peak = np.zeros(len(uniq))
    np.maximum.at(peak, inv, w)
    order = np.argsort(inv, kind="stable") if with_orientation else None
    starts = np.concatenate([[0], np.cumsum(vol)]) if with_orientation else None
    out = []
    for bid, c in enumerate(keep):
        if tot[c] <= 0.0:
            raise ValueError("blob has no positive intensity")
        cx, cy, cz = sx[c] / tot[c], sy[c] / tot[c], sz[c] / tot[c]
        det = ParticleDetection(blob_id=bid, x_vox=float(cx), y_vox=float(cy), z_vox=float(cz),
                                x=float(cx) * g.pitch, y=float(cy) * g.pitch, z=g.z0 + float(cz) * g.dz,
                                volume=int(vol[c]), peak_intensity=float(peak[c]))
        if with_orientation and vol[c] >= 2:
            members = order[starts[c]:starts[c + 1]]
            pos = kij[members][:, [2, 1, 0]].astype(np.float64)
            est = principal_axis(pos, w[members])
            if est.reliable:
                det.axis = est.axis
                det.elongation = est.elongation
        out.append(det)
    return out
