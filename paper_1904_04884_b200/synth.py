"""Input side of the path: scenes, GPU hologram rendering,
noise and residual formation, mirroring synth.py / preprocess.py of the reference.

Scene sampling and noise use numpy's ``default_rng`` exactly like the
reference (same draws for the same seed); the expensive part -- the
nonlinear render, one full-plane FFT per particle in the reference
(synth.py:161-181, 0.1 s/particle at 1024^2) -- runs on the GPU:
``holo_render_spectrum`` accumulates every particle's masked, propagated
spectrum in fp64 and the library FFT inverts it.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass, replace

import numpy as np

from . import _native as nat

__all__ = ["Particle", "Scene", "generate_scene", "advect_scene", "particle_mask", "render_hologram", "add_noise",
           "shadow_density", "invert_residual", "preprocess_background"]


@dataclass
class Particle:
    """synth.py:31-50."""

    x: float
    y: float
    z: float
    diameter: float
    opacity: float = 1.0
    orientation: np.ndarray | None = None
    length: float | None = None

    def __post_init__(self):
        if self.diameter <= 0:
            raise ValueError(f"particle diameter must be positive, got {self.diameter}")
        if not 0.0 <= self.opacity <= 1.0:
            raise ValueError(f"opacity must be in [0, 1], got {self.opacity}")
        if self.orientation is not None:
            self.orientation = np.asarray(self.orientation, dtype=np.float64)
            if abs(float(np.linalg.norm(self.orientation)) - 1.0) > 1e-9:
                raise ValueError("orientation must be unit norm")


@dataclass
class Scene:
    """synth.py:53-71."""

    particles: list
    geom: object
    rng_seed: int = 0

    def __post_init__(self):
        g = self.geom
        for i, p in enumerate(self.particles):
            if not (0.0 <= p.x <= g.nx * g.pitch and 0.0 <= p.y <= g.ny * g.pitch):
                raise ValueError(f"particle {i} lateral position outside the volume")
            if not (g.z0 <= p.z <= g.z0 + g.nz * g.dz):
                raise ValueError(f"particle {i} depth {p.z} outside [{g.z0}, {g.z0 + g.nz * g.dz}]")

    def positions(self) -> np.ndarray:
        if not self.particles:
            return np.zeros((0, 3))
        return np.array([[p.x, p.y, p.z] for p in self.particles])


def generate_scene(n, geom, diameter, seed=0, opacity=1.0, margin_planes=0) -> Scene:
    """Uniform particles, same draw order as synth.py:74-106 (x, y, z per particle)."""
    if n < 0:
        raise ValueError(f"particle count must be nonnegative, got {n}")
    if margin_planes < 0:
        raise ValueError("margin_planes must be nonnegative")
    if n > 0 and 2 * margin_planes >= geom.nz:
        raise ValueError("margin_planes leaves no depth range to sample")
    rng = np.random.default_rng(seed)
    zlo = geom.z0 + margin_planes * geom.dz
    zhi = geom.z0 + (geom.nz - margin_planes) * geom.dz
    out = []
    for _ in range(n):
        x = rng.uniform(0.0, geom.nx * geom.pitch)
        y = rng.uniform(0.0, geom.ny * geom.pitch)
        z = rng.uniform(zlo, zhi)
        out.append(Particle(x=x, y=y, z=z, diameter=diameter, opacity=opacity))
    return Scene(out, geom, rng_seed=seed)


def advect_scene(scene: Scene, velocity_field, dt: float) -> Scene:
    """Forward-Euler step with periodic wrap (synth.py:109-126)."""
    if dt <= 0:
        raise ValueError(f"dt must be positive, got {dt}")
    g = scene.geom
    lx, ly, lz = g.nx * g.pitch, g.ny * g.pitch, g.nz * g.dz
    moved = []
    for p in scene.particles:
        v = np.asarray(velocity_field((p.x, p.y, p.z)), dtype=np.float64)
        moved.append(replace(p, x=(p.x + dt * v[0]) % lx, y=(p.y + dt * v[1]) % ly,
                             z=g.z0 + (p.z + dt * v[2] - g.z0) % lz))
    return Scene(moved, g, rng_seed=scene.rng_seed)


def particle_mask(p: Particle, geom):
    """Opaque-mask pixels (rows, cols, amplitude) of one particle (synth.py:129-158):
    a disk, an oriented rectangle for rods, or one pixel below the pitch."""
    g = geom
    if p.diameter < g.pitch:
        warnings.warn(f"particle diameter {p.diameter:g} below pixel pitch {g.pitch:g}; using a single-pixel mask",
                      stacklevel=3)
        iy = int(np.clip(round(p.y / g.pitch), 0, g.ny - 1))
        ix = int(np.clip(round(p.x / g.pitch), 0, g.nx - 1))
        return np.array([iy]), np.array([ix]), np.array([p.opacity])
    if p.orientation is None or p.length is None:
        reach = p.diameter / 2.0
    else:
        lat = float(np.linalg.norm(p.orientation[:2]))
        reach = max(p.length * lat, p.diameter) / 2.0 + p.diameter / 2.0
    ix0 = max(0, int(np.floor((p.x - reach) / g.pitch)) - 1)
    ix1 = min(g.nx, int(np.ceil((p.x + reach) / g.pitch)) + 2)
    iy0 = max(0, int(np.floor((p.y - reach) / g.pitch)) - 1)
    iy1 = min(g.ny, int(np.ceil((p.y + reach) / g.pitch)) + 2)
    xs = (np.arange(ix0, ix1) * g.pitch - p.x)[np.newaxis, :]
    ys = (np.arange(iy0, iy1) * g.pitch - p.y)[:, np.newaxis]
    if p.orientation is None or p.length is None:
        inside = (xs ** 2 + ys ** 2) <= (p.diameter / 2.0) ** 2
    else:
        axis = p.orientation[:2]
        lat = np.linalg.norm(axis)
        proj = max(p.length * lat, p.diameter)
        ux, uy = (axis / lat) if lat > 1e-12 else (1.0, 0.0)
        u = ux * xs + uy * ys
        v = -uy * xs + ux * ys
        inside = (np.abs(u) <= proj / 2.0) & (np.abs(v) <= p.diameter / 2.0)
    r, c = np.nonzero(inside)
    return r + iy0, c + ix0, np.full(len(r), float(p.opacity))


def _spectrum_on_gpu(scene: Scene):
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
    g = scene.geom
    lib = nat.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    rows, cols, amps, offs, zl = [], [], [], [0], []
    for p in scene.particles:
        r, c, a = particle_mask(p, g)
        rows.append(r)
        cols.append(c)
        amps.append(a)
        offs.append(offs[-1] + len(a))
        zl.append(p.z / g.wavelength)
    n = len(scene.particles)
    yx = np.stack([np.concatenate(rows), np.concatenate(cols)], axis=1) if n else np.zeros((0, 2))

    def dv(a, dt):
        return torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(dev)

    t_zl, t_off = dv(np.array(zl), np.float64), dv(np.array(offs), np.int32)
    t_yx, t_a = dv(yx, np.int32), dv(np.concatenate(amps) if n else np.zeros(0), np.float64)
    spec = torch.empty((g.ny, g.nx, 2), dtype=torch.float64, device=dev)
    ptr = lambda t: ctypes.c_void_p(t.data_ptr() if t.numel() else 0)  # noqa: E731
    nat.check(lib.holo_render_spectrum(ptr(t_zl), ptr(t_off), ptr(t_yx), ptr(t_a), n, g.ny, g.nx, float(g.pitch),
                                       float(g.wavelength), ptr(spec),
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
              "holo_render_spectrum")
    return spec


def render_hologram(scene: Scene) -> np.ndarray:
    """|1 - ifft2(sum_p fft2(mask_p) H(-z_p))|^2 (synth.py:161-181) on the GPU."""
    import torch
    from .engine import session
    g = scene.geom
    spec = _spectrum_on_gpu(scene)
    flat = type("PlaneGeom", (), dict(nx=g.nx, ny=g.ny, nz=1, pitch=g.pitch, dz=g.dz, z0=g.z0,
                                      wavelength=g.wavelength, plane_shape=(g.ny, g.nx)))()
    c64 = torch.view_as_complex(spec.to(torch.float32).contiguous()).reshape(1, g.ny, g.nx)
    eng = session(flat)
    nat.check(eng.lib.holo_op_fft2(eng.h, ctypes.c_void_p(c64.data_ptr()), 1, 1,
                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "holo_op_fft2")
    fld = c64[0].cpu().numpy().astype(np.complex128)
    return np.abs(1.0 - fld) ** 2


def add_noise(image, gaussian_sigma, seed=0):
    """Clamped white Gaussian noise, same draws as synth.py:184-191."""
    if gaussian_sigma < 0:
        raise ValueError(f"sigma must be nonnegative, got {gaussian_sigma}")
    if gaussian_sigma == 0:
        return np.array(image, copy=True)
    rng = np.random.default_rng(seed)
    return np.maximum(image + rng.normal(0.0, gaussian_sigma, np.shape(image)), 0.0)


def shadow_density(n_s: float, depth: float, d: float) -> float:
    """synth.py:194-202."""
    if n_s < 0 or depth < 0 or d < 0:
        raise ValueError("shadow density inputs must be nonnegative")
    return (n_s * d) * (depth * d)


def invert_residual(image, normalize: bool = True):
    """1 - I / mean(I) (preprocess.py:41-53)."""
    image = np.asarray(image, dtype=np.float64)
    if normalize:
        m = image.mean()
        if m <= 0:
            raise ValueError("image mean must be positive to normalize")
        return 1.0 - image / m
    return 1.0 - image


def preprocess_background(images, window: int = 151) -> np.ndarray:
    """(I - M) / sqrt(M), sliding temporal mean without the frame itself (preprocess.py:17-38), GPU."""
    import torch
    images = np.asarray(images, dtype=np.float64)
    if images.ndim != 3:
        raise ValueError(f"expected a (T, ny, nx) stack, got shape {images.shape}")
    T = images.shape[0]
    if window % 2 != 1 or window < 3 or window > T:
        raise ValueError(f"window must be odd, >= 3 and <= {T}, got {window}")
    dev = torch.device("cuda", torch.cuda.current_device())
    src = torch.as_tensor(np.ascontiguousarray(images)).to(dev)
    out = torch.empty_like(src)
    nat.check(nat.load().holo_background(ctypes.c_void_p(src.data_ptr()), T, images.shape[1], images.shape[2], window,
                                         ctypes.c_void_p(out.data_ptr()),
                                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "holo_background")
    return out.cpu().numpy()
