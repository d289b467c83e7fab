"""CPU oracle for the RIHVR fused-lasso FISTA hot path (numpy, float64).

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this file.
It may be imported only by ``tests/``, ``__graft_entry__.smoke()`` (as the
checker) and ``bench.py`` (the ``cpu_baseline`` leg and ``--impl reference``).

What it is: a dense-volume restatement of the reference package ``holotrack``
(``/root/reference/pkg/src/holotrack``), written from its behaviour, not copied.
Each function cites the reference lines it restates.  The reference keeps
iterates as COO planes; with ``drop_tol = 0`` COO <-> dense is exact
(``sparsevol.py:75-88``), so a dense restatement computes the same numbers.

Parity pin: ``tests/golden/make_golden.py`` imported the reference in the build
container and wrote ``tests/golden/*.npz``; ``tests/test_oracle.py`` checks
this oracle against every one of those vectors (operators and end-to-end
``fista``) on CPU.
"""

from __future__ import annotations

import math
from collections import deque

import numpy as np

DIVERGENCE_FACTOR = 1e6  # solver.py:35


# ---------------------------------------------------------------- optics ----

def freq_axis(n: int, pitch: float) -> np.ndarray:
    """numpy.fft.fftfreq(n, d=pitch): the sample grid of optics.py:120-121."""
    return np.fft.fftfreq(n, d=pitch)


def propagation_root(ny: int, nx: int, pitch: float, wavelength: float):
    """sqrt(1 - (lam fx)^2 - (lam fy)^2) and the propagating mask (optics.py:98-116)."""
    fy = freq_axis(ny, pitch)[:, None]
    fx = freq_axis(nx, pitch)[None, :]
    arg = 1.0 - (wavelength * fx) ** 2 - (wavelength * fy) ** 2
    keep = arg >= 0.0
    root = np.sqrt(np.where(keep, arg, 0.0))
    return root, keep


def transfer(ny, nx, pitch, wavelength, z) -> np.ndarray:
    """H(fx, fy; z) = exp(i 2 pi (z/lam) root), 0 where evanescent (optics.py:98-122)."""
    root, keep = propagation_root(ny, nx, pitch, wavelength)
    phase = 2.0 * np.pi * (z / wavelength) * root
    return np.where(keep, np.exp(1j * phase), 0.0).astype(np.complex128)


class Geometry:
    """nx, ny, nz, pitch, dz, z0, wavelength -- the fields of optics.py:62-95."""

    def __init__(self, nx, ny, nz, pitch, dz, z0, wavelength):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.pitch, self.dz, self.z0, self.wavelength = float(pitch), float(dz), float(z0), float(wavelength)

    @property
    def shape(self):
        return (self.ny, self.nx)

    @property
    def voxels(self):
        return self.nx * self.ny * self.nz

    @classmethod
    def of(cls, g):
        return cls(g.nx, g.ny, g.nz, g.pitch, g.dz, g.z0, g.wavelength)


def transfer_stack(g: Geometry, k0: int, k1: int, conj: bool = False) -> np.ndarray:
    """Planes k0..k1-1 of the ladder H_k = H(z0) * H(dz)^k (optics.py:146-169).

    The recurrence (one complex multiply per plane, complex128) is kept so the
    rounding matches the reference's ladder, not a fresh exp per plane.
    """
    h0 = transfer(g.ny, g.nx, g.pitch, g.wavelength, g.z0)
    step = transfer(g.ny, g.nx, g.pitch, g.wavelength, g.dz)
    cur = h0 * step ** k0 if k0 else h0.copy()
    out = np.empty((k1 - k0, g.ny, g.nx), dtype=np.complex128)
    for i in range(k1 - k0):
        out[i] = cur
        if i + 1 < k1 - k0:
            cur = cur * step
    return np.conj(out) if conj else out


def sensor_forward(vol: np.ndarray, g: Geometry, chunk: int = 16) -> np.ndarray:
    """A x = Re ifft2( sum_k fft2(x_k) conj(H_k) ), zero planes skipped (solver.py:110-124)."""
    spec = np.zeros(g.shape, dtype=np.complex128)
    nonzero = [bool(np.any(vol[k] != 0)) for k in range(g.nz)]
    for k0 in range(0, g.nz, chunk):
        k1 = min(g.nz, k0 + chunk)
        if not any(nonzero[k0:k1]):
            continue
        hs = transfer_stack(g, k0, k1, conj=True)
        for k in range(k0, k1):
            if nonzero[k]:
                spec += np.fft.fft2(vol[k].astype(np.complex128)) * hs[k - k0]
    return np.fft.ifft2(spec).real


def back_project(r: np.ndarray, g: Geometry, chunk: int = 16) -> np.ndarray:
    """A^H r: plane k = ifft2(H_k fft2(r)) (optics.py:215-230; solver.py:126-132 is 2x this)."""
    spec = np.fft.fft2(np.asarray(r, dtype=np.complex128))
    out = np.empty((g.nz,) + g.shape, dtype=np.complex128)
    for k0 in range(0, g.nz, chunk):
        k1 = min(g.nz, k0 + chunk)
        out[k0:k1] = np.fft.ifft2(transfer_stack(g, k0, k1) * spec[None], axes=(-2, -1))
    return out


def cosine_stack(g: Geometry) -> np.ndarray:
    """C_k = cos(2 pi (z0 + k dz) q) on the rfft half grid, by the fp64 angle-addition
    recurrence of the real engine (solver.py:165-182)."""
    fy = freq_axis(g.ny, g.pitch)
    fx = np.fft.rfftfreq(g.nx, d=g.pitch)
    FY, FX = np.meshgrid(fy, fx, indexing="ij")
    arg = 1.0 - (g.wavelength * FY) ** 2 - (g.wavelength * FX) ** 2
    keep = arg >= 0
    root = np.sqrt(np.where(keep, arg, 0.0))
    c = np.cos(2 * np.pi * (g.z0 / g.wavelength) * root) * keep
    sn = np.sin(2 * np.pi * (g.z0 / g.wavelength) * root) * keep
    cg = np.cos(2 * np.pi * (g.dz / g.wavelength) * root)
    sg = np.sin(2 * np.pi * (g.dz / g.wavelength) * root)
    out = np.empty((g.nz,) + c.shape)
    for k in range(g.nz):
        out[k] = c
        c, sn = c * cg - sn * sg, c * sg + sn * cg
    return out


def real_forward(vol, g: Geometry, cs=None) -> np.ndarray:
    """Real-nonnegative engine forward: irfft2(sum_k rfft2(Re x_k) C_k) (solver.py:184-193)."""
    cs = cosine_stack(g) if cs is None else cs
    spec = np.zeros(cs.shape[1:], dtype=np.complex128)
    for k in range(g.nz):
        xk = np.real(vol[k])
        if np.any(xk != 0):
            spec += np.fft.rfft2(xk) * cs[k]
    return np.fft.irfft2(spec, s=g.shape)


def real_back_project(r, g: Geometry, cs=None) -> np.ndarray:
    """Real engine adjoint: plane k = irfft2(C_k rfft2(r)) (solver.py:195-200 is 2x this)."""
    cs = cosine_stack(g) if cs is None else cs
    rs = np.fft.rfft2(np.asarray(r, dtype=np.float64))
    return np.fft.irfft2(cs * rs[None], s=g.shape, axes=(-2, -1))


# ------------------------------------------------------------------ prox ----

def _grad2(x):
    """Backward differences, zero on the first row / column (prox.py:43-49)."""
    gy = np.zeros_like(x)
    gx = np.zeros_like(x)
    gy[..., 1:, :] = np.diff(x, axis=-2)
    gx[..., :, 1:] = np.diff(x, axis=-1)
    return gy, gx


def _grad2_adj(py, px):
    """Adjoint of _grad2: a[i,j] = py[i,j]-py[i+1,j] + px[i,j]-px[i,j+1] (prox.py:52-58)."""
    a = py + px
    a[..., :-1, :] -= py[..., 1:, :]
    a[..., :, :-1] -= px[..., :, 1:]
    return a


def tv_norm(plane) -> float:
    """Isotropic TV of a real plane, sum sqrt(dy^2 + dx^2) (prox.py:61-72)."""
    gy, gx = _grad2(np.asarray(plane, dtype=np.float64))
    return float(np.sum(np.sqrt(gy * gy + gx * gx)))


def soft_threshold(v, tau: float):
    """Complex-modulus shrinkage; |v| <= tau -> exact 0 (prox.py:83-96)."""
    if tau < 0:
        raise ValueError("tau must be nonnegative")
    v = np.asarray(v)
    if tau == 0:
        return v.copy()
    mag = np.abs(v)
    with np.errstate(invalid="ignore", divide="ignore"):
        gain = np.where(mag > tau, 1.0 - tau / mag, 0.0)
    return v * gain


def _tv_cost(x, v, tau):
    d = (x - v).ravel()
    return tau * tv_norm(x) + 0.5 * float(d @ d)


def fgp_tv(v, tau: float, iters: int = 5, guard: bool = True):
    """Beck-Teboulle fast gradient projection for the 2D TV prox, with the
    per-plane 'never worse than v' guard (prox.py:104-148).  guard=False
    (tests only) returns the FGP output without the guard's select."""
    if tau < 0 or iters < 1:
        raise ValueError("bad tau / iters")
    v = np.asarray(v, dtype=np.float64)
    if tau == 0:
        return v.copy()
    py = np.zeros_like(v)
    px = np.zeros_like(v)
    ey, ex = py, px  # extrapolated dual
    t = 1.0
    lr = 1.0 / (8.0 * tau)
    for _ in range(iters):
        gy, gx = _grad2(v - tau * _grad2_adj(ey, ex))
        ny_ = ey + lr * gy
        nx_ = ex + lr * gx
        scale = np.maximum(1.0, np.sqrt(ny_ * ny_ + nx_ * nx_))
        ny_ /= scale
        nx_ /= scale
        t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t * t))
        mom = (t - 1.0) / t_next
        ey = ny_ + mom * (ny_ - py)
        ex = nx_ + mom * (nx_ - px)
        py, px, t = ny_, nx_, t_next
    out = v - tau * _grad2_adj(py, px)
    if not guard:
        return out
    flat_o = out.reshape(-1, *out.shape[-2:])
    flat_v = v.reshape(-1, *v.shape[-2:])
    for i in range(flat_o.shape[0]):
        if _tv_cost(flat_o[i], flat_v[i], tau) > _tv_cost(flat_v[i], flat_v[i], tau):
            flat_o[i] = flat_v[i]
    return out


def fgp_beta_schedule(iters: int):
    """The data-independent FGP momentum coefficients (prox.py:132-133)."""
    t, out = 1.0, []
    for _ in range(iters):
        tn = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t * t))
        out.append((t - 1.0) / tn)
        t = tn
    return out


def fused_prox(v, tau_l1: float, tau_tv: float, iters: int = 5, guard: bool = True):
    """prox_l1(prox_tv(Re) + i prox_tv(Im)) (prox.py:151-165, solver.py:139-144)."""
    v = np.asarray(v)
    if tau_tv > 0:
        if np.iscomplexobj(v):
            w = fgp_tv(v.real, tau_tv, iters, guard) + 1j * fgp_tv(v.imag, tau_tv, iters, guard)
        else:
            w = fgp_tv(v, tau_tv, iters, guard)
    else:
        w = v
    return soft_threshold(w, tau_l1)


# ---------------------------------------------------------------- solver ----

def power_start(g: Geometry, seed: int = 0, real: bool = False) -> np.ndarray:
    """The power iteration's start vector: default_rng(seed) normals (solver.py:231-237)."""
    rng = np.random.default_rng(seed)
    shp = (g.nz,) + g.shape
    if real:
        v = rng.standard_normal(shp)
    else:
        v = rng.standard_normal(shp) + 1j * rng.standard_normal(shp)
    return v / np.linalg.norm(v)


def power_norm(g: Geometry, iters: int = 10, seed: int = 0, real: bool = False) -> float:
    """||A||^2 by power iteration from default_rng(seed) (solver.py:225-247)."""
    v = power_start(g, seed, real)
    cs = cosine_stack(g) if real else None
    nrm = 1.0
    for _ in range(iters):
        if real:
            w = real_back_project(real_forward(v, g, cs), g, cs)
        else:
            w = back_project(sensor_forward(v, g, chunk=g.nz), g, chunk=64)
        nrm = float(np.linalg.norm(w))
        v = w / nrm
    return nrm


def _penalty(vol, lam_l1, lam_tv, real=False):
    """sum over planes of lam_l1 |x|_1 + lam_tv (TV re + TV im) (solver.py:146-151, 282-283);
    real engine: lam_l1 sum x + lam_tv TV(x) (solver.py:212-216)."""
    total = 0.0
    for k in range(vol.shape[0]):
        p = vol[k]
        if not np.any(p != 0):
            continue
        if real:
            total += lam_l1 * float(np.sum(p.real))
            if lam_tv > 0:
                total += lam_tv * tv_norm(p.real)
            continue
        total += lam_l1 * float(np.sum(np.abs(p)))
        if lam_tv > 0:
            total += lam_tv * (tv_norm(p.real) + tv_norm(p.imag))
    return total


class OracleResult:
    def __init__(self, x, history, iterations, step, restarts, diverged):
        self.x, self.history, self.iterations = x, history, iterations
        self.step, self.restarts, self.diverged = step, restarts, diverged

    @property
    def nnz(self):
        return int(np.count_nonzero(self.x))


def fista_solve(b, g: Geometry, lam_l1=0.5, lam_tv=0.2, max_iters=100, inner=5,
                policy="backtracking", step_size=None, shrink=0.5, stop_tol=0.0,
                chunk=16, real=False) -> OracleResult:
    """Dense restatement of solver.fista (solver.py:254-379); real=True is the
    real-nonnegative engine (solver.py:154-216)."""
    bb = np.asarray(b, dtype=np.float64).real
    if bb.shape != g.shape:
        raise ValueError("hologram / geometry shape mismatch")
    if step_size is not None:
        step = float(step_size)
    else:
        s2 = power_norm(g, real=real)
        step = 1.0 / (2.0 * s2) if s2 > 0 else 1.0
    cs = cosine_stack(g) if real else None

    def fwd(vol):
        return real_forward(vol, g, cs) if real else sensor_forward(vol, g, chunk)

    def data_misfit(vol):
        r = fwd(vol) - bb
        return float(np.sum(r * r))

    def attempt(y, step_local):
        # one prox-gradient step from y with backtracking (solver.py:297-327)
        res = fwd(y) - bb
        f_y = float(np.sum(res * res))
        rs = np.fft.fft2(res.astype(np.complex128))
        while True:
            new = np.empty_like(y)
            ip = 0.0
            dx2 = 0.0
            for k0 in range(0, g.nz, chunk):
                k1 = min(g.nz, k0 + chunk)
                yk = y[k0:k1]
                if real:
                    grad = 2.0 * np.fft.irfft2(cs[k0:k1] * np.fft.rfft2(res)[None], s=g.shape, axes=(-2, -1))
                    w = yk.real - step_local * grad
                    if lam_tv > 0:
                        w = fgp_tv(w, step_local * lam_tv, inner)
                    cand = np.maximum(w - step_local * lam_l1, 0.0).astype(np.complex128)
                    d = cand.real - yk.real
                    ip += float(np.sum(grad * d))
                    dx2 += float(np.sum(d * d))
                else:
                    grad = 2.0 * np.fft.ifft2(transfer_stack(g, k0, k1) * rs[None], axes=(-2, -1))
                    cand = fused_prox(yk - step_local * grad, step_local * lam_l1, step_local * lam_tv, inner)
                    d = cand - yk
                    ip += float(np.sum((grad.conj() * d).real))
                    dx2 += float(np.sum((d * d.conj()).real))
                new[k0:k1] = cand
            f_new = data_misfit(new)
            if policy != "backtracking":
                return new, f_new, step_local
            bound = f_y + ip + dx2 / (2.0 * step_local)
            if f_new <= bound + 1e-12 * max(1.0, abs(bound)) or step_local < 1e-30:
                return new, f_new, step_local
            step_local *= shrink

    x = np.zeros((g.nz,) + g.shape, dtype=np.complex128)
    x_old = x
    t = 1.0
    f0 = float(np.sum(bb * bb))
    last = f0
    hist = []
    restarts = 0
    for it in range(max_iters):
        tn = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t * t))
        beta = (t - 1.0) / tn
        y = (1.0 + beta) * x - beta * x_old if beta != 0.0 else x
        new, f_new, step = attempt(y, step)
        obj = f_new + _penalty(new, lam_l1, lam_tv, real)
        if obj > last and it > 0:  # adaptive restart (solver.py:339-349)
            restarts += 1
            t = tn = 1.0
            new, f_new, step = attempt(x, step)
            obj = f_new + _penalty(new, lam_l1, lam_tv, real)
            if obj > last:
                new, obj = x, last
        x_old, x, t = x, new, tn
        hist.append(obj)
        if obj > DIVERGENCE_FACTOR * max(f0, 1e-300):
            return OracleResult(x, hist, it + 1, step, restarts, True)
        if stop_tol > 0 and last > 0 and abs(last - obj) / max(last, 1e-300) < stop_tol:
            break
        last = obj
    return OracleResult(x, hist, len(hist), step, restarts, False)


# ------------------------------------------------------------- detection ----

_NBR = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1) if (a, b, c) != (0, 0, 0)]


def detect_particles(vol: np.ndarray, rel_tol: float, min_vox: int):
    """Threshold at rel_tol*max|x|, 26-connected components, keep volume > min_vox,
    |x|-weighted centroids (x, y, z) in voxels (segment.py:79-225).

    Returns an (n, 4) array of (x_vox, y_vox, z_vox, volume), blobs ordered by
    their smallest (k, i, j) voxel like segment.connected_components."""
    mag = np.abs(vol)
    if not np.any(mag > 0):
        return np.zeros((0, 4))
    keep = mag > 0
    if rel_tol > 0:
        keep &= mag >= rel_tol * mag.max()
    ks, iis, jjs = np.nonzero(keep)  # lexicographic (k, i, j) order
    lookup = {(int(k), int(i), int(j)): n for n, (k, i, j) in enumerate(zip(ks, iis, jjs))}
    label = np.full(len(ks), -1)
    rows = []
    for start in range(len(ks)):
        if label[start] >= 0:
            continue
        label[start] = start
        members = [start]
        todo = deque([start])
        while todo:
            n = todo.popleft()
            k, i, j = int(ks[n]), int(iis[n]), int(jjs[n])
            for dk, di, dj in _NBR:
                m = lookup.get((k + dk, i + di, j + dj))
                if m is not None and label[m] < 0:
                    label[m] = start
                    members.append(m)
                    todo.append(m)
        if len(members) <= min_vox:
            continue
        idx = np.array(members)
        w = mag[ks[idx], iis[idx], jjs[idx]]
        tot = float(w.sum())
        rows.append((float((w * jjs[idx]).sum() / tot), float((w * iis[idx]).sum() / tot),
                     float((w * ks[idx]).sum() / tot), float(len(idx))))
    return np.array(rows).reshape(-1, 4)


# ------------------------------------------------------- synthetic inputs ----

def make_scene(n, g: Geometry, diameter, seed=0, margin_planes=0):
    """(n, 3) particle centres (x, y, z) in metres, uniform, seeded (synth.py:74-106)."""
    rng = np.random.default_rng(seed)
    zlo = g.z0 + margin_planes * g.dz
    zhi = g.z0 + (g.nz - margin_planes) * g.dz
    pts = np.empty((n, 3))
    for p in range(n):  # same draw order as the reference: x, y, z per particle
        pts[p, 0] = rng.uniform(0.0, g.nx * g.pitch)
        pts[p, 1] = rng.uniform(0.0, g.ny * g.pitch)
        pts[p, 2] = rng.uniform(zlo, zhi)
    return pts


def render_hologram(points, g: Geometry, diameter, opacity=1.0):
    """|1 - ifft2(sum_p fft2(disk_p) H(-z_p))|^2 for opaque disks (synth.py:129-181).
    diameter >= pitch only (the single-pixel branch of synth.py:134-143 is not restated)."""
    if diameter < g.pitch:
        raise ValueError("sub-pixel particles are not restated")
    root, keep = propagation_root(g.ny, g.nx, g.pitch, g.wavelength)
    xs = np.arange(g.nx) * g.pitch
    ys = np.arange(g.ny) * g.pitch
    spec = np.zeros(g.shape, dtype=np.complex128)
    for px_, py_, pz in points:
        disk = ((xs[None, :] - px_) ** 2 + (ys[:, None] - py_) ** 2) <= (diameter / 2.0) ** 2
        h = np.exp(-1j * 2.0 * np.pi * (pz / g.wavelength) * root) * keep
        spec += np.fft.fft2(disk.astype(np.float64) * opacity) * h
    return np.abs(1.0 - np.fft.ifft2(spec)) ** 2


def add_noise(img, sigma, seed=0):
    """Clamped white Gaussian noise (synth.py:184-191)."""
    if sigma == 0:
        return np.array(img, copy=True)
    rng = np.random.default_rng(seed)
    return np.maximum(img + rng.normal(0.0, sigma, np.shape(img)), 0.0)


def invert_residual(img):
    """b = 1 - I / mean(I) (preprocess.py:41-53)."""
    img = np.asarray(img, dtype=np.float64)
    m = img.mean()
    if m <= 0:
        raise ValueError("image mean must be positive")
    return 1.0 - img / m
