"""Small solves over every kernel family, for the bounds-checked build
(HOLO_LIB_PATH=paper_1904_04884_b200/libholo_b200_checked.so; common.cuh
HOLO_CHECKS) and, for comparison, the normal one: prints one line per case
(iterations, guard fix-ups, skipped planes, the objective history and a hash
of the solution bytes) and the check bits last.  Cases:

  strip    128x128x8,  T = 5   single-pass strip prox (edge + interior regions), FFT passes, COO export
  walk     256x128x6,  T = 13  multi-pass strip walk (first / middle / last pass kinds)
  generic  32x32x4,    T = 5   generic tile prox (planes < 64)
  real     128x128x8,  T = 5   packed real engine
  skip     128x128x16, T = 5   all-zero planes skipped by the forward passes
  group    128x128x6,  2 ranks in-process rank group (peer-memory scatter / gather)
  guard    256x256x1   guard fix-up (forced prox rerun) on the strip kernel
  gsides   100x72x4 and 99x70x3 (packed real)  mixed-radix passes (gfft.cu), odd nx
"""
import ctypes
import hashlib
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_04884_b200 import RegularizerWeights, SolverConfig, VolumeGeometry, synth  # noqa: E402
from paper_1904_04884_b200 import _native as nat  # noqa: E402
from paper_1904_04884_b200.engine import HoloEngine  # noqa: E402
from paper_1904_04884_b200.solver import native_config  # noqa: E402


def hologram(nx, ny, seed, nz=8):
    """A rendered particle hologram (GPU render), b = 1 - I / mean(I)."""
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
    sc = synth.generate_scene(max(4, nx * ny // 2048), g, 20e-6, seed=seed, margin_planes=1)
    return np.ascontiguousarray(synth.invert_residual(synth.render_hologram(sc)))


def digest(eng):
    x = eng.solution_dense().cpu().numpy()
    assert np.all(np.isfinite(x)), "non-finite solution"
    return hashlib.sha256(x.tobytes()).hexdigest()[:16]


def solve(name, nx, ny, nz, T, lam=(0.2, 0.1), iters=3, z0=5e-3, b=None, real=False, step=None):
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, z0, 632e-9)
    eng = HoloEngine(g)
    cfg = native_config(SolverConfig(weights=RegularizerWeights(*lam), max_iters=iters, tv_inner_iters=T,
                                     real_nonnegative=real, step_size=step))
    _, rep, hist = eng.solve(hologram(nx, ny, nx + nz, nz) if b is None else b, cfg)
    eng.export_coo()
    h = digest(eng)
    eng.close()
    print(f"{name}: it {rep.iterations} nnz {rep.nnz} fixups {rep.guard_fixups} skipped {rep.skipped_planes} "
          f"hist {' '.join(f'{v:.9g}' for v in hist)} x {h}", flush=True)
    return rep


def group(nx, ny, nz, nranks):
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
    cfg = native_config(SolverConfig(weights=RegularizerWeights(0.2, 0.1), max_iters=2))
    b = hologram(nx, ny, 7, nz)
    engs = HoloEngine.local_group(g, nranks)
    out = [None] * nranks
    th = [threading.Thread(target=lambda r=r: out.__setitem__(r, engs[r].solve(b, cfg))) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    hs = [digest(e) for e in engs]
    for e in engs:
        e.close()
    print(f"group x{nranks}: it {[o[1].iterations for o in out]} hist {' '.join(f'{v:.9g}' for v in out[0][2])} "
          f"x {' '.join(hs)}", flush=True)


if __name__ == "__main__":
    torch.cuda.init()
    which = sys.argv[1:] or ["strip", "walk", "generic", "real", "skip", "group", "guard", "gsides"]
    if "strip" in which:
        solve("strip", 128, 128, 8, 5)
    if "walk" in which:
        solve("walk", 256, 128, 6, 13)
    if "generic" in which:
        solve("generic", 32, 32, 4, 5)
    if "real" in which:
        solve("real", 128, 128, 8, 5, lam=(0.3, 0.2), real=True, step=1.0 / 16)
    if "skip" in which:
        solve("skip", 128, 128, 16, 5, lam=(3.0, 0.2), iters=4, step=1.0 / 32)
    if "group" in which:
        group(128, 128, 6, 2)
    if "guard" in which:
        b = np.zeros((256, 256))
        b[60:140, 90:200] = 1.0
        rep = solve("guard", 256, 256, 1, 5, lam=(0.02, 1.0), iters=2, z0=0.0, b=b)
        assert rep.guard_fixups > 0
    if "gsides" in which:
        solve("gsides", 100, 72, 4, 5)
        solve("gsides-real", 99, 70, 3, 5, lam=(0.3, 0.2), real=True, step=1.0 / 12)
    v = ctypes.c_uint32(0)
    checked = nat.load().holo_debug_checks(ctypes.byref(v))
    print(f"checked-build {checked} check-bits {v.value:#x}", flush=True)
