"""Small solves that touch every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

  * 128x128x8, T = 5   -> single-pass strip prox (edge + interior regions), column/row FFT passes,
                          TMA-staged forward columns, sensor, reductions, COO export
  * 128x256x6, T = 13  -> multi-pass strip walk (first / middle / last pass kinds, saved rows)
  * 32x32x4,   T = 5   -> generic tile prox (planes < 64)
  * 128x128x6, 2 ranks -> in-process rank group: peer-memory scatter / gather / flag waits
  * 256x256x1 plateau  -> the guard fix-up (forced prox rerun) on the strip kernel

usage: compute-sanitizer --tool racecheck python tools/sanitize_solve.py
"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_04884_b200 import RegularizerWeights, SolverConfig, VolumeGeometry  # noqa: E402
from paper_1904_04884_b200.engine import HoloEngine  # noqa: E402
from paper_1904_04884_b200.solver import native_config  # noqa: E402


def hologram(nx, ny, seed):
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(rng.standard_normal((ny, nx)) * 0.05)


def solve(nx, ny, nz, T, lam=(0.05, 0.1), iters=3, z0=5e-3, b=None):
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, z0, 632e-9)
    eng = HoloEngine(g)
    cfg = native_config(SolverConfig(weights=RegularizerWeights(*lam), max_iters=iters, tv_inner_iters=T))
    _, rep, hist = eng.solve(hologram(nx, ny, nx + nz) if b is None else b, cfg)
    eng.export_coo()
    eng.close()
    print(f"{nx}x{ny}x{nz} T={T}: {rep.iterations} it, guard fix-ups {rep.guard_fixups}, obj {hist[-1]:.6g}",
          flush=True)
    return rep


def group(nx, ny, nz, nranks):
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
    cfg = native_config(SolverConfig(weights=RegularizerWeights(0.05, 0.1), max_iters=2))
    b = hologram(nx, ny, 7)
    engs = HoloEngine.local_group(g, nranks)
    out = [None] * nranks
    th = [threading.Thread(target=lambda r=r: out.__setitem__(r, engs[r].solve(b, cfg))) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in engs:
        e.close()
    print(f"rank group x{nranks}: {[o[1].iterations for o in out]}", flush=True)


if __name__ == "__main__":
    torch.cuda.init()
    which = sys.argv[1:] or ["strip", "walk", "generic", "group", "guard"]
    if "strip" in which:
        solve(128, 128, 8, 5)
    if "walk" in which:
        solve(256, 128, 6, 13)
    if "generic" in which:
        solve(32, 32, 4, 5)
    if "group" in which:
        group(128, 128, 6, 2)
    if "guard" in which:
        b = np.zeros((256, 256))
        b[60:140, 90:200] = 1.0
        rep = solve(256, 256, 1, 5, lam=(0.02, 1.0), iters=2, z0=0.0, b=b)
        assert rep.guard_fixups > 0
