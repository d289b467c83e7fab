"""Sparsity-aware forward A/B (HOLO_NO_PLANE_SKIP): a 1024^2 x 256 volume whose
particles sit in the first 64 planes' depth range, solved at several lambda_L1
with plane skipping on and off.  Prints per-run solve time, dead planes at the
end and the planes the forward passes skipped.  usage: time_plane_skip.py [iters]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_04884_b200 import RegularizerWeights, SolverConfig, VolumeGeometry, synth  # noqa: E402
from paper_1904_04884_b200.engine import HoloEngine  # noqa: E402
from paper_1904_04884_b200.solver import native_config  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nx = ny = 1024
nz = 256
g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
slab = VolumeGeometry(nx, ny, 64, 10e-6, 10e-6, 5e-3, 632e-9)
sc = synth.generate_scene(400, slab, 20e-6, seed=5, margin_planes=2)
b = synth.invert_residual(synth.add_noise(synth.render_hologram(sc), 0.02, seed=11))
bd = torch.as_tensor(b, dtype=torch.float64, device="cuda")


def engine(skip):
    if skip:
        os.environ.pop("HOLO_NO_PLANE_SKIP", None)
    else:
        os.environ["HOLO_NO_PLANE_SKIP"] = "1"
    e = HoloEngine(g)
    os.environ.pop("HOLO_NO_PLANE_SKIP", None)
    return e


engs = {True: engine(True), False: engine(False)}
for l1 in (0.5, 1.5, 3.0):
    cfg = native_config(SolverConfig(weights=RegularizerWeights(l1, 0.2), max_iters=iters, tv_inner_iters=5,
                                     step_size=1.0 / (2 * nz)))
    res = {}
    for rep in range(2):
        for skip in (True, False):
            e = engs[skip]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            code, r, hist = e.solve(bd, cfg, stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            per = e.plane_nnz()
            res[skip] = (hist[-1], per.copy())
            print(f"lambda_L1 {l1} skip {int(skip)} rep {rep}: {dt * 1e3:8.1f} ms  "
                  f"{nx * ny * nz * r.iterations / dt:.3e} voxel-iter/s  it {r.iterations}  "
                  f"dead planes {int((per == 0).sum())}/{nz}  skipped {r.skipped_planes}  "
                  f"nnz {int(per.sum())}  obj {hist[-1]:.9g}", flush=True)
    same = res[True][0] == res[False][0] and np.array_equal(res[True][1], res[False][1])
    print(f"lambda_L1 {l1}: skip/no-skip objective and per-plane nnz identical: {same}", flush=True)
