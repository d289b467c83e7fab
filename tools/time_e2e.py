"""Break down the public fista() call (host buffers) into phases."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_04884_b200 import ComplexField2D, RegularizerWeights, SolverConfig, VolumeGeometry
from paper_1904_04884_b200.engine import session
from paper_1904_04884_b200.solver import native_config, _check_b
from paper_1904_04884_b200.sparsevol import SparseVolume
import bench

it = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = bench.CONFIGS["c3"]
b = bench.make_hologram(cfg, torch.device("cuda", 0))
g = VolumeGeometry(1024, 1024, 512, 10e-6, 10e-6, 5e-3, 632e-9)
scfg = SolverConfig(weights=RegularizerWeights(0.5, 0.2), max_iters=it)
for rep in range(2):
    t = [time.perf_counter()]
    bb = _check_b(ComplexField2D(b, 10e-6, 632e-9), g); t.append(time.perf_counter())
    eng = session(g); t.append(time.perf_counter())
    code, r, hist = eng.solve(bb, native_config(scfg)); t.append(time.perf_counter())
    per = eng.plane_nnz(); t.append(time.perf_counter())
    per, rows, cols, vals = eng.export_coo(); t.append(time.perf_counter())
    vol = SparseVolume.from_coo(g, per, rows, cols, vals); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: check {d[0]:.1f} session {d[1]:.1f} solve {d[2]:.1f} (wall_time {r.wall_time*1e3:.1f}) nnz-count {d[3]:.1f} export {d[4]:.1f} from_coo {d[5]:.1f} ms  nnz={r.nnz}", flush=True)
