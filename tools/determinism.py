"""Two identical solves of a config must agree bit for bit (races in the
TMA / mbarrier pipelines would show up here).  usage: determinism.py [config] [iters]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1904_04884_b200 import RegularizerWeights, SolverConfig, VolumeGeometry
from paper_1904_04884_b200.engine import HoloEngine
from paper_1904_04884_b200.solver import native_config

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = bench.CONFIGS[name]
nx, ny, nz, _, _, _, l1, tv, inner, _ = cfg
g = VolumeGeometry(nx, ny, nz, bench.PITCH, bench.DZ, bench.Z0, bench.LAM)
b = torch.as_tensor(bench.make_hologram(cfg), dtype=torch.float64, device="cuda")
eng = HoloEngine(g)
ncfg = native_config(SolverConfig(weights=RegularizerWeights(l1, tv), max_iters=iters, tv_inner_iters=inner))
outs = []
for _ in range(2):
    _, rep, hist = eng.solve(b, ncfg)
    outs.append((eng.solution_dense().view(torch.float32).clone(), np.array(hist)))
same = torch.equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
print(f"{name} {iters} it: solutions bitwise equal = {same}, max |diff| = "
      f"{(outs[0][0] - outs[1][0]).abs().max().item():.3e}")
sys.exit(0 if same else 1)
