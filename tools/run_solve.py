"""Run one device-resident fista solve (for ncu / timing).  usage: run_solve.py nx ny nz iters [T]"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_04884_b200 import VolumeGeometry
from paper_1904_04884_b200.engine import HoloEngine
from paper_1904_04884_b200.solver import SolverConfig, native_config
from paper_1904_04884_b200.prox import RegularizerWeights
from oracle.holo_oracle import Geometry, make_scene, render_hologram, invert_residual, add_noise

nx, ny, nz, iters = map(int, sys.argv[1:5])
T = int(sys.argv[5]) if len(sys.argv) > 5 else 5
g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
if nx * ny > 1024 * 1024:  # large planes: the package's GPU render (the oracle's CPU render is minutes)
    from paper_1904_04884_b200 import synth
    sc = synth.generate_scene(2000, g, 20e-6, seed=3, margin_planes=2)
    b = synth.invert_residual(synth.add_noise(synth.render_hologram(sc), 0.02, seed=10))
else:
    og = Geometry.of(g)
    pts = make_scene(200, og, 20e-6, seed=3, margin_planes=2)
    b = invert_residual(add_noise(render_hologram(pts, og, 20e-6), 0.02, seed=10))
eng = HoloEngine(g)
cfg = native_config(SolverConfig(weights=RegularizerWeights(0.5, 0.2), max_iters=iters, tv_inner_iters=T))
bd = torch.as_tensor(b, dtype=torch.float64, device="cuda")
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    code, r, hist = eng.solve(bd, cfg, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"solve {rep}: {dt*1e3:.1f} ms  {nx*ny*nz*r.iterations/dt:.3e} voxel-iter/s  obj {hist[-1]:.6g}", flush=True)
