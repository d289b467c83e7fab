"""Per-kernel-class times of a device-resident solve, power-of-two vs general
plane sides.  usage: time_general.py nx ny nz iters [T]"""
import ctypes, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_04884_b200 import VolumeGeometry, synth
from paper_1904_04884_b200.engine import HoloEngine
from paper_1904_04884_b200.solver import SolverConfig, native_config
from paper_1904_04884_b200.prox import RegularizerWeights

nx, ny, nz, iters = map(int, sys.argv[1:5])
T = int(sys.argv[5]) if len(sys.argv) > 5 else 5
g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
sc = synth.generate_scene(max(50, nz * 4), g, 20e-6, seed=3, margin_planes=2)
b = synth.invert_residual(synth.add_noise(synth.render_hologram(sc), 0.02, seed=10))
eng = HoloEngine(g)
lib = eng.lib
cfg = native_config(SolverConfig(weights=RegularizerWeights(0.5, 0.2), max_iters=iters, tv_inner_iters=T))
bd = torch.as_tensor(b, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
eng.solve(bd, cfg, stream=st)
lib.holo_profile_classes(eng.h, 0xFFFFFFFF)
lib.holo_profile_enable(eng.h, 1)
torch.cuda.synchronize(); t0 = time.perf_counter()
code, r, hist = eng.solve(bd, cfg, stream=st)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
n = ctypes.c_int32(); names = ctypes.create_string_buffer(32 * 16)
kms = (ctypes.c_double * 16)(); kcnt = (ctypes.c_int64 * 16)()
lib.holo_profile_read(eng.h, ctypes.byref(n), names, kms, kcnt)
prof = {names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): round(kms[i], 2) for i in range(n.value)}
print(f"{nx}x{ny}x{nz} T={T} {r.iterations} it: {dt*1e3:.1f} ms  {nx*ny*nz*r.iterations/dt:.3e} voxel-iter/s  {prof}",
      flush=True)
