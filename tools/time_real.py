"""Real-nonnegative engine timing on a C3-sized volume (per-kernel ms per solve)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1904_04884_b200 import RegularizerWeights, SolverConfig, VolumeGeometry, _native as nat
from paper_1904_04884_b200.engine import HoloEngine
from paper_1904_04884_b200.solver import native_config
cfgn = sys.argv[1] if len(sys.argv) > 1 else "c3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = bench.CONFIGS[cfgn]
nx, ny, nz, _, _, _, l1, tv, inner, _ = cfg
g = VolumeGeometry(nx, ny, nz, bench.PITCH, bench.DZ, bench.Z0, bench.LAM)
b = torch.as_tensor(bench.make_hologram(cfg), dtype=torch.float64, device="cuda")
eng = HoloEngine(g)
step = 1.0 / (2.0 * eng.operator_norm(real=True))
lib = nat.load()
for real in (False, True):
    ncfg = native_config(SolverConfig(weights=RegularizerWeights(l1, tv), max_iters=iters, tv_inner_iters=inner,
                                      real_nonnegative=real, step_size=step if real else None))
    eng.solve(b, ncfg)
    lib.holo_profile_enable(eng.h, 1)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(); _, rep, hist = eng.solve(b, ncfg); ev1.record(); torch.cuda.synchronize()
    n = ctypes.c_int32(); names = ctypes.create_string_buffer(32 * 16); ms = (ctypes.c_double * 16)(); cnt = (ctypes.c_int64 * 16)()
    lib.holo_profile_read(eng.h, ctypes.byref(n), names, ms, cnt)
    lib.holo_profile_enable(eng.h, 0)
    prof = {names.raw[32*i:32*i+32].split(b"\0")[0].decode(): round(ms[i], 2) for i in range(n.value)}
    print(f"{cfgn} real={real}: {ev0.elapsed_time(ev1):.1f} ms, {rep.iterations} it, obj {hist[-1]:.6g}, nnz {rep.nnz}", prof, flush=True)
