"""Per-plane kernel times vs volume depth (does a small, L2-sized volume run
its FFT passes faster per plane?).  usage: l2_probe.py [nz ...]"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_04884_b200 import RegularizerWeights, SolverConfig, VolumeGeometry, _native as nat
from paper_1904_04884_b200.engine import HoloEngine
from paper_1904_04884_b200.solver import native_config
lib = nat.load()
rng = np.random.default_rng(0)
b = torch.as_tensor(rng.standard_normal((1024, 1024)) * 0.05, dtype=torch.float64, device="cuda")
for nz in [int(x) for x in sys.argv[1:]] or [4, 8, 16, 512]:
    g = VolumeGeometry(1024, 1024, nz, 10e-6, 10e-6, 5e-3, 632e-9)
    eng = HoloEngine(g)
    cfg = native_config(SolverConfig(weights=RegularizerWeights(0.5, 0.2), max_iters=10))
    eng.solve(b, cfg)
    lib.holo_profile_enable(eng.h, 1)
    eng.solve(b, cfg)
    n = ctypes.c_int32(); names = ctypes.create_string_buffer(32 * 16); ms = (ctypes.c_double * 16)(); cnt = (ctypes.c_int64 * 16)()
    lib.holo_profile_read(eng.h, ctypes.byref(n), names, ms, cnt)
    out = {}
    for i in range(n.value):
        nm = names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode()
        if cnt[i]: out[nm] = ms[i] / cnt[i] / nz * 1e3  # us per plane per launch
    print(f"nz={nz:4d} us/plane/launch:", {k: round(v, 2) for k, v in out.items() if k in ("adj_cols", "adj_rows", "prox", "fwd_rows", "fwd_cols")}, flush=True)
    eng.close()
