import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_04884_b200 import VolumeGeometry
from paper_1904_04884_b200.engine import HoloEngine
from oracle import holo_oracle as O
rng = np.random.default_rng(0)
mode = sys.argv[1] if len(sys.argv) > 1 else "sweep"
shapes = [(1024, 1024, 4)] if mode == "one" else [(1024, 1024, 2), (1024, 1024, 3), (1024, 1024, 4), (512, 512, 8), (512, 512, 16), (256, 256, 64), (2048, 2048, 2)]
for (nx, ny, nz) in shapes:
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
    og = O.Geometry.of(g)
    eng = HoloEngine(g)
    r = rng.standard_normal((ny, nx))
    a_gpu = eng.adjoint(r)
    a_ref = O.back_project(r, og)
    errs = [float(np.linalg.norm(a_gpu[k] - a_ref[k]) / np.linalg.norm(a_ref[k])) for k in range(nz)]
    bad = [k for k, e in enumerate(errs) if e > 1e-5]
    print(f"{nx}x{ny}x{nz}: max plane err {max(errs):.2e} bad planes {bad[:10]}", flush=True)
    if bad:
        k = bad[0]
        d = np.abs(a_gpu[k] - a_ref[k])
        iy, ix = np.nonzero(d > 1e-3 * np.abs(a_ref[k]).max())
        print("   bad rows", np.unique(iy)[:20], "n rows", len(np.unique(iy)), "bad cols", np.unique(ix)[:10], len(np.unique(ix)))
    eng.close()
