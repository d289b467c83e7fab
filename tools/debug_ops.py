"""Operator parity sweep vs the fp64 oracle over plane shapes (GPU)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_04884_b200 import VolumeGeometry
from paper_1904_04884_b200.engine import HoloEngine
from oracle import holo_oracle as O

def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

rng = np.random.default_rng(0)
for (nx, ny, nz) in [(256, 256, 4), (512, 512, 2), (1024, 256, 2), (256, 1024, 2), (1024, 1024, 1), (1024, 1024, 4), (2048, 64, 1), (64, 2048, 1)]:
    g = VolumeGeometry(nx, ny, nz, 10e-6, 10e-6, 5e-3, 632e-9)
    og = O.Geometry.of(g)
    eng = HoloEngine(g)
    x = (rng.standard_normal((nz, ny, nx)) + 1j * rng.standard_normal((nz, ny, nx))) * (rng.random((nz, ny, nx)) < 0.01)
    r = rng.standard_normal((ny, nx))
    f_gpu, f_ref = eng.forward(x), O.sensor_forward(x, og)
    a_gpu, a_ref = eng.adjoint(r), O.back_project(r, og)
    h_gpu, h_ref = eng.transfer(0, nz), O.transfer_stack(og, 0, nz)
    X = rng.standard_normal((1, ny, nx)) + 1j * rng.standard_normal((1, ny, nx))
    print(f"{nx}x{ny}x{nz}: transfer {np.max(np.abs(h_gpu-h_ref)):.2e} fwd {rel(f_gpu, f_ref):.2e} adj {rel(a_gpu, a_ref):.2e} "
          f"fft2 {rel(eng.fft2(X), np.fft.fft2(X)):.2e} ifft2 {rel(eng.fft2(X, inverse=True), np.fft.ifft2(X)):.2e}", flush=True)
    eng.close()
