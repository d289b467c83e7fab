"""Time the plain batched 2D FFT (k_fft_rows + k_fft_cols, direct loads and
stores) over a 1024^2 x nz volume: the column pass with both a strided load
and a strided store is what a rows-first adjoint / columns-first forward would
need.  usage: time_fft_passes.py [nz]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_04884_b200 import VolumeGeometry
from paper_1904_04884_b200.engine import HoloEngine

nz = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = VolumeGeometry(1024, 1024, nz, 10e-6, 10e-6, 5e-3, 632e-9)
eng = HoloEngine(g)
x = torch.randn(nz, 1024, 1024, dtype=torch.complex64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    assert eng.lib.holo_op_fft2(eng.h, ctypes.c_void_p(x.data_ptr()), nz, 0, ctypes.c_void_p(s)) == 0
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    eng.lib.holo_op_fft2(eng.h, ctypes.c_void_p(x.data_ptr()), nz, 0, ctypes.c_void_p(s))
b.record()
torch.cuda.synchronize()
print(f"fft2 over {nz} planes: {a.elapsed_time(b) / 5:.3f} ms (rows + cols)")
