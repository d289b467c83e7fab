"""Device-resident timing of holo_op_prox_fl (all passes of one prox call) on a
random 1024^2 stack.  usage: time_prox_op.py [nplanes] [T ...]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_04884_b200 import _native as nat
from paper_1904_04884_b200.engine import prox_session

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
Ts = [int(t) for t in sys.argv[2:]] or [5, 20]
eng = prox_session()
g = torch.Generator(device="cuda").manual_seed(0)
v = (0.3 * torch.randn(n, 1024, 1024, 2, device="cuda", generator=g)).contiguous()
out = torch.empty_like(v)
s = torch.cuda.current_stream()
for T in Ts:
    call = lambda: nat.check(eng.lib.holo_op_prox_fl(eng.h, ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(out.data_ptr()), n,
                                                     1024, 1024, 0.02, 1.0 if T > 8 else 0.2, T, ctypes.c_void_p(s.cuda_stream)), "prox")
    for _ in range(2):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        call()
    e1.record()
    torch.cuda.synchronize()
    print(f"T={T} planes={n}: {e0.elapsed_time(e1) / 5:.3f} ms per prox call ({e0.elapsed_time(e1) / 5 / n * 512:.2f} ms per 512 planes)")
