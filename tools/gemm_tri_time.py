"""Event-timed f64 products of the potrf pullback through the library's GEMM
(plain 4096^3 and the three triangular products P' = tril(L^T Lbar),
W = P' L^-1, Z = L^-T W, via the gemm profiling hook), for A/B of the
DLA_GEMM_TMA switch:   DLA_GEMM_TMA=0|1 python tools/gemm_tri_time.py [n B]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402
from paper_1710_08717_b200._lib import lib  # noqa: E402

n, B = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 1)))
torch.manual_seed(0)
f = dict(dtype=torch.float64, device="cuda")
a = torch.randn(B, n, n, **f)
c = torch.empty(B, n, n, **f)
for _ in range(2):
    L.gemm_into(c, a, a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    L.gemm_into(c, a, a)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"plain {n}^3 x{B}: {ms * 1e3:8.1f} us {2 * B * n ** 3 / ms / 1e9:6.1f} TF/s")
x = torch.randn(B, n, n, **f)
spd = x @ x.transpose(-1, -2) + n * torch.eye(n, **f)
l = L.potrf(0.5 * (spd + spd.transpose(-1, -2)))
lbar = torch.randn(B, n, n, **f).tril()
lib_ = lib().lib
for _ in range(2):
    L.potrf_backward(lbar, l)
torch.cuda.synchronize()
lib_.dla_prof_enable(1)
for _ in range(3):
    L.potrf_backward(lbar, l)
torch.cuda.synchronize()
ms, fl = C.c_double(), C.c_double()
cnt = lib_.dla_prof_read(C.byref(ms), C.byref(fl))
mms, mfl = C.c_double(), C.c_double()
lib_.dla_prof_read_max(C.byref(mms), C.byref(mfl))
lib_.dla_prof_enable(0)
print(f"potrf_bwd GEMMs: {cnt} launches, {ms.value / 3 * 1e3:.1f} us per pullback (event-summed), "
      f"{fl.value / (ms.value / 1e3) / 1e12:.1f} TF/s; largest launch {mms.value * 1e3:.1f} us "
      f"{mfl.value / (mms.value / 1e3) / 1e12:.1f} TF/s")
