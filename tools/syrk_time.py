"""syrk (f64, A A^T) through the C-ABI: correctness vs torch and event timing.
The TMA trailing-update kernel (syrk_tma.cu) serves it when eligible; DLA_SYRK_TMA=0 compares the generic GEMM.
    python tools/syrk_time.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

torch.manual_seed(0)
for m, k, B in ((3968, 64, 1), (3968, 128, 1), (2048, 64, 1), (1000, 64, 3), (960, 64, 8), (300, 40, 2)):
    a = torch.randn(B, m, k, dtype=torch.float64, device="cuda")
    c = torch.empty(B, m, m, dtype=torch.float64, device="cuda")
    L.syrk_into(c, a, False, -0.5)
    ref = -0.5 * a @ a.transpose(-1, -2)
    err = ((c - ref).abs().max() / ref.abs().max()).item()
    sym = (c - c.transpose(-1, -2)).abs().max().item()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 20
    e0.record()
    for _ in range(R):
        L.syrk_into(c, a, False, -0.5)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    print(f"m={m} k={k} B={B}: {ms * 1e3:8.1f} us (incl. mirror)  {B * m * m * k / ms / 1e9:6.1f} TF/s lower-half  "
          f"relerr {err:.1e} asym {sym}", flush=True)
