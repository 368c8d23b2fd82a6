"""Plain / masked / triangular f64 GEMM timings through the C-ABI (event-timed).
    python tools/gemm_time.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

torch.manual_seed(0)
for (B, m, n, k) in ((1, 4096, 4096, 4096), (8, 1024, 1024, 1024), (512, 128, 128, 128), (1, 4096, 4096, 64)):
    a = torch.randn(B, m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(B, k, n, dtype=torch.float64, device="cuda")
    c = torch.empty(B, m, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        L.gemm_into(c, a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 10
    e0.record()
    for _ in range(R):
        L.gemm_into(c, a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    print(f"gemm B={B} {m}x{n}x{k}: {ms * 1e3:8.1f} us {2 * B * m * n * k / ms / 1e9:6.1f} TF/s", flush=True)
