"""Rank-64 update throughput (the blocked Cholesky's trailing SYRK shape):
C[m, m] += A[m, 64] A^T through the C-ABI GEMM, fp64, CUDA-event timed.
    python tools/syrk_k64.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

for m in (3968, 2048, 1024):
    for k in (64, 128, 256):
        a = torch.randn(1, m, k, dtype=torch.float64, device="cuda")
        c = torch.randn(1, m, m, dtype=torch.float64, device="cuda")
        for _ in range(3):
            L.gemm_into(c, a, a, False, True, -1.0, 1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        R = 20
        for _ in range(R):
            L.gemm_into(c, a, a, False, True, -1.0, 1.0)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / R
        print(f"m={m} k={k}: {ms * 1e3:8.1f} us  {2 * m * m * k / ms / 1e9:6.1f} TF/s  "
              f"C traffic {16 * m * m / ms / 1e6:6.0f} GB/s")
