"""fp32 GEMM on tcgen05 (3xTF32) vs an fp64 torch reference: every
transposition, ragged shapes, batch, alpha/beta; prints the max relative
error and the 4096^3 throughput."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1710_08717_b200 import linalg as L  # noqa: E402

torch.manual_seed(0)
worst = 0.0
for (B, m, n, k) in ((1, 128, 128, 32), (1, 256, 256, 256), (2, 300, 130, 77), (3, 129, 200, 1000), (1, 512, 64, 40)):
    for ta in (False, True):
        for tb in (False, True):
            a = torch.randn(B, *((k, m) if ta else (m, k)), device="cuda")
            b = torch.randn(B, *((n, k) if tb else (k, n)), device="cuda")
            c0 = torch.randn(B, m, n, device="cuda")
            c = c0.clone()
            L.gemm_into(c, a, b, ta, tb, 0.7, 0.3)
            ad, bd = a.double(), b.double()
            ref = 0.7 * (ad.transpose(-1, -2) if ta else ad) @ (bd.transpose(-1, -2) if tb else bd) + 0.3 * c0.double()
            err = ((c.double() - ref).abs().max() / ref.abs().max()).item()
            worst = max(worst, err)
            print(f"B={B} m={m} n={n} k={k} ta={int(ta)} tb={int(tb)} relerr={err:.2e}", flush=True)
print("worst", worst)
n = 4096
x = torch.randn(1, n, n, device="cuda")
y = torch.randn(1, n, n, device="cuda")
c = torch.empty_like(x)
ms = bench.timed(torch, lambda: L.gemm2_into(c, x, y), 5, 2, 1)
print(f"sgemm 4096^3 tcgen05 3xTF32: {ms:.3f} ms, {2 * n ** 3 / ms / 1e9:.1f} TFLOP/s (fp32-accurate)")
