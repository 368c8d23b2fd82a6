"""One fp32 4096^3 GEMM (tcgen05 3xTF32 path) for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

n = 4096
x = torch.randn(1, n, n, device="cuda")
y = torch.randn(1, n, n, device="cuda")
c = torch.empty_like(x)
for _ in range(2):
    L.gemm2_into(c, x, y)
torch.cuda.synchronize()
