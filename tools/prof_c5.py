"""One C5 step at a reduced batch (for ncu launch lists)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200.c5 import MarginalLikelihoods  # noqa: E402

B, n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192, 128
x = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
s = x @ x.transpose(-1, -2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
y = torch.randn(B, n, 1, dtype=torch.float64, device="cuda")
m = MarginalLikelihoods(B, n)
for _ in range(1):
    m.step(s, y, math.log(0.3))
torch.cuda.synchronize()
