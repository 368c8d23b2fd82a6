"""A few GP NLL+grad steps at n (for ncu captures of the GP-specific kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200.gp import GPNLL  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(1, n, 8, dtype=torch.float64, device="cuda", generator=g)
y = torch.randn(1, n, 1, dtype=torch.float64, device="cuda", generator=g)
m = GPNLL(n, 8, 1, "cuda", want_xbar=True)
for _ in range(2):
    m.step(x, y, 1.0, 1.0, 0.1)
torch.cuda.synchronize()
