"""potrf (and optionally its backward) at n = 32, batch 65536, fp64, a few calls (ncu target).
    python tools/potrf32_once.py [bwd]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

B, n = 65536, 32
torch.manual_seed(0)
x = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
spd = x @ x.transpose(-1, -2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
a = torch.empty_like(spd)
info = torch.zeros(B, dtype=torch.int32, device="cuda")
for _ in range(3):
    a.copy_(spd)
    L.potrf_inplace(a, check=False, info=info)
torch.cuda.synchronize()
