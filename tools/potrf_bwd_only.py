"""potrf_backward alone at n x B (fp64), for ncu launch lists / captures.

    python tools/potrf_bwd_only.py [n B reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

n, B, R = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (1024, 8, 3)))
torch.manual_seed(0)
x = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
a = x @ x.transpose(-1, -2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
l = L.potrf(0.5 * (a + a.transpose(-1, -2)))
lbar = torch.randn(B, n, n, dtype=torch.float64, device="cuda").tril()
for _ in range(R):
    L.potrf_backward(lbar, l)
torch.cuda.synchronize()
