"""The fused C1 chain at a given batch, a few calls (ncu target).
    python tools/c1_once.py [batch reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (input generator only)
from paper_1710_08717_b200 import linalg as L  # noqa: E402

B, R = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (64, 5)))
r = O.rng(7)
a = torch.from_numpy(O.random_spd(32, r, batch=B)).cuda()
y = torch.from_numpy(r.standard_normal((B, 32, 1))).cuda()
phi = torch.empty(B, dtype=torch.float64, device="cuda")
ab, yb = torch.empty_like(a), torch.empty_like(y)
info = torch.zeros(B, dtype=torch.int32, device="cuda")
for _ in range(R):
    L.chol_chain_fwdbwd(a, y, phi, ab, yb, check=False, info=info)
torch.cuda.synchronize()
