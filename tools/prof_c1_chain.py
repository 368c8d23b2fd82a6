"""One fused C1 chain launch (batch 64 x 32^2 fp64) for ncu:
    ncu --set full -k regex:k_chol_chain_warp python tools/prof_c1_chain.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1710_08717_b200 import linalg as L  # noqa: E402

B, n = 64, 32
r = O.rng(7)
a = torch.from_numpy(O.random_spd(n, r, batch=B)).cuda()
y = torch.from_numpy(r.standard_normal((B, n, 1))).cuda()
phi = torch.empty(B, dtype=torch.float64, device="cuda")
abar, ybar = torch.empty_like(a), torch.empty_like(y)
info = torch.zeros(B, dtype=torch.int32, device="cuda")
for _ in range(3):
    L.chol_chain_fwdbwd(a, y, phi, abar, ybar, check=False, info=info)
torch.cuda.synchronize()
