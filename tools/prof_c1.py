"""The fused C1 chain at batch 64 x 32^2 (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (input generator only)
from paper_1710_08717_b200 import linalg as L  # noqa: E402

r = O.rng(7)
a = torch.from_numpy(O.random_spd(32, r, batch=64)).cuda()
y = torch.from_numpy(r.standard_normal((64, 32, 1))).cuda()
for _ in range(3):
    L.chol_chain_fwdbwd(a, y, check=False)
torch.cuda.synchronize()
