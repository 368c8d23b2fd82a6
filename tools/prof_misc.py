"""One launch each of the fused / special kernels for an ncu --set full capture:
k_chol_chain_warp (C1, batch 65536), k_syevd_small (C4), k_lq_panel (C3),
k_potrf_panel + k_trsv (n = 4096)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (input generator only)
from paper_1710_08717_b200 import linalg as L  # noqa: E402

f = dict(dtype=torch.float64, device="cuda")
B = 65536
a = torch.from_numpy(O.random_spd(32, O.rng(3), batch=1)).cuda().expand(B, 32, 32).contiguous()
y = torch.randn(B, 32, 1, **f)
L.chol_chain_fwdbwd(a, y, check=False)
x = torch.randn(1024, 64, 64, **f)
u = 0.5 * (x + x.transpose(-1, -2))
L.syevd_inplace(u, torch.empty(1024, 64, **f), check=False)
q = torch.randn(256, 128, 512, **f)
L.gelqf_inplace(q, torch.empty(256, 128, 128, **f), check=False)
n = 4096
xx = torch.randn(1, n, n, **f)
s = xx @ xx.transpose(-1, -2) + n * torch.eye(n, **f)
L.potrf_inplace(s, check=False)
L.trsm_inplace(s, torch.randn(1, n, 1, **f), check=False)
torch.cuda.synchronize()
