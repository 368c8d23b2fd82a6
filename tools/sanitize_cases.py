"""Small invocations of every kernel family for compute-sanitizer runs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (input generator only)
from paper_1710_08717_b200 import gp  # noqa: E402
from paper_1710_08717_b200 import linalg as L  # noqa: E402

r = O.rng(1)
f = dict(dtype=torch.float64, device="cuda")
for n, B in ((16, 3), (32, 5), (40, 2), (100, 3), (128, 2), (200, 2), (256, 1)):
    a = torch.from_numpy(O.random_spd(n, r, batch=B)).cuda()
    l = L.potrf(a)
    L.potrf_backward(torch.tril(torch.randn_like(l)), l)
    L.potri(l)
    y = torch.randn(B, n, 1, **f)
    L.trsm(l, y)
    L.trsm(l, y, False, True, True)
    L.chol_chain_fwdbwd(a, y)
x = torch.randn(2, 64, 64, **f)
L.syevd(0.5 * (x + x.transpose(-1, -2)))
q = torch.randn(2, 80, 120, **f)
L.gelqf(q)
L.gemm2(torch.randn(2, 130, 70, **f), torch.randn(2, 70, 90, **f))
gp.gp_nll_grad(torch.randn(256, 8, **f), torch.randn(256, 1, **f), 1.0, 1.0, 0.1)
gp.gp_nll_grad(torch.randn(512, 8, **f), torch.randn(512, 1, **f), 1.0, 1.0, 0.1)  # early inverse + fused tail
# single-vector / rank-1 streaming kernels, syrk (TMA at m >= 256), LQ (CholeskyQR2 at m >= 64), SVD
g = torch.randn(4, 128, 128, **f)
v = torch.randn(4, 128, 1, **f)
L.gemm2(g, v)
L.gemm2(g, v, True, False)
L.gemm2(v, v, False, True)
L.syrk(torch.randn(2, 300, 40, **f))
L.gelqf(torch.randn(2, 128, 512, **f))
L.gesvd(torch.randn(2, 40, 60, **f))
# a plain product with >= 2 waves of 128 x 128 tiles: the TMA-fed GEMM (run the
# whole script with DLA_GEMM_TMA=2 to put every product >= 256 on it)
L.gemm2(torch.randn(1, 2560, 300, **f), torch.randn(1, 300, 2560, **f))
# batched Kalman NLL + gradient: the compile-time-size kernels (h = d = 8, 4, 8 x 4) and the runtime-size one
from paper_1710_08717_b200 import kalman as K  # noqa: E402
for h, d, T, B in ((8, 8, 6, 3), (4, 4, 5, 2), (8, 4, 4, 2), (5, 3, 4, 2)):
    m = O.random_kalman(O.rng(3), h, d, T, batch=B)
    K.KalmanNLL(h, d, T, B).step(*[torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in m])
# n = 32 forward, upper output (R = L^T from the lane's shared-memory row)
L.potrf(torch.from_numpy(O.random_spd(32, r, batch=9)).cuda(), False)
torch.cuda.synchronize()
print("sanitize cases done")
