"""potrf correctness at large n vs torch (cuSOLVER used only as a checker here)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

torch.manual_seed(0)
for n, B in ((4096, 1), (2048, 1), (1024, 8), (1000, 2)):
    xx = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
    spd = xx @ xx.transpose(-1, -2)
    spd = 0.5 * (spd + spd.transpose(-1, -2)) + n * torch.eye(n, dtype=torch.float64, device="cuda")
    a = spd.clone()
    info = torch.zeros(B, dtype=torch.int32, device="cuda")
    L.potrf_inplace(a, check=False, info=info)
    ref = torch.linalg.cholesky(spd)
    err = ((a - ref).abs().max() / ref.abs().max()).item()
    print(f"n={n} B={B} depth={os.environ.get('DLA_POTRF_DEPTH')} info={info.tolist()} relerr={err:.2e}", flush=True)
