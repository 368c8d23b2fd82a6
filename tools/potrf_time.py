"""Event-timed potrf (and potrf fwd+bwd) at the north-star / C2 sizes, fp64.

    python tools/potrf_time.py [n:B ...]     default 4096:1 1024:8 2048:1 512:8
Env tuning switches (DLA_POTRF_*) are read by the library, so one binary can
compare schedules: DLA_POTRF_MODE=3 python tools/potrf_time.py 4096:1
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

cases = [tuple(int(v) for v in s.split(":")) for s in sys.argv[1:]] or [(4096, 1), (1024, 8), (2048, 1), (512, 8)]
torch.manual_seed(0)
for n, B in cases:
    xx = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
    spd = xx @ xx.transpose(-1, -2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
    spd = 0.5 * (spd + spd.transpose(-1, -2))
    a = spd.clone()
    info = torch.zeros(B, dtype=torch.int32, device="cuda")
    lbar = torch.randn(B, n, n, dtype=torch.float64, device="cuda").tril()
    R = 10 if n >= 2048 else 20

    def fwd():
        a.copy_(spd)
        L.potrf_inplace(a, check=False, info=info)

    for _ in range(3):
        fwd()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    # the copy alone, to subtract
    e[0].record()
    for _ in range(R):
        a.copy_(spd)
    e[1].record()
    for _ in range(R):
        fwd()
    e[2].record()
    torch.cuda.synchronize()
    cp = e[0].elapsed_time(e[1]) / R
    ms = e[1].elapsed_time(e[2]) / R - cp
    ref = torch.linalg.cholesky(spd)
    err = ((a - ref).abs().max() / ref.abs().max()).item()
    fl = B * n ** 3 / 3
    l = a.clone()
    ab = L.potrf_backward(lbar, l)
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(R):
        ab = L.potrf_backward(lbar, l)
    e[1].record()
    torch.cuda.synchronize()
    mb = e[0].elapsed_time(e[1]) / R
    print(f"n={n} B={B}: potrf {ms * 1e3:8.1f} us ({fl / ms / 1e9:5.1f} TF/s)  bwd {mb * 1e3:8.1f} us "
          f"({4 * fl / mb / 1e9:5.1f} TF/s 4n^3/3)  fwd+bwd {(ms + mb) * 1e3:8.1f} us  "
          f"{B / (ms + mb) * 1e3:8.1f} mat/s  relerr {err:.1e} info {int(info.abs().sum())}", flush=True)
