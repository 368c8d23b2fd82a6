"""C1 fused-chain latency probe: device time per launch vs batch (graph-replayed,
200 back-to-back launches).  Used to pick the latency/throughput kernel split."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1710_08717_b200 import linalg as L  # noqa: E402

n = 32
for B in [1, 8, 64, 148, 296, 297, 592, 4096]:
    r = O.rng(7)
    a0 = torch.from_numpy(O.random_spd(n, r, batch=B)).cuda()
    y0 = torch.from_numpy(r.standard_normal((B, n, 1))).cuda()
    phi = torch.empty(B, dtype=torch.float64, device="cuda")
    ab, yb = torch.empty_like(a0), torch.empty_like(y0)
    info = torch.zeros(B, dtype=torch.int32, device="cuda")
    f = lambda: L.chol_chain_fwdbwd(a0, y0, phi, ab, yb, check=False, info=info)  # noqa: E731
    g = bench.graphed(torch, f)
    ms = bench.timed(torch, g, 200, 5, 1)
    print(f"B={B:5d}  {ms * 1e3:8.2f} us/launch  {B / ms * 1e3 / 1e6:7.3f} M mat/s", flush=True)
