"""Per-kernel device time of one GP NLL+grad step (n=4096), CUPTI via
torch.profiler, eager launches: python tools/kernel_times_gp.py"""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import gp  # noqa: E402

n, d = 4096, 8
torch.manual_seed(0)
x = torch.randn(1, n, d, dtype=torch.float64, device="cuda")
y = torch.randn(1, n, 1, dtype=torch.float64, device="cuda")
g = gp.GPNLL(n, d, 1, "cuda")
for _ in range(3):
    g.step(x, y, 1.0, 1.0, 0.1)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        g.step(x, y, 1.0, 1.0, 0.1)
    torch.cuda.synchronize()
tot = collections.defaultdict(lambda: [0.0, 0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name[:60]
        tot[k][0] += e.device_time_total / 3
        tot[k][1] += 1
for k, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{t:9.1f} us  n={c // 3:4d}  {k}")
