"""Per-kernel time breakdown (torch.profiler / CUPTI) of one C5 step.

    python tools/timeline_c5.py [batch]
"""
import collections
import json
import math
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200.c5 import MarginalLikelihoods  # noqa: E402

B, n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192, 128
x = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
s = x @ x.transpose(-1, -2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
y = torch.randn(B, n, 1, dtype=torch.float64, device="cuda")
m = MarginalLikelihoods(B, n)
for _ in range(3):
    m.step(s, y, math.log(0.3))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m.step(s, y, math.log(0.3))
    torch.cuda.synchronize()
out = "gpurun_out/timeline_c5.json"
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
tot = collections.OrderedDict()
for e in ev:
    nm = e["name"].replace("dlab::(anonymous namespace)::", "").replace("void ", "")[:90]
    print(f"{e['ts'] - t0:9.1f} +{e['dur']:8.1f} s{e['args'].get('stream')} {nm} grid {e['args'].get('grid')}")
print("span", ev[-1]["ts"] + ev[-1]["dur"] - t0, "us; kernel sum", sum(e["dur"] for e in ev))
