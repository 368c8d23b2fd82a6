"""Kernel timeline (torch.profiler / CUPTI) of one potrf fwd + bwd call.

    python tools/timeline_op.py n batch [out.json]
"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

n, B = int(sys.argv[1]), int(sys.argv[2])
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/timeline_op.json"
torch.manual_seed(0)
f = dict(dtype=torch.float64, device="cuda")
xx = torch.randn(B, n, n, **f)
spd = xx @ xx.transpose(-1, -2) + n * torch.eye(n, **f)
spd = 0.5 * (spd + spd.transpose(-1, -2))
a = spd.clone()
lbar = torch.randn(B, n, n, **f).tril()
info = torch.zeros(B, dtype=torch.int32, device="cuda")


def step():
    a.copy_(spd)
    L.potrf_inplace(a, check=False, info=info)
    return L.potrf_backward(lbar, a)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev:
    nm = e["name"].replace("dlab::(anonymous namespace)::", "").replace("void ", "")[:70]
    print(f"{e['ts'] - t0:9.1f} +{e['dur']:8.1f} s{e['args'].get('stream')} {nm} grid {e['args'].get('grid')}")
