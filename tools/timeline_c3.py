"""Per-kernel breakdown (torch.profiler / CUPTI) of one C3 step (gelqf fwd+bwd,
batch 256 of 128 x 512, fp64) and one C4 step (syevd fwd+bwd, 1024 x 64^2).

    python tools/timeline_c3.py"""
import collections
import json
import os
import re
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

torch.manual_seed(0)
f = dict(dtype=torch.float64, device="cuda")
B, m, n = 256, 128, 512
a0 = torch.cat([torch.eye(m, **f).expand(B, m, m), torch.randn(B, m, n - m, **f)], dim=2).contiguous()
qb = torch.randn(B, m, n, **f)
lb = torch.randn(B, m, m, **f).tril()
q = torch.empty_like(a0)
l = torch.empty(B, m, m, **f)
ab = torch.empty_like(a0)


def c3():
    q.copy_(a0)
    L.gelqf_inplace(q, l, check=False)
    L.gelqf_backward_into(ab, qb, lb, q, l)


x = torch.randn(1024, 64, 64, **f)
s0 = 0.5 * (x + x.transpose(-1, -2))


def c4():
    lam, u = L.syevd(s0)
    L.syevd_backward(torch.randn_like(lam), torch.randn_like(u), lam, u)


for name, fn in (("C3", c3), ("C4", c4)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    path = f"gpurun_out/timeline_{name}.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        k = re.sub(r"\(.*", "", e["name"]).replace("void ", "").replace("dlab::(anonymous namespace)::", "")[:70]
        agg[k][0] += 1
        agg[k][1] += e["dur"]
    ev.sort(key=lambda e: e["ts"])
    span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
    print(f"== {name}: span {span:.1f} us, kernel sum {sum(v[1] for v in agg.values()):.1f} us")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]:
        print(f"  {t:9.1f} {c:3d} {k}")
