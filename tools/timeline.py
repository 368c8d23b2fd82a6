"""Kernel timeline of one potrf n=4096 (torch.profiler / CUPTI): per-kernel
start/end on every stream, summarised as the critical-chain gaps.

    python tools/timeline.py [n] [out.json] [batch]
"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline.json"
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
torch.manual_seed(0)
xx = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
spd = xx @ xx.transpose(-1, -2)
spd = 0.5 * (spd + spd.transpose(-1, -2)) + n * torch.eye(n, dtype=torch.float64, device="cuda")
a = spd.clone()
info = torch.zeros(B, dtype=torch.int32, device="cuda")
for _ in range(3):
    a.copy_(spd)
    L.potrf_inplace(a, check=False, info=info)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    a.copy_(spd)
    L.potrf_inplace(a, check=False, info=info)
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
rows = []
for e in ev:
    nm = e["name"]
    short = "panel" if "potrf_panel" in nm else ("gemm128" if "128, 128" in nm else ("gemm64" if "64, 64" in nm else nm[:30]))
    rows.append((e["ts"] - t0, e["dur"], e["args"].get("stream"), short, e["args"].get("grid")))
for r in rows[:40]:
    print(f"{r[0]:9.1f} +{r[1]:7.1f} us  stream {r[2]}  {r[3]:10s} grid {r[4]}")
print("...")
for r in rows[-12:]:
    print(f"{r[0]:9.1f} +{r[1]:7.1f} us  stream {r[2]}  {r[3]:10s} grid {r[4]}")
tot = rows[-1][0] + rows[-1][1]
by = {}
for r in rows:
    by.setdefault(r[3], [0, 0.0])
    by[r[3]][0] += 1
    by[r[3]][1] += r[1]
print(f"total span {tot:.1f} us; busy per kind:", {k: (v[0], round(v[1], 1)) for k, v in by.items()})
