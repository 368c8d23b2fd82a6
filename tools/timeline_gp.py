"""Kernel timeline of one GP NLL+grad step (n=4096): busy time per phase and
the idle gaps on the device (torch.profiler / CUPTI, eager launches).

    python tools/timeline_gp.py [out.json]
"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import gp  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline_gp.json"
n, d = 4096, 8
torch.manual_seed(0)
x = torch.randn(1, n, d, dtype=torch.float64, device="cuda")
y = torch.randn(1, n, 1, dtype=torch.float64, device="cuda")
g = gp.GPNLL(n, d, 1, "cuda")
for _ in range(3):
    g.step(x, y, 1.0, 1.0, 0.1)
torch.cuda.synchronize()
step = lambda: g.step(x, y, 1.0, 1.0, 0.1)  # noqa: E731
if os.environ.get("GRAPH", "1") != "0":  # as bench.py times it: CUDA graph replay
    import bench  # noqa: E402

    step = bench.graphed(torch, step)
    step()
    torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
end = max(e["ts"] + e["dur"] for e in ev)
# union of busy intervals -> idle gaps
busy, cur_s, cur_e = 0.0, None, None
gaps = []
for e in ev:
    s, f = e["ts"], e["ts"] + e["dur"]
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            gaps.append((cur_e - t0, s - cur_e))
            busy += cur_e - cur_s
        cur_s, cur_e = s, f
    else:
        cur_e = max(cur_e, f)
busy += cur_e - cur_s
print(f"span {end - t0:.1f} us, device busy (any kernel) {busy:.1f} us, idle {end - t0 - busy:.1f} us")
for at, gap in sorted(gaps, key=lambda g: -g[1])[:8]:
    nxt = next(e for e in ev if e["ts"] - t0 >= at + gap - 0.01)
    print(f"  gap {gap:7.1f} us at {at:8.1f} before {nxt['name'][:70]}")
# coarse phases in order of first launch
marks = []
for e in ev:
    nm = e["name"]
    key = ("rbf" if "rbf" in nm else "panel" if "potrf_panel" in nm else "trsv" if "trsv" in nm
           else "trtri" if "trtri" in nm else "gemm" if "dgemm" in nm else nm.split("(")[0][-28:])
    marks.append((e["ts"] - t0, e["dur"], e["args"].get("stream"), key))
phase = {}
for t, dur, st, key in marks:
    p = phase.setdefault((key, st), [t, t + dur, 0.0, 0])
    p[0] = min(p[0], t)
    p[1] = max(p[1], t + dur)
    p[2] += dur
    p[3] += 1
for (key, st), (a, b, tot, cnt) in sorted(phase.items(), key=lambda kv: kv[1][0]):
    print(f"{key:30s} stream {st}: [{a:8.1f}, {b:8.1f}] us  busy {tot:8.1f} us  n={cnt}")

if os.environ.get("DUMP"):
    for e in ev:
        print(f"{e['ts'] - t0:9.1f} +{e['dur']:7.1f} s{e['args'].get('stream')} "
              f"{e['name'].replace('dlab::(anonymous namespace)::', '')[:90]}")
