"""Kernel timeline (torch.profiler / CUPTI) of one potrf fwd + bwd step through
the fused split entry points, in CUDA graph replay as bench.py times it.

    python tools/timeline_potrf_split.py [n] [batch] [out.json]
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402  (input generator only)
from paper_1710_08717_b200._lib import lib as _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/timeline_potrf_split.json"
lib = _lib().lib
r = O.rng(11)
a0 = torch.from_numpy(O.random_spd(n, r, batch=B)).cuda()
lb0 = torch.from_numpy(np.tril(r.standard_normal((B, n, n)))).cuda()
a, ab = torch.empty_like(a0), torch.empty_like(a0)
info = torch.zeros(B, dtype=torch.int32, device="cuda")
nb = int(lib.dla_potrf_bwd_ws_bytes_f64(B, n))
ws = torch.empty(max(nb, 8), dtype=torch.uint8, device="cuda")
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def step():
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    a.copy_(a0)
    assert lib.dla_gp_potrf_inv_f64(B, n, P(a), P(info), P(ws), nb, st) == 0
    assert lib.dla_potrf_bwd_end_f64(B, n, P(ab), P(lb0), P(a), 1, P(ws), nb, st) == 0


g = bench.graphed(torch, step)
for _ in range(3):
    g()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g()
    torch.cuda.synchronize()
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev:
    print(f"{e['ts'] - t0:8.1f} +{e['dur']:7.1f} s{e['args'].get('stream')} {e['name'][:70]} grid {e['args'].get('grid')}")
print(f"span {max(e['ts'] + e['dur'] for e in ev) - t0:.1f} us")
