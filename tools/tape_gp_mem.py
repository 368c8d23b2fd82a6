"""make_gp (dl/models.hpp:115-135) on the device tape at n = 4096, d = 8:
node-value memory with the memory plan off / on, and forward + backward time
(the tape's many small nodes vs the fused GP driver, paper_1710_08717_b200.gp).

    python tools/tape_gp_mem.py [n]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1710_08717_b200 import tape as TP  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
r = O.rng(1234)
x, y = r.standard_normal((n, 8)), r.standard_normal((n, 1))
out = {"n": n}
for plan in (False, True):
    g = TP.Graph()
    m = TP.make_gp(g, x, y, 1.0, 1.0, 0.1)
    g.set_use_memory_plan(plan)
    g.forward()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        g.forward()
        gs = g.backward(m["loss"])
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    out["plan_on" if plan else "plan_off"] = {
        "peak_node_bytes": g.peak_bytes, "nodes": g.num_nodes(), "hand_offs": g.planned_reuse_count(),
        "fwd_bwd_ms": ms, "nll": float(g.value(m["loss"]).item()),
        "grad_log_sigma2": float(gs.at(m["log_sigma2"]).item())}
print(json.dumps(out))
