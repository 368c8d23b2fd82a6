"""potrf fwd (+ copy) and fwd+bwd at n = 32, batch 65536, fp64: CUDA-graph replay, event timed.
    python tools/potrf32_time.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402  (input generator only)
from paper_1710_08717_b200 import linalg as L  # noqa: E402

n, B = 32, 65536
a0 = torch.from_numpy(O.random_spd(n, O.rng(11), batch=B)).cuda()
a = torch.empty_like(a0)
info = torch.zeros(B, dtype=torch.int32, device="cuda")


def fwd():
    a.copy_(a0)
    L.potrf_inplace(a, True, check=False, info=info)


ms = bench.timed(torch, bench.graphed(torch, fwd), 30, 5, 1)
print(f"copy+fwd {ms * 1e3:.1f} us; fwd+bwd line {bench.run_potrf_batch(torch, n, B, 30, 5, 1) * 1e3:.1f} us")
