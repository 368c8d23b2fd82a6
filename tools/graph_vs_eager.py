"""potrf / GP step timing eager vs CUDA-graph replay (look-ahead streams in graphs)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1710_08717_b200 import linalg as L  # noqa: E402

for n, B in ((4096, 1), (1024, 8)):
    x = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
    a0 = x @ x.transpose(-1, -2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
    a = torch.empty_like(a0)
    info = torch.zeros(B, dtype=torch.int32, device="cuda")

    def step():
        a.copy_(a0)
        L.potrf_inplace(a, check=False, info=info)

    e = bench.timed(torch, step, 10, 3, 1)
    g = bench.timed(torch, bench.graphed(torch, step), 10, 3, 1)
    print(f"potrf n={n} B={B}: eager {e:.3f} ms, graph {g:.3f} ms")
