"""Run one operator a few times (for ncu launch lists / captures).

    python tools/prof_op.py potrf 4096 [reps] [batch]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_08717_b200 import linalg as L  # noqa: E402


def main():
    op, n = sys.argv[1], int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    batch = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    torch.manual_seed(0)
    x = torch.randn(batch, n, n, dtype=torch.float64, device="cuda")
    a0 = x @ x.transpose(-1, -2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
    l = L.potrf(a0)
    lb = torch.tril(torch.randn_like(l))
    for _ in range(reps):
        if op == "potrf":
            a = a0.clone()
            L.potrf_inplace(a, check=False)
        elif op == "potrf_bwd":
            L.potrf_backward(lb, l)
        elif op == "trsm":
            L.trsm_inplace(l, x.clone(), True, False, True, 1.0, check=False)
        elif op == "trsv":
            L.trsm_inplace(l, torch.randn(1, n, 1, dtype=torch.float64, device="cuda"), check=False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
