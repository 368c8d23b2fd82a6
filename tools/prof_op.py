"""Run one operator a few times (for ncu launch lists / captures).

    python tools/prof_op.py potrf|potrf_bwd|trsm|trsv|syevd|gelqf n [reps] [batch]
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
    f = dict(dtype=torch.float64, device="cuda")
    if op == "syevd":
        x = torch.randn(batch, n, n, **f)
        a0 = 0.5 * (x + x.transpose(-1, -2))
        u = torch.empty_like(a0)
        lam = torch.empty(batch, n, **f)
        ub, lb, ab = torch.randn_like(a0), torch.randn(batch, n, **f), torch.empty_like(a0)
        for _ in range(reps):
            u.copy_(a0)
            L.syevd_inplace(u, lam, check=False)
            L.syevd_backward_into(ab, ub, lb, u, lam)
        torch.cuda.synchronize()
        return
    if op == "gelqf":  # m = n, cols = 4 n (C3: 128 x 512)
        a0 = torch.randn(batch, n, 4 * n, **f)
        q = torch.empty_like(a0)
        l = torch.empty(batch, n, n, **f)
        qb, lb, ab = torch.randn_like(a0), torch.tril(torch.randn_like(l)), torch.empty_like(a0)
        for _ in range(reps):
            q.copy_(a0)
            L.gelqf_inplace(q, l, check=False)
            L.gelqf_backward_into(ab, qb, lb, q, l)
        torch.cuda.synchronize()
        return
    x = torch.randn(batch, n, n, **f)
    a0 = x @ x.transpose(-1, -2) + n * torch.eye(n, **f)
    l = L.potrf(a0)
    lb = torch.tril(torch.randn_like(l))
    ab = torch.empty_like(l)
    a = torch.empty_like(a0)
    for _ in range(reps):
        if op == "potrf":
            a.copy_(a0)
            L.potrf_inplace(a, check=False)
        elif op == "potrf_bwd":
            L.potrf_backward_into(ab, lb, l)
        elif op == "trsm":
            L.trsm_inplace(l, x.clone(), True, False, True, 1.0, check=False)
        elif op == "trsv":
            L.trsm_inplace(l, torch.randn(batch, n, 1, **f), check=False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
