"""Generate tests/golden/ref_vectors.npz from the REAL reference.

Runs oracle/_ref/libdla_ref.so (compiled from /root/reference/proj/include by
oracle/Makefile) on seeded Philox inputs and stores inputs + outputs, so the
oracle restatement and the GPU path can be pinned to the reference's own
outputs even where /root/reference is absent (the GPU box).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def main():
    O.build(ref=True)
    ref = O.ref()
    r = O.rng(20260816)
    out = {}
    for n in (3, 32, 70):
        a = O.random_spd(n, r)
        for lower in (1, 0):
            name = f"potrf:{n}:{lower}"
            l = ref.potrf(a, lower)
            lbar = r.standard_normal((n, n))
            out[name + "/a"], out[name + "/l"] = a, l
            out[name + "/lbar"], out[name + "/abar"] = lbar, ref.potrf_bwd(lbar, l, lower)
    for flags in ("000", "011", "101", "110"):
        right, tr, lo = (int(c) for c in flags)
        m, n = 9, 6
        nt = n if right else m
        t = r.standard_normal((nt, nt))
        t[np.diag_indices(nt)] = np.abs(t[np.diag_indices(nt)]) + 2
        x = r.standard_normal((m, n))
        name = f"trsm:{m}x{n}:{flags}"
        out[name + "/t"], out[name + "/x"] = t, x
        out[name + "/y"] = ref.trsm(t, x, right, tr, lo, 0.8)
    a = r.standard_normal((16, 40))
    q, l = ref.gelqf(a)
    out["gelqf:16x40/a"], out["gelqf:16x40/q"], out["gelqf:16x40/l"] = a, q, l
    a = O.random_sym(24, r)
    u, lam = ref.syevd(a)
    out["syevd:24/a"], out["syevd:24/u"], out["syevd:24/lam"] = a, u, lam
    x = r.standard_normal((96, 8))
    y = r.standard_normal((96, 1))
    out["gp:96/x"], out["gp:96/y"] = x, y
    o, xb, yb = ref.gp_nll_grad(x, y, 1.0, 1.0, 0.1, with_xy=True)
    out["gp:96/out"], out["gp:96/xbar"], out["gp:96/ybar"] = o, xb, yb
    x = r.standard_normal((300, 8))
    y = r.standard_normal((300, 1))
    o, xb, yb = ref.gp_nll_grad(x, y, 1.3, 0.7, 0.05, with_xy=True)
    out["gp:300/x"], out["gp:300/y"], out["gp:300/out"] = x, y, o
    out["gp:300/xbar"], out["gp:300/ybar"] = xb, yb
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.npz")
    np.savez_compressed(dst, **out)
    print("wrote", dst, len(out), "arrays")


if __name__ == "__main__":
    main()
