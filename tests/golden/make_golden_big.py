"""Generate tests/golden/ref_big.npz: the REAL reference's outputs at the
configurations that carry the metric (VERDICT r1 "pin the metric-carrying
configs").

Runs oracle/_ref/libdla_ref.so (compiled from /root/reference/proj/include by
oracle/Makefile; TEST INFRASTRUCTURE) on seeded Philox inputs:

  c2        make_gp + Graph::backward (dl/models.hpp:94-135, dl/tape.hpp:461)
            at n=4096, d=8 on bench.py's own inputs (rng 1234): nll, the 3
            log-parameter gradients, xbar [4096,8], ybar [4096]   (~150 s)
  potrf1024 potrf + potrf_backward_into (dl/cholesky.hpp:35-88,
            dl/adjoints.hpp:175-191), batch 2 of 1024^2, Lbar = tril(N(0,1))
  potri128/256  potri + potri_backward_into (dl/cholesky.hpp:97-130,
            dl/adjoints.hpp:195-222), batch 2, Bbar = N(0,1)
  syevd96   syevd + syevd_backward_into (dl/eigen_sym.hpp, dl/adjoints.hpp:
            260-296), batch 2 of 96^2 (full outputs)
  gelqf128x512  gelqf + gelqf_backward_into (dl/lq.hpp, dl/adjoints.hpp:
            228-252), the C3 slice shape

Matrices >= 128 are stored as SUMMARIES (fixture size): the exact diagonal,
row sums, column sums, Frobenius norm and 4096 sampled entries per slice;
each row/column sum touches every element, so a wrong element anywhere moves
at least two of them.  Inputs are regenerated from the seed by the tests
(x, y, N(0,1) draws are exact; SPD = X X^T + nI goes through numpy matmul, so
a checksum of the input is stored and checked at 1e-12).

    python tests/golden/make_golden_big.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

NSAMP = 4096


def summarize(out, key, m, seed):
    """Per-slice summary of m [batch, r, c] under key."""
    m = np.asarray(m, np.float64)
    if m.ndim == 2:
        m = m[None]
    b, r, c = m.shape
    g = O.rng(seed)
    ii = g.integers(0, r, size=NSAMP)
    jj = g.integers(0, c, size=NSAMP)
    out[key + "/diag"] = np.stack([np.diagonal(s) for s in m]) if r == c else np.zeros((b, 0))
    out[key + "/rowsum"] = m.sum(axis=2)
    out[key + "/colsum"] = m.sum(axis=1)
    out[key + "/fro"] = np.sqrt((m * m).sum(axis=(1, 2)))
    out[key + "/ii"], out[key + "/jj"] = ii, jj
    out[key + "/vals"] = m[:, ii, jj]


def inputs_potrf1024():
    r = O.rng(11)
    a = O.random_spd(1024, r, batch=2)
    lbar = np.tril(r.standard_normal((2, 1024, 1024)))
    return a, lbar


def inputs_potri(n):
    r = O.rng(100 + n)
    a = O.random_spd(n, r, batch=2)
    bbar = r.standard_normal((2, n, n))
    return a, bbar


def inputs_syevd96():
    r = O.rng(96)
    a = O.random_sym(96, r, batch=2)
    ubar = r.standard_normal((2, 96, 96))
    lbar = r.standard_normal((2, 96))
    return a, ubar, lbar


def inputs_gelqf():
    r = O.rng(512)
    a = r.standard_normal((1, 128, 512))
    qbar = r.standard_normal((1, 128, 512))
    lbar = np.tril(r.standard_normal((1, 128, 128)))
    return a, qbar, lbar


def inputs_c2():
    """bench.py run_c2's inputs (rank 0)."""
    r = O.rng(1234)
    x = r.standard_normal((1, 4096, 8))
    y = r.standard_normal((1, 4096, 1))
    return x, y


def main():
    O.build(ref=True)
    ref = O.ref()
    out = {}
    t0 = time.time()

    a, lbar = inputs_potrf1024()
    out["potrf1024/a_sum"] = a.sum(axis=(1, 2))
    _, res = ref.potrf_fwdbwd_batch(a, lbar, threads=2)
    summarize(out, "potrf1024/l", res["l"], 1)
    summarize(out, "potrf1024/abar", res["abar"], 2)
    print(f"potrf1024 {time.time() - t0:.1f}s", flush=True)

    for n in (128, 256):
        a, bbar = inputs_potri(n)
        out[f"potri{n}/a_sum"] = a.sum(axis=(1, 2))
        ls, bs, lbs = [], [], []
        for s in range(2):
            l = ref.potrf(a[s])
            b = ref.potri(l)
            ls.append(l)
            bs.append(b)
            lbs.append(ref.potri_bwd(bbar[s], l, b))
        summarize(out, f"potri{n}/b", np.stack(bs), 3)
        summarize(out, f"potri{n}/lbar", np.stack(lbs), 4)

    a, ubar, lmb = inputs_syevd96()
    us, lams, abs_ = [], [], []
    for s in range(2):
        u, lam = ref.syevd(a[s])
        us.append(u)
        lams.append(lam)
        abs_.append(ref.syevd_bwd(ubar[s], lmb[s], u, lam))
    out["syevd96/u"], out["syevd96/lam"], out["syevd96/abar"] = np.stack(us), np.stack(lams), np.stack(abs_)

    a, qbar, lbar = inputs_gelqf()
    _, res = ref.gelqf_fwdbwd_batch(a, qbar, lbar, threads=1)
    summarize(out, "gelqf128x512/q", res["q"], 5)
    summarize(out, "gelqf128x512/l", res["l"], 6)
    summarize(out, "gelqf128x512/abar", res["abar"], 7)
    print(f"small cases done {time.time() - t0:.1f}s", flush=True)

    x, y = inputs_c2()
    t1 = time.time()
    o, xb, yb = ref.gp_nll_grad(x[0], y[0], 1.0, 1.0, 0.1, with_xy=True)
    out["c2/out"], out["c2/xbar"], out["c2/ybar"] = o, xb, yb
    out["c2/seconds_1core"] = np.array([time.time() - t1])
    print(f"c2 {time.time() - t0:.1f}s nll={o[0]!r}", flush=True)

    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_big.npz")
    np.savez_compressed(dst, **out)
    print("wrote", dst, len(out), "arrays", os.path.getsize(dst), "bytes")


if __name__ == "__main__":
    main()
