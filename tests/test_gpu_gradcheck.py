"""The reference's gradient-check registry (dl/gradcheck.hpp:206-478:
29 entries -- gemm2 x4, syrk x2, trmm x8, trsm x8, potrf x2, potri x2,
gelqf, syevd, gesvd) run against the DEVICE operators, at the reference's
sizes {2, 3, 5, 8, 16} x 10 trials in fp64 (acceptance criterion 1,
proj/tests/acceptance_main.cpp:59-78) and the fp32 smoke grid {3} x 2
(proj/tests/test_gradcheck.cpp:99-104), with its ToleranceConfig defaults
(dl/common.hpp:67-79) and its pass rule (compare_grads,
dl/gradcheck.hpp:150-164).

Each check forms phi(x) = sum_k <cotangent_k, output_k(x)> and compares the
device pullback with central differences (step fd_step; symmetric inputs
perturbed in (i,j)/(j,i) pairs and halved, as finite_diff_grad does).  The
B200 twist: every perturbed input of one check is a slice of ONE batched
device call (2 x #coordinates slices), so a check is a handful of launches.
Inputs come from numpy's Philox (the reference's std::normal_distribution
is libstdc++-specific), seeded per (entry, n, trial) from 20260816.
"""
import itertools

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1710_08717_b200 import linalg as L  # noqa: E402

GRID = {torch.float64: ((2, 3, 5, 8, 16), 10), torch.float32: ((3,), 2)}
BASE_SEED = 20260816
CFG = {torch.float64: dict(eps_gap=1e-8, fd_step=1e-6, rtol=1e-5, atol=1e-7, min_gap=1e-3),
       torch.float32: dict(eps_gap=1e-4, fd_step=1e-2, rtol=1e-2, atol=1e-4, min_gap=1e-2)}


def dev(x, dt):
    return torch.from_numpy(np.ascontiguousarray(x)).to(device="cuda", dtype=dt)


def fd_grad(phi, x0, h, symmetric):
    """Central differences of the batched functional phi([B, r, c]) -> [B]
    (dl/gradcheck.hpp:120-148), all perturbations in one batch."""
    r, c = x0.shape
    coords = [(i, j) for i in range(r) for j in range(c) if not (symmetric and j > i)]
    k = len(coords)
    xs = x0.unsqueeze(0).repeat(2 * k, 1, 1)
    for q, (i, j) in enumerate(coords):
        for sgn, base in ((1.0, 0), (-1.0, k)):
            xs[base + q, i, j] += sgn * h
            if symmetric and i != j:
                xs[base + q, j, i] += sgn * h
    f = phi(xs)
    g = torch.zeros(r, c, dtype=torch.float64, device="cuda")
    d = (f[:k].double() - f[k:].double()) / (2.0 * h)
    for q, (i, j) in enumerate(coords):
        v = d[q] / 2.0 if (symmetric and i != j) else d[q]
        g[i, j] = v
        if symmetric and i != j:
            g[j, i] = v
    return g


def compare(analytic, fd, cfg):
    """compare_grads (dl/gradcheck.hpp:150-164)."""
    err = (analytic.double() - fd).abs().max().item()
    denom = max(fd.abs().max().item(), cfg["atol"])
    return err <= cfg["atol"] or err / denom <= cfg["rtol"], err / denom


def dot(cot, out):
    """sum over each slice of <cotangent, output> (output [B, ...])."""
    return (cot.unsqueeze(0) * out).reshape(out.shape[0], -1).sum(dim=1)


def rep(x, b):
    return x.unsqueeze(0).expand(b, *x.shape).contiguous()


def spd(n, r):
    x = r.standard_normal((n, n))
    return x @ x.T + n * np.eye(n)


def entries():
    out = []
    for ta, tb in itertools.product([False, True], repeat=2):
        out.append((f"gemm2[{'tn'[not ta]}{'tn'[not tb]}]", "gemm2", dict(ta=ta, tb=tb)))
    for ta in (False, True):
        out.append((f"syrk[{'tn'[not ta]}]", "syrk", dict(ta=ta)))
    for op in ("trmm", "trsm"):
        for rs, tr, lo in itertools.product([False, True], repeat=3):
            out.append((f"{op}[{'rl'[not rs]}{'tn'[not tr]}{'lo' if lo else 'up'}]", op,
                        dict(right=rs, trans=tr, lower=lo)))
    for op in ("potrf", "potri"):
        for lo in (False, True):
            out.append((f"{op}[{'lo' if lo else 'up'}]", op, dict(lower=lo)))
    out += [("gelqf", "gelqf", {}), ("syevd", "syevd", {}), ("gesvd", "gesvd", {})]
    return out


ENTRIES = entries()


def run_check(kind, kw, n, r, dt, cfg):
    h = cfg["fd_step"]
    R = lambda *s: dev(r.standard_normal(s), dt)  # noqa: E731
    parts = []
    if kind == "gemm2":
        ta, tb, alpha = kw["ta"], kw["tb"], 1.25
        k, m = n + 1, n + 2
        a = R(k, n) if ta else R(n, k)
        b = R(m, k) if tb else R(k, m)
        cbar = R(n, m)
        abar, bbar = L.gemm2_backward(cbar, a, b, ta, tb, alpha)
        parts.append(compare(abar, fd_grad(lambda X: dot(cbar, L.gemm2(X, rep(b, X.shape[0]), ta, tb, alpha)), a, h,
                                           False), cfg))
        parts.append(compare(bbar, fd_grad(lambda X: dot(cbar, L.gemm2(rep(a, X.shape[0]), X, ta, tb, alpha)), b, h,
                                           False), cfg))
    elif kind == "syrk":
        ta, alpha, k = kw["ta"], 0.75, n + 1
        a = R(k, n) if ta else R(n, k)
        bbar = R(n, n)
        abar = L.syrk_backward(bbar, a, ta, alpha)
        parts.append(compare(abar, fd_grad(lambda X: dot(bbar, L.syrk(X, ta, alpha)), a, h, False), cfg))
    elif kind in ("trmm", "trsm"):
        rs, tr, lo = kw["right"], kw["trans"], kw["lower"]
        if kind == "trmm":
            alpha = 1.5
            t = R(n, n)
            t = torch.tril(t) if lo else torch.triu(t)
        else:
            alpha = 0.8
            t = L.potrf(dev(spd(n, r), dt), lo)
        a = R(n + 1, n) if rs else R(n, n + 1)
        fwd = L.trmm if kind == "trmm" else L.trsm
        bbar = R(*a.shape)
        if kind == "trmm":
            abar, tbar = L.trmm_backward(bbar, t, a, rs, tr, lo, alpha)
        else:
            b = L.trsm(t, a, rs, tr, lo, alpha)
            abar, tbar = L.trsm_backward(bbar, t, b, rs, tr, lo, alpha)
        parts.append(compare(tbar, fd_grad(lambda X: dot(bbar, fwd(X, rep(a, X.shape[0]), rs, tr, lo, alpha)), t, h,
                                           False), cfg))
        parts.append(compare(abar, fd_grad(lambda X: dot(bbar, fwd(rep(t, X.shape[0]), X, rs, tr, lo, alpha)), a, h,
                                           False), cfg))
    elif kind == "potrf":
        lo = kw["lower"]
        a = dev(spd(n, r), dt)
        l = L.potrf(a, lo)
        lbar = R(n, n)
        lbar = torch.tril(lbar) if lo else torch.triu(lbar)
        abar = L.potrf_backward(lbar, l, lo)
        parts.append(compare(abar, fd_grad(lambda X: dot(lbar, L.potrf(X, lo)), a, h, True), cfg))
    elif kind == "potri":
        lo = kw["lower"]
        l = L.potrf(dev(spd(n, r), dt), lo)
        b = L.potri(l, lo)
        bbar = R(n, n)
        lbar = L.potri_backward(bbar, l, b, lo)
        parts.append(compare(lbar, fd_grad(lambda X: dot(bbar, L.potri(X, lo)), l, h, False), cfg))
    elif kind == "gelqf":
        m, cols = n, n + 3
        a = R(m, cols)
        q, l = L.gelqf(a)
        qbar, lbar = R(m, cols), torch.tril(R(m, m))
        abar = L.gelqf_backward(qbar, lbar, q, l)

        def phi(X):
            qx, lx = L.gelqf(X)
            return dot(qbar, qx) + dot(lbar, lx)
        parts.append(compare(abar, fd_grad(phi, a, h, False), cfg))
    elif kind == "syevd":
        for _ in range(64):  # random_symmetric_gapped (dl/gradcheck.hpp:78-91)
            x = r.standard_normal((n, n))
            a = 0.5 * (x + x.T) * np.sqrt(n)
            ev = np.linalg.eigvalsh(a)
            if n == 1 or np.diff(ev).min() >= cfg["min_gap"]:
                break
        a = dev(a, dt)
        u, lam = L.syevd(a)
        ubar, lbar = R(n, n), R(n)
        abar = L.syevd_backward(ubar, lbar, u, lam, cfg["eps_gap"])

        def phi(X):
            ux, lx = L.syevd(X)
            return dot(ubar, ux) + dot(lbar, lx)
        parts.append(compare(abar, fd_grad(phi, a, h, True), cfg))
    elif kind == "gesvd":
        m, cols = n, n + 3
        for _ in range(64):  # random_wide_gapped (dl/gradcheck.hpp:93-105)
            a = r.standard_normal((m, cols))
            s = np.linalg.svd(a, compute_uv=False)[::-1]
            if s[0] >= cfg["min_gap"] and (m == 1 or np.diff(s).min() >= cfg["min_gap"]):
                break
        a = dev(a, dt)
        u, lam, v = L.gesvd(a)
        ubar, lbar, vbar = R(m, m), R(m), R(m, cols)
        abar = L.gesvd_backward(ubar, lbar, vbar, u, lam, v, cfg["eps_gap"])

        def phi(X):
            ux, lx, vx = L.gesvd(X)
            return dot(ubar, ux) + dot(lbar, lx) + dot(vbar, vx)
        parts.append(compare(abar, fd_grad(phi, a, h, False), cfg))
    ok = all(p[0] for p in parts)
    return ok, max(p[1] for p in parts)


@pytest.mark.parametrize("dt", [torch.float64, torch.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("entry", range(len(ENTRIES)), ids=[e[0] for e in ENTRIES])
def test_reference_gradcheck_registry_on_device(entry, dt):
    name, kind, kw = ENTRIES[entry]
    cfg = CFG[dt]
    fails, worst = [], 0.0
    sizes, trials = GRID[dt]
    for n in sizes:
        for trial in range(trials):
            r = np.random.Generator(np.random.Philox([BASE_SEED, entry, n, trial, int(dt == torch.float32)]))
            ok, w = run_check(kind, kw, n, r, dt, cfg)
            worst = max(worst, w)
            if not ok:
                fails.append((n, trial, w))
    assert not fails, f"{name}: {len(fails)} failing checks, worst rel {worst:.3g}: {fails[:5]}"
