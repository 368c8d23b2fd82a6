"""Pin the CPU oracle (C restatement, oracle/oracle_impl.h) before trusting it.

1. Against the reference's own known-answer tests (tests/golden/kat.json,
   restated from proj/tests/test_*.cpp with file:line citations).
2. Against the REAL reference compiled from /root/reference headers
   (oracle/_ref/libdla_ref.so) on seeded inputs over every op and flag
   combination: the restatement keeps the reference's loop orders, so the
   results must be bit-identical.
3. Against committed golden vectors produced by the real reference
   (tests/golden/ref_vectors.npz, made by tests/golden/make_golden.py), so the
   pin also holds where /root/reference is absent.
"""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
KAT = json.load(open(os.path.join(HERE, "golden", "kat.json")))
DTYPES = [np.float64, np.float32]


def A(x, dt=np.float64):
    return np.array(x, dtype=dt)


# ----------------------------------------------------------------- KATs
@pytest.mark.parametrize("dt", DTYPES)
def test_kat_potrf(port, dt):
    k = KAT["potrf_lower"]
    assert np.array_equal(port.potrf(A(k["a"], dt)), A(k["l"], dt))
    k = KAT["potrf_upper"]
    assert np.array_equal(port.potrf(A(k["a"], dt), lower=False), A(k["r"], dt))


def test_kat_potrf_errors(port):
    k = KAT["potrf_not_spd"]
    with pytest.raises(O.OracleError) as e:
        port.potrf(A(k["a"]))
    assert e.value.status == O.DLA_ERR_NOT_SPD and e.value.index == k["step"]
    with pytest.raises(O.OracleError) as e:
        port.potrf(A(KAT["potrf_asymmetric"]["a"]))
    assert e.value.status == O.DLA_ERR_ASYMMETRIC


@pytest.mark.parametrize("dt", DTYPES)
def test_kat_potri(port, dt):
    k = KAT["potri"]
    b = port.potri(A(k["l"], dt))
    np.testing.assert_allclose(b, A(k["b"], dt), rtol=1e-6)
    assert np.array_equal(b, b.T)


def test_kat_trsm(port):
    k = KAT["trsm"]
    np.testing.assert_allclose(port.trsm(A(k["t"]), A(k["x"])), A(k["y"]), rtol=1e-14)
    k = KAT["trsm_singular"]
    with pytest.raises(O.OracleError) as e:
        port.trsm(A(k["t"]), A(k["x"]))
    assert e.value.status == O.DLA_ERR_SINGULAR and e.value.index == k["index"]


@pytest.mark.parametrize("dt", DTYPES)
def test_kat_gelqf(port, dt):
    k = KAT["gelqf"]
    q, l = port.gelqf(A(k["a"], dt))
    np.testing.assert_allclose(l, A(k["l"], dt), rtol=1e-6)
    np.testing.assert_allclose(q, A(k["q"], dt), rtol=1e-6)
    with pytest.raises(O.OracleError) as e:
        port.gelqf(A(KAT["gelqf_rank_deficient"]["a"]))
    assert e.value.status == O.DLA_ERR_SINGULAR
    with pytest.raises(O.OracleError) as e:
        port.gelqf(np.zeros(KAT["gelqf_tall"]["shape"]))
    assert e.value.status == O.DLA_ERR_SHAPE


@pytest.mark.parametrize("dt", DTYPES)
def test_kat_syevd(port, dt):
    k = KAT["syevd_sign_rule"]
    u, lam = port.syevd(A(k["a"], dt))
    np.testing.assert_allclose(lam, A(k["lambda"], dt), atol=1e-6)
    np.testing.assert_allclose(u, A(k["u"], dt), atol=1e-6)
    k = KAT["syevd_diag_sort"]
    u, lam = port.syevd(A(k["a"], dt))
    np.testing.assert_allclose(lam, A(k["lambda"], dt), atol=1e-6)
    for i, j in k["u_ones"]:
        assert abs(u[i, j] - 1) < 1e-6
    with pytest.raises(O.OracleError) as e:
        port.syevd(A(KAT["syevd_asymmetric"]["a"]))
    assert e.value.status == O.DLA_ERR_ASYMMETRIC


def test_kat_syevd_bwd_small_gap(port):
    k = KAT["syevd_bwd_small_gap"]
    abar = port.syevd_bwd(A(k["ubar"]), A(k["lambdabar"]), A(k["u"]), A(k["lambda"]))
    assert np.all(np.isfinite(abar))
    assert np.array_equal(abar, abar.T)


def test_kat_recon_tolerances(port):
    r = O.rng(23)
    for n in KAT["potrf_recon_tol"]["sizes"]:
        a = O.random_spd(n, r)
        l = port.potrf(a)
        assert np.all(np.triu(l, 1) == 0) and np.all(np.diag(l) > 0)
        assert np.abs(l @ l.T - a).max() / max(np.abs(a).max(), 1) < 1e-12
        rr = port.potrf(a, lower=False)
        assert np.abs(rr.T @ rr - a).max() / max(np.abs(a).max(), 1) < 1e-12
    for n in KAT["potri_inverse_tol"]["sizes"]:
        a = O.random_spd(n, r)
        lo = port.potri(port.potrf(a))
        up = port.potri(port.potrf(a, lower=False), lower=False)
        assert np.abs(a @ lo - np.eye(n)).max() < 1e-11
        assert np.abs(lo - up).max() / max(np.abs(up).max(), 1) < 1e-12
    for m, n in KAT["gelqf_recon_tol"]["shapes"]:
        a = r.standard_normal((m, n))
        q, l = port.gelqf(a)
        assert np.abs(q @ q.T - np.eye(m)).max() < 1e-13
        assert np.abs(l @ q - a).max() / max(np.abs(a).max(), 1) < 1e-13
        assert np.all(np.diag(l) > 0)
    for n in KAT["syevd_recon_tol"]["sizes"]:
        a = O.random_sym(n, r)
        u, lam = port.syevd(a)
        assert np.all(np.diff(lam) >= 0)
        assert np.abs(u @ u.T - np.eye(n)).max() < 1e-13
        assert np.abs(u.T @ np.diag(lam) @ u - a).max() / max(np.abs(a).max(), 1) < 1e-12


def test_kat_potrf_bwd_fd(port):
    """tests/test_adjoints.cpp:174-190: potrf backward vs symmetric FD."""
    r = O.rng(71)
    n = 4
    a = O.random_spd(n, r)
    lbar = np.tril(r.standard_normal((n, n)))
    abar = port.potrf_bwd(lbar, port.potrf(a))
    h = 1e-6
    fd = np.zeros_like(a)
    for i in range(n):
        for j in range(i + 1):
            ap, am = a.copy(), a.copy()
            ap[i, j] += h; am[i, j] -= h
            if i != j:
                ap[j, i] += h; am[j, i] -= h
            g = (np.sum(lbar * port.potrf(ap)) - np.sum(lbar * port.potrf(am))) / (2 * h)
            if i != j:
                g /= 2
            fd[i, j] = fd[j, i] = g
    assert np.abs(abar - fd).max() / max(np.abs(fd).max(), 1) < 1e-6


# ----------------------------------------------------- restatement == ref
FLAGS = list(itertools.product([0, 1], repeat=3))


def _tri(n, r, lower, dt):
    t = O.random_spd(n, r)
    l = np.linalg.cholesky(t)
    t = l if lower else l.T.copy()
    return (t + np.triu(r.standard_normal((n, n)), 1) * 0 if lower else t).astype(dt)


@pytest.mark.parametrize("dt", DTYPES)
def test_port_matches_reference_blas(port, ref, dt):
    r = O.rng(7)
    for m, n, k in [(3, 5, 4), (1, 1, 1), (17, 9, 33), (64, 70, 65)]:
        for ta, tb in itertools.product([0, 1], repeat=2):
            a = r.standard_normal((k, m) if ta else (m, k)).astype(dt)
            b = r.standard_normal((n, k) if tb else (k, n)).astype(dt)
            c0 = r.standard_normal((m, n)).astype(dt)
            for acc in (0, 1):
                assert np.array_equal(port.gemm(a, b, ta, tb, 1.25, c0, acc),
                                      ref.gemm(a, b, ta, tb, 1.25, c0, acc))
            cb = r.standard_normal((m, n)).astype(dt)
            pa, pb = port.gemm2_bwd(cb, a, b, ta, tb, 0.75)
            ra, rb = ref.gemm2_bwd(cb, a, b, ta, tb, 0.75)
            assert np.array_equal(pa, ra) and np.array_equal(pb, rb)
        for ta in (0, 1):
            a = r.standard_normal((k, n) if ta else (n, k)).astype(dt)
            assert np.array_equal(port.syrk(a, ta, 0.75), ref.syrk(a, ta, 0.75))
            bb = r.standard_normal((n, n)).astype(dt)
            assert np.array_equal(port.syrk_bwd(bb, a, ta, 0.5), ref.syrk_bwd(bb, a, ta, 0.5))


@pytest.mark.parametrize("dt", DTYPES)
def test_port_matches_reference_triangular(port, ref, dt):
    r = O.rng(13)
    for m, n in [(4, 3), (1, 5), (33, 17), (70, 65)]:
        for right, tr, lo in FLAGS:
            nt = n if right else m
            t = r.standard_normal((nt, nt)).astype(dt)
            t[np.diag_indices(nt)] = np.abs(t[np.diag_indices(nt)]) + 2
            x = r.standard_normal((m, n)).astype(dt)
            assert np.array_equal(port.trmm(t, x, right, tr, lo, 1.5), ref.trmm(t, x, right, tr, lo, 1.5))
            assert np.array_equal(port.trsm(t, x, right, tr, lo, 0.8), ref.trsm(t, x, right, tr, lo, 0.8))
            bb = r.standard_normal((m, n)).astype(dt)
            for p, q in zip(port.trmm_bwd(bb, t, x, right, tr, lo, 1.5), ref.trmm_bwd(bb, t, x, right, tr, lo, 1.5)):
                assert np.array_equal(p, q)
            b = ref.trsm(t, x, right, tr, lo, 0.8)
            for p, q in zip(port.trsm_bwd(bb, t, b, right, tr, lo, 0.8), ref.trsm_bwd(bb, t, b, right, tr, lo, 0.8)):
                assert np.array_equal(p, q)


@pytest.mark.parametrize("dt", DTYPES)
def test_port_matches_reference_cholesky(port, ref, dt):
    r = O.rng(29)
    for n in [1, 2, 5, 17, 63, 64, 70, 129]:
        a = O.random_spd(n, r, dt)
        for lower in (1, 0):
            l = port.potrf(a, lower)
            assert np.array_equal(l, ref.potrf(a, lower))
            assert np.array_equal(port.potri(l, lower), ref.potri(l, lower))
            lbar = r.standard_normal((n, n)).astype(dt)
            assert np.array_equal(port.potrf_bwd(lbar, l, lower), ref.potrf_bwd(lbar, l, lower))
            b = ref.potri(l, lower)
            bbar = r.standard_normal((n, n)).astype(dt)
            assert np.array_equal(port.potri_bwd(bbar, l, b, lower), ref.potri_bwd(bbar, l, b, lower))


@pytest.mark.parametrize("dt", DTYPES)
def test_port_matches_reference_lq_eig(port, ref, dt):
    r = O.rng(37)
    for m, n in [(1, 1), (2, 5), (4, 4), (7, 11), (16, 16), (32, 128)]:
        a = r.standard_normal((m, n)).astype(dt)
        q, l = port.gelqf(a)
        rq, rl = ref.gelqf(a)
        assert np.array_equal(q, rq) and np.array_equal(l, rl)
        qb = r.standard_normal((m, n)).astype(dt)
        lb = np.tril(r.standard_normal((m, m))).astype(dt)
        assert np.array_equal(port.gelqf_bwd(qb, lb, q, l), ref.gelqf_bwd(qb, lb, q, l))
    for n in [1, 2, 3, 8, 16, 25, 64]:
        a = O.random_sym(n, r, dt)
        u, lam = port.syevd(a)
        ru, rlam = ref.syevd(a)
        assert np.array_equal(u, ru) and np.array_equal(lam, rlam)
        ub = r.standard_normal((n, n)).astype(dt)
        lb = r.standard_normal(n).astype(dt)
        assert np.array_equal(port.syevd_bwd(ub, lb, u, lam), ref.syevd_bwd(ub, lb, u, lam))


@pytest.mark.parametrize("dt", DTYPES)
def test_port_matches_reference_gesvd(port, ref, dt):
    # dl/svd.hpp:26-284 + dl/adjoints.hpp:315-382, bit for bit
    r = O.rng(43)
    for m, n in [(1, 1), (2, 6), (5, 5), (8, 13), (16, 19), (24, 80)]:
        a = r.standard_normal((m, n)).astype(dt)
        u, lam, v = port.gesvd(a)
        ru, rlam, rv = ref.gesvd(a)
        assert np.array_equal(u, ru) and np.array_equal(lam, rlam) and np.array_equal(v, rv)
        ub = r.standard_normal((m, m)).astype(dt)
        lb = r.standard_normal(m).astype(dt)
        vb = r.standard_normal((m, n)).astype(dt)
        assert np.array_equal(port.gesvd_bwd(ub, lb, vb, u, lam, v), ref.gesvd_bwd(ub, lb, vb, ru, rlam, rv))


@pytest.mark.parametrize("dt", DTYPES)
def test_kat_gesvd(port, dt):
    # proj/tests/test_svd.cpp:13-20 (hand value), :55-64 (tall rejected, zero matrix)
    u, lam, v = port.gesvd(np.array([[3.0, 4.0]], dt))
    assert abs(lam[0] - 5) < 1e-6 and abs(u[0, 0] - 1) < 1e-6
    assert abs(v[0, 0] - 0.6) < 1e-6 and abs(v[0, 1] - 0.8) < 1e-6
    with pytest.raises(O.OracleError):
        port.gesvd(np.zeros((4, 2), dt))
    u, lam, v = port.gesvd(np.zeros((3, 5), dt))
    assert np.all(lam == 0) and np.abs(u @ u.T - np.eye(3)).max() < 1e-6
    # reconstruction / orthonormal rows (test_svd.cpp:22-42)
    r = O.rng(47)
    for m, n in [(1, 1), (2, 6), (5, 5), (8, 13), (16, 16)]:
        a = r.standard_normal((m, n))
        u, lam, v = port.gesvd(a)
        assert np.all(np.diff(lam) >= 0) and np.all(lam >= 0)
        assert np.abs(u @ u.T - np.eye(m)).max() < 1e-13 and np.abs(v @ v.T - np.eye(m)).max() < 1e-13
        assert np.abs(u.T @ np.diag(lam) @ v - a).max() / np.abs(a).max() < 1e-12


def test_port_matches_reference_sumlogdiag(port, ref):
    r = O.rng(41)
    for n in [1, 2, 32, 100]:
        l = port.potrf(O.random_spd(n, r))
        v, g = ref.sumlogdiag(l, with_grad=True)
        assert port.sumlogdiag(l) == v
        assert np.array_equal(port.sumlogdiag_bwd(1.0, l), g)


def test_port_errors_match_reference(port, ref):
    bad = A(KAT["potrf_not_spd"]["a"])
    for lib in (port, ref):
        with pytest.raises(O.OracleError) as e:
            lib.potrf(bad)
        assert (e.value.status, e.value.index) == (O.DLA_ERR_NOT_SPD, 2)
    sing = A(KAT["trsm_singular"]["t"])
    for lib in (port, ref):
        with pytest.raises(O.OracleError) as e:
            lib.trsm(sing, A([[1.0], [1.0]]))
        assert (e.value.status, e.value.index) == (O.DLA_ERR_SINGULAR, 1)


def test_ref_gp_closed_forms(ref):
    for key in ("gp_closed_form_y0", "gp_closed_form_y1"):
        k = KAT[key]
        out = ref.gp_nll_grad(A(k["x"]), A(k["y"]), k["sigma2"], k["ell2"], k["lam"])
        assert abs(out[0] - k["nll"]) < 1e-12


# ------------------------------------------------------ golden vectors
GOLD = os.path.join(HERE, "golden", "ref_vectors.npz")


@pytest.mark.skipif(not os.path.exists(GOLD), reason="golden vectors not generated")
def test_port_matches_committed_golden(port):
    g = np.load(GOLD)
    names = sorted({k.split("/")[0] for k in g.files})
    assert names, "empty golden file"
    for name in names:
        op = name.split(":")[0]
        if op == "potrf":
            lower = int(name.split(":")[2])
            assert np.array_equal(port.potrf(g[name + "/a"], lower), g[name + "/l"])
            assert np.array_equal(port.potrf_bwd(g[name + "/lbar"], g[name + "/l"], lower), g[name + "/abar"])
        elif op == "trsm":
            f = [int(c) for c in name.split(":")[2]]
            assert np.array_equal(port.trsm(g[name + "/t"], g[name + "/x"], *f, 0.8), g[name + "/y"])
        elif op == "gelqf":
            q, l = port.gelqf(g[name + "/a"])
            assert np.array_equal(q, g[name + "/q"]) and np.array_equal(l, g[name + "/l"])
        elif op == "syevd":
            u, lam = port.syevd(g[name + "/a"])
            assert np.array_equal(u, g[name + "/u"]) and np.array_equal(lam, g[name + "/lam"])
        elif op == "gp":
            pass  # checked in test_gp_golden (needs the GP driver)


# --------------------------------------------------------------- Kalman NLL
KGOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "kalman_ref.npz")
KNAMES = ("a", "b", "sh", "sv", "mu0", "s0", "obs")


def _kcase(g, name):
    return tuple(g[f"{name}/in/{k}"] for k in KNAMES)


def test_kat_kalman_random_walk():
    # proj/tests/test_models.cpp:187-197: hand value of the scalar random walk
    one, zero = np.ones((1, 1)), np.zeros((1, 1))
    nll, _ = O.kalman_port(one, one, one, one, zero, one, np.zeros((2, 1)))
    assert abs(nll - 2.6425960226263948) < 1e-12 * 2.65


def test_kalman_port_matches_committed_golden():
    """The restatement (oracle_impl.h o_kalman) against the reference's own
    make_kalman + Graph::backward outputs and its dense joint-Gaussian oracle."""
    g = np.load(KGOLD)
    for name in g["cases"]:
        nll, grads = O.kalman_port(*_kcase(g, name))
        ref_nll = float(g[f"{name}/nll"])
        assert abs(nll - ref_nll) <= 1e-14 * abs(ref_nll), name
        # the recursive filter equals the dense joint Gaussian (test_models.cpp:199-217)
        assert abs(ref_nll - float(g[f"{name}/joint"])) < 1e-8 * max(1.0, abs(ref_nll)), name
        for k, v in zip(KNAMES, grads):
            w = g[f"{name}/grad/{k}"]
            assert np.abs(v - w).max() <= 1e-13 * max(1.0, np.abs(w).max()), (name, k)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_kalman_port_matches_live_reference():
    r = O.rng(2024)
    for h, d, T in [(2, 2, 6), (5, 3, 17), (7, 9, 11)]:
        m = O.random_kalman(r, h, d, T)
        nll, grads = O.kalman_port(*m)
        rn, rg, _ = O.kalman_ref(*m)
        assert abs(nll - rn) <= 1e-14 * abs(rn)
        for v, w in zip(grads, rg):
            assert np.abs(v - w).max() <= 1e-13 * max(1.0, np.abs(w).max())


def test_kalman_port_fd():
    """Central finite differences of the restated NLL on every leaf
    (proj/tests/test_models.cpp:219-241 perturbs A, B, Sh, Sv, mu0, S0, v1)."""
    r = O.rng(137)
    m = list(O.random_kalman(r, 2, 2, 4))
    _, grads = O.kalman_port(*m)
    eps = 1e-6
    for li in range(7):
        x = m[li]
        it = np.nditer(x, flags=["multi_index"])
        for _ in it:
            ix = it.multi_index
            sym = KNAMES[li] in ("sh", "sv", "s0")  # PerturbMode::Symmetric in the reference test
            if sym and ix[0] > ix[1]:
                continue
            xp, xm = x.copy(), x.copy()
            tw = (ix[1], ix[0])
            for y, sgn in ((xp, 1.0), (xm, -1.0)):
                y[ix] += sgn * eps
                if sym and tw != ix:
                    y[tw] += sgn * eps
            mp, mm_ = list(m), list(m)
            mp[li], mm_[li] = xp, xm
            fd = (O.kalman_port(*mp)[0] - O.kalman_port(*mm_)[0]) / (2 * eps)
            an = grads[li][ix] + (grads[li][tw] if sym and tw != ix else 0.0)
            assert abs(fd - an) < 1e-6 * max(1.0, abs(fd)), (KNAMES[li], ix)
