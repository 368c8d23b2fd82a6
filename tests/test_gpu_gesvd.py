"""gesvd forward + pullback on the device vs the oracle (a C restatement
pinned bit-exact to the reference's dl/svd.hpp / dl/adjoints.hpp:315-382,
tests/test_oracle.py) and the reference's own test_svd.cpp assertions.

Tolerances (fp64 / fp32): the device factorization is LQ + one-sided
Jacobi, the reference Golub-Kahan-Reinsch, so values agree to rounding:
singular values rel 1e-12 / 2e-5; singular vectors (well separated spectra,
so the sign rule makes them unique) and the pullback rel 1e-9 / 2e-3 of the
array's max magnitude.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1710_08717_b200 import linalg as L  # noqa: E402

TOL = {np.float64: (1e-12, 1e-9), np.float32: (2e-5, 2e-3)}


def rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(1e-30, np.abs(b).max()))


def assert_sign_rule(u):
    # dl/eigen_sym.hpp:316-333: each row's largest-|.| entry (first on ties) is >= 0
    for row in u:
        assert row[int(np.argmax(np.abs(row)))] >= 0


def align(ud, vd, uo, tol):
    """Rows whose sign differs from the reference's are allowed only where the
    sign rule is ill-posed at this precision: the reference row's two largest
    magnitudes tie to within tol.  Returns the device factors with those rows
    flipped (U and V in lockstep, as the rule flips them)."""
    ud, vd = ud.copy(), vd.copy()
    for i in range(ud.shape[0]):
        if np.dot(ud[i].astype(np.float64), uo[i]) < 0:
            top = np.sort(np.abs(uo[i]))[::-1]
            assert len(top) > 1 and top[0] - top[1] <= 10 * tol * top[0], (i, top[:2])
            ud[i], vd[i] = -ud[i], -vd[i]
    return ud, vd


def gapped(m, n, r, dt, min_gap=1e-2):
    # the reference gradcheck's random_wide_gapped (dl/gradcheck.hpp:93-105)
    for _ in range(64):
        a = r.standard_normal((m, n))
        s = np.linalg.svd(a, compute_uv=False)[::-1]
        if s[0] >= min_gap and (m == 1 or np.diff(s).min() >= min_gap):
            return a.astype(dt)
    raise RuntimeError("resampling exhausted")


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("m,n", [(1, 1), (2, 6), (5, 5), (8, 13), (16, 19), (24, 80), (64, 200), (100, 260)])
def test_gesvd_fwd_bwd_matches_oracle(port, dt, m, n):
    r = O.rng(1000 * m + n)
    batch = 3
    a = np.stack([gapped(m, n, r, dt) for _ in range(batch)])
    ub = r.standard_normal((batch, m, m)).astype(dt)
    lb = r.standard_normal((batch, m)).astype(dt)
    vb = r.standard_normal((batch, m, n)).astype(dt)
    u, lam, v = L.gesvd(torch.from_numpy(a).cuda())
    ab = L.gesvd_backward(torch.from_numpy(ub).cuda(), torch.from_numpy(lb).cuda(), torch.from_numpy(vb).cuda(),
                          u, lam, v)
    tl, tv = TOL[dt]
    for s in range(batch):
        uo, lo, vo = port.gesvd(a[s])
        ud, ld, vd = u[s].cpu().numpy(), lam[s].cpu().numpy(), v[s].cpu().numpy()
        assert rel(ld, lo) < tl
        assert_sign_rule(ud)
        ua, va = align(ud, vd, uo, tv)
        assert rel(ua, uo) < tv and rel(va, vo) < tv
        # the pullback on identical (U, lambda, V): the device's
        ao = port.gesvd_bwd(ub[s], lb[s], vb[s], ud, ld, vd)
        assert rel(ab[s].cpu().numpy(), ao) < tv * 10
    un, vn = u.cpu().numpy().astype(np.float64), v.cpu().numpy().astype(np.float64)
    eye = np.eye(m)
    orth = 1e-12 if dt == np.float64 else max(2e-5, 3e-7 * m)  # rotation count grows with m
    assert np.abs(un @ np.swapaxes(un, 1, 2) - eye).max() < orth
    assert np.abs(vn @ np.swapaxes(vn, 1, 2) - eye).max() < orth


def test_gesvd_reference_kats():
    # proj/tests/test_svd.cpp:13-20 hand value, :55-64 tall rejected and zero matrix
    for dt in (torch.float32, torch.float64):
        u, lam, v = L.gesvd(torch.tensor([[3.0, 4.0]], dtype=dt, device="cuda"))
        assert abs(lam[0].item() - 5) < 1e-5 and abs(u[0, 0].item() - 1) < 1e-6
        assert abs(v[0, 0].item() - 0.6) < 1e-6 and abs(v[0, 1].item() - 0.8) < 1e-6
    with pytest.raises(L.ShapeError):
        L.gesvd(torch.zeros(4, 2, dtype=torch.float64, device="cuda"))
    u, lam, v = L.gesvd(torch.zeros(3, 5, dtype=torch.float64, device="cuda"))
    assert torch.all(lam == 0)
    assert (u @ u.T - torch.eye(3, dtype=torch.float64, device="cuda")).abs().max().item() < 1e-14
    # the pullback refuses a zero singular value: SingularError(0)
    with pytest.raises(L.SingularError) as e:
        L.gesvd_backward(torch.ones(3, 3, dtype=torch.float64, device="cuda"),
                         torch.ones(3, dtype=torch.float64, device="cuda"),
                         torch.ones(3, 5, dtype=torch.float64, device="cuda"), u, lam, v)
    assert e.value.index == 0
    # singular values match syevd of the gram matrix (test_svd.cpp:44-53)
    r = O.rng(53)
    a = torch.from_numpy(r.standard_normal((5, 8))).cuda()
    _, lam, _ = L.gesvd(a)
    _, ev = L.syevd(L.syrk(a))
    assert torch.allclose(lam * lam, ev, rtol=1e-10, atol=0)


def test_gesvd_rank_deficient_and_batch_invariance():
    r = O.rng(9)
    x = r.standard_normal((4, 2))
    a = np.repeat((x @ r.standard_normal((2, 9)))[None], 2, axis=0)  # 4 x 9 of rank 2
    u, lam, v = L.gesvd(torch.from_numpy(a).cuda())
    lam = lam.cpu().numpy()
    assert np.abs(lam[:, :2]).max() < 1e-13 and lam[0, 2] > 1e-3
    recon = np.swapaxes(u.cpu().numpy(), 1, 2) @ (lam[:, :, None] * v.cpu().numpy())
    assert np.abs(recon - a).max() < 1e-12
    b = torch.from_numpy(np.stack([gapped(6, 11, r, np.float64) for _ in range(5)])).cuda()
    ub, lb, vb = L.gesvd(b)
    for i in range(5):
        u1, l1, v1 = L.gesvd(b[i])
        assert torch.equal(u1, ub[i]) and torch.equal(l1, lb[i]) and torch.equal(v1, vb[i])
