"""GPU parity of the fused C1 likelihood chain (dla_chol_chain_fwdbwd_*)
against the oracle's composition of the reference operators:
L = potrf(A), z = trsm(L, y), phi = 1/2 z^T z + sumlogdiag(L), and the
pullback (trsm_bwd with zbar = z, + diag(1/L_ii), potrf_bwd) — the chain
SURVEY §8d defines for BASELINE config C1 (dl/models.hpp:99-103)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1710_08717_b200 import linalg as L  # noqa: E402

TOL = {np.float64: 1e-10, np.float32: 2e-3}


def oracle_chain(port, a, y):
    lo = port.potrf(a)
    zo = port.trsm(lo, y)
    so, to = port.trsm_bwd(zo, lo, zo)
    to = to + np.diag(1.0 / np.diag(lo))
    ao = port.potrf_bwd(to, lo)
    phi = 0.5 * float(zo[:, 0] @ zo[:, 0]) + port.sumlogdiag(lo)
    return phi, ao, so


def rel(got, want):
    return np.abs(got - want).max() / max(1.0, np.abs(want).max())


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("n", [1, 2, 5, 17, 31, 32, 33, 70])  # <= 32 fused warp kernel, > 32 composed
def test_chain_matches_oracle(port, dt, n):
    r = O.rng(100 + n)
    B = 5
    a = O.random_spd(n, r, batch=B)
    y = r.standard_normal((B, n, 1))
    phi, abar, ybar = L.chol_chain_fwdbwd(torch.from_numpy(a.astype(dt)).cuda(),
                                          torch.from_numpy(y.astype(dt)).cuda())
    phi, abar, ybar = phi.cpu().numpy(), abar.cpu().numpy(), ybar.cpu().numpy()
    tol = TOL[dt]
    for b in range(B):
        wphi, wa, wy = oracle_chain(port, a[b], y[b])
        assert abs(phi[b] - wphi) / max(1.0, abs(wphi)) < tol
        assert rel(abar[b], wa) < tol
        assert rel(ybar[b], wy) < tol
        assert np.array_equal(abar[b], abar[b].T), "Abar must be bit-symmetric"


def test_chain_matches_operator_chain_batch64():
    """C1 shape: batch 64 x 32^2; same answer as the per-operator C-ABI chain."""
    r = O.rng(7)
    B, n = 64, 32
    a = torch.from_numpy(O.random_spd(n, r, batch=B)).cuda()
    y = torch.from_numpy(r.standard_normal((B, n, 1))).cuda()
    phi, abar, ybar = L.chol_chain_fwdbwd(a, y)
    l = L.potrf(a)
    z = L.trsm(l, y)
    ld = L.sumlogdiag(l)
    q = (z[:, :, 0] * z[:, :, 0]).sum(-1) * 0.5
    yb, lb = L.trsm_backward(z, l, z, False, False, True)
    L.sumlogdiag_backward_into(lb, torch.ones(B, dtype=torch.float64, device="cuda"), l, accumulate=True)
    ab = L.potrf_backward(lb, l)
    assert torch.allclose(phi, q + ld, rtol=1e-12, atol=1e-12)
    assert (abar - ab).abs().max().item() < 1e-12 * max(1.0, ab.abs().max().item())
    assert (ybar - yb).abs().max().item() < 1e-12


def test_chain_failures_leave_slice_untouched():
    r = O.rng(9)
    B, n = 3, 16
    a = O.random_spd(n, r, batch=B)
    a[1, 5, 5] = -100.0  # not SPD at step 5
    y = r.standard_normal((B, n, 1))
    ad, yd = torch.from_numpy(a).cuda(), torch.from_numpy(y).cuda()
    abar = torch.full_like(ad, 7.0)
    with pytest.raises(L.NotPositiveDefiniteError) as e:
        L.chol_chain_fwdbwd(ad, yd, abar=abar)
    assert e.value.batch_index == 1 and e.value.step == 5
    assert torch.all(abar[1] == 7.0)
    assert not torch.any(abar[0] == 7.0)
    a2 = O.random_spd(n, r, batch=1)
    a2[0, 0, 3] += 1.0  # asymmetric beyond rtol
    with pytest.raises(L.ShapeError):
        L.chol_chain_fwdbwd(torch.from_numpy(a2).cuda(), torch.from_numpy(y[:1]).cuda())
