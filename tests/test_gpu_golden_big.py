"""Parity at the configurations that carry the metric, against the REAL
reference's outputs (tests/golden/ref_big.npz, written by
tests/golden/make_golden_big.py from oracle/_ref — the reference compiled
from its own headers).

  * C2 headline: GP NLL + gradient at n=4096, d=8 on bench.py's inputs —
    nll, d/dlog(sigma2, ell2, lam), xbar, ybar (dl/models.hpp:94-135).
  * north star: potrf fwd+bwd at n=1024 (batch 2), Lbar = tril(N(0,1)).
  * potri / potri_backward at n=128 (the C5 size) and 256 — the DMMA
    level-batched inverse path.
  * syevd / syevd_backward at n=96 (> 64: the global-memory Jacobi).
  * gelqf / gelqf_backward at the C3 slice shape 128x512.

Tolerances (north star: "within a stated tolerance scaled by condition
number"): the SPD inputs have kappa <~ 5, so fp64 values agree to
~n*u*kappa; we require rel <= 1e-10 on factors and <= 1e-9 on gradients
(normalised by the array's max magnitude), and the full-size C2 quantities to
rel 1e-9.  Summaries (diag / row sums / column sums / samples / Frobenius
norm) are compared with the same bars.
"""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import make_golden_big as MG  # noqa: E402  (input generators only)

from paper_1710_08717_b200 import gp  # noqa: E402
from paper_1710_08717_b200 import linalg as L  # noqa: E402

G = np.load(os.path.join(HERE, "golden", "ref_big.npz"))


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(1e-300, np.abs(b).max()))


def check_summary(key, m, tol):
    m = np.asarray(m, np.float64)
    if m.ndim == 2:
        m = m[None]
    d = G[key + "/diag"]
    if d.size:
        assert rel(np.stack([np.diagonal(s) for s in m]), d) < tol, key + " diag"
    assert rel(m.sum(axis=2), G[key + "/rowsum"]) < tol * 10, key + " rowsum"
    assert rel(m.sum(axis=1), G[key + "/colsum"]) < tol * 10, key + " colsum"
    assert rel(np.sqrt((m * m).sum(axis=(1, 2))), G[key + "/fro"]) < tol, key + " fro"
    assert rel(m[:, G[key + "/ii"], G[key + "/jj"]], G[key + "/vals"]) < tol, key + " samples"


def test_c2_n4096_matches_reference():
    x, y = MG.inputs_c2()
    g = gp.GPNLL(4096, 8, 1, "cuda", want_xbar=True)
    nll, grads, xbar, ybar = g.step(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), 1.0, 1.0, 0.1)
    g.check()
    out = G["c2/out"]
    assert abs(nll.item() - out[0]) / abs(out[0]) < 1e-12
    gr = grads.cpu().numpy().reshape(-1)
    for i in range(3):  # each log-parameter gradient on its own
        assert abs(gr[i] - out[1 + i]) / max(1.0, abs(out[1 + i])) < 1e-9, (i, gr[i], out[1 + i])
    assert rel(xbar.cpu().numpy().reshape(4096, 8), G["c2/xbar"]) < 1e-9
    assert rel(ybar.cpu().numpy().reshape(-1), G["c2/ybar"].reshape(-1)) < 1e-9


def test_potrf_n1024_fwd_bwd_matches_reference():
    a, lbar = MG.inputs_potrf1024()
    assert rel(a.sum(axis=(1, 2)), G["potrf1024/a_sum"]) < 1e-12
    ad = torch.from_numpy(a).cuda()
    l = L.potrf(ad)
    abar = L.potrf_backward(torch.from_numpy(lbar).cuda(), l)
    ln, abn = l.cpu().numpy(), abar.cpu().numpy()
    assert np.count_nonzero(np.triu(ln, 1)) == 0
    check_summary("potrf1024/l", ln, 1e-10)
    check_summary("potrf1024/abar", abn, 1e-9)
    assert np.array_equal(abn, np.swapaxes(abn, 1, 2))  # bit-symmetric
    # backward error (north star): ||A - L L^T|| / ||A|| <= 1e-12
    for s in range(2):
        r = np.linalg.norm(a[s] - ln[s] @ ln[s].T) / np.linalg.norm(a[s])
        assert r < 1e-12


@pytest.mark.parametrize("n", [128, 256])
def test_potri_and_bwd_match_reference(n):
    a, bbar = MG.inputs_potri(n)
    assert rel(a.sum(axis=(1, 2)), G[f"potri{n}/a_sum"]) < 1e-12
    l = L.potrf(torch.from_numpy(a).cuda())
    b = L.potri(l)
    lb = L.potri_backward(torch.from_numpy(bbar).cuda(), l, b)
    bn, lbn = b.cpu().numpy(), lb.cpu().numpy()
    assert np.array_equal(bn, np.swapaxes(bn, 1, 2))
    assert np.count_nonzero(np.triu(lbn, 1)) == 0
    check_summary(f"potri{n}/b", bn, 1e-10)
    check_summary(f"potri{n}/lbar", lbn, 1e-9)


def test_syevd_n96_fwd_bwd_matches_reference():
    a, ubar, lmb = MG.inputs_syevd96()
    u, lam = L.syevd(torch.from_numpy(a).cuda())
    abar = L.syevd_backward(torch.from_numpy(ubar).cuda(), torch.from_numpy(lmb).cuda(), u, lam)
    assert rel(lam.cpu().numpy(), G["syevd96/lam"]) < 1e-12
    # rows = eigenvectors with the reference's sign rule: elementwise parity
    assert rel(u.cpu().numpy(), G["syevd96/u"]) < 1e-9
    ab = abar.cpu().numpy()
    assert np.array_equal(ab, np.swapaxes(ab, 1, 2))
    assert rel(ab, G["syevd96/abar"]) < 1e-8


def test_gelqf_c3_shape_matches_reference():
    a, qbar, lbar = MG.inputs_gelqf()
    q, l = L.gelqf(torch.from_numpy(a).cuda())
    abar = L.gelqf_backward(torch.from_numpy(qbar).cuda(), torch.from_numpy(lbar).cuda(), q, l)
    check_summary("gelqf128x512/q", q.cpu().numpy(), 1e-10)
    check_summary("gelqf128x512/l", l.cpu().numpy(), 1e-10)
    check_summary("gelqf128x512/abar", abar.cpu().numpy(), 1e-9)
