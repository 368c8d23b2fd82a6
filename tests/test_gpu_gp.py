"""GP NLL + gradient driver (C2 graph) on the GPU vs the REAL reference's
make_gp + Graph::backward (golden vectors from oracle/_ref, and the live
reference when it is built)."""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1710_08717_b200 import gp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "ref_vectors.npz"))
PARAMS = {"gp:96": (1.0, 1.0, 0.1), "gp:300": (1.3, 0.7, 0.05)}


def rel(a, b):
    return np.abs(a - b).max() / max(1.0, np.abs(b).max())


@pytest.mark.parametrize("key", sorted(PARAMS))
def test_gp_matches_reference_golden(key):
    x, y = GOLD[key + "/x"], GOLD[key + "/y"]
    s2, l2, lam = PARAMS[key]
    nll, grads, xbar, ybar = gp.gp_nll_grad(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), s2, l2, lam)
    out = GOLD[key + "/out"]
    assert abs(nll.item() - out[0]) / max(1, abs(out[0])) < 1e-10
    assert rel(grads.cpu().numpy(), out[1:]) < 1e-9
    assert rel(xbar.cpu().numpy(), GOLD[key + "/xbar"]) < 1e-9
    assert rel(ybar.cpu().numpy().reshape(-1), GOLD[key + "/ybar"].reshape(-1)) < 1e-9


def test_gp_closed_forms():
    # tests/test_models.cpp:61-74
    for yv, want in ((0.0, 1.2655121234846454), (1.0, 1.5155121234846453)):
        nll, *_ = gp.gp_nll_grad(torch.zeros(1, 1, dtype=torch.float64, device="cuda"),
                                 torch.full((1, 1), yv, dtype=torch.float64, device="cuda"), 1.0, 1.0, 1.0)
        assert abs(nll.item() - want) < 1e-12


def test_gp_batched_equals_per_slice():
    r = O.rng(5)
    x = r.standard_normal((3, 130, 8))
    y = r.standard_normal((3, 130, 1))
    xb, yb = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    nll, grads, xbar, _ = gp.gp_nll_grad(xb, yb, 1.1, 0.9, 0.2)
    for i in range(3):
        n1, g1, x1, _ = gp.gp_nll_grad(xb[i], yb[i], 1.1, 0.9, 0.2)
        assert torch.equal(n1, nll[i]) and torch.equal(g1, grads[i]) and torch.equal(x1, xbar[i])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_gp_matches_live_reference_n512():
    r = O.rng(9)
    x = r.standard_normal((512, 8))
    y = r.standard_normal((512, 1))
    out, xb, yb = O.ref().gp_nll_grad(x, y, 1.0, 1.0, 0.1, with_xy=True)
    nll, grads, xbar, ybar = gp.gp_nll_grad(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), 1.0, 1.0, 0.1)
    assert abs(nll.item() - out[0]) / abs(out[0]) < 1e-10
    assert rel(grads.cpu().numpy(), out[1:]) < 1e-8
    assert rel(xbar.cpu().numpy(), xb) < 1e-8


@pytest.mark.parametrize("n,batch", [(1024, 1), (1536, 2), (4096, 1)])
def test_gp_early_inverse_matches_split(monkeypatch, n, batch):
    # dla_gp_potrf_inv_f64 (L11^-1 and L21 L11^-1 formed while the blocked
    # factorization's second half runs) vs potrf + dla_potrf_bwd_begin_f64
    r = O.rng(n)
    x = torch.from_numpy(r.standard_normal((batch, n, 8))).cuda()
    y = torch.from_numpy(r.standard_normal((batch, n, 1))).cuda()
    outs = []
    for early in (False, True):
        monkeypatch.setattr(gp, "_EARLY", early)
        g = gp.GPNLL(n, 8, batch, "cuda")
        outs.append([t.clone() for t in g.step(x, y, 1.0, 1.0, 0.1)])
        g.check()
        assert torch.count_nonzero(torch.triu(g.a, 1)) == 0  # potrf contract: L's strict upper is zero
    # same kernels on the same blocks in a different order: bitwise equal
    for a, b in zip(*outs):
        assert torch.equal(a, b)
