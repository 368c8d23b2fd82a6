"""Device-resident tape (paper_1710_08717_b200/tape.py + csrc/tape_ew.cu):
the reference's Graph semantics, GradStore and memory plan on the GPU,
checked against the reference's own tape tests, its model graphs' outputs
(committed golden vectors of make_gp / make_kalman + Graph::backward) and its
memory-plan hand-off counts (tests/golden/make_golden_tape.py)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1710_08717_b200 import linalg as L  # noqa: E402
from paper_1710_08717_b200 import tape as TP  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GP = np.load(os.path.join(HERE, "golden", "ref_vectors.npz"))
KG = np.load(os.path.join(HERE, "golden", "kalman_ref.npz"))
PLAN = json.load(open(os.path.join(HERE, "golden", "tape_ref.json")))
GP_PARAMS = {"gp:96": (1.0, 1.0, 0.1), "gp:300": (1.3, 0.7, 0.05)}


def host(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return np.abs(a - b).max() / max(1.0, np.abs(b).max())


def test_memory_plan_reference_case():
    # proj/tests/test_tape.cpp:124-148
    x0 = O.rng(97).standard_normal((4, 4))
    g = TP.Graph()
    x = g.leaf(x0, "x")
    t1 = g.neg(x)
    t2 = g.neg(t1)
    t3 = g.neg(t2)
    loss = g.sum(t3)
    g.forward()
    plain = host(g.value(loss))[0, 0]
    assert g.planned_reuse_count() == 2  # t2 claims t1, t3 claims t2
    g.set_use_memory_plan(True)
    g.forward()
    assert host(g.value(loss))[0, 0] == plain
    with pytest.raises(L.Error, match="released"):
        g.value(t1)
    grads = g.backward(loss)
    assert np.all(host(grads.at(x)) == -1.0)


def test_graph_errors():
    g = TP.Graph()
    x = g.leaf(np.ones((2, 3)), "x")
    y = g.leaf(np.ones((3, 3)), "y")
    with pytest.raises(L.ShapeError):
        g.add(x, y)
    with pytest.raises(L.ShapeError):
        g.potrf(x)
    s = g.sum(x)
    with pytest.raises(L.Error):
        g.forward([(s, np.ones((1, 1)))])  # not a leaf
    with pytest.raises(L.ShapeError):
        g.forward([(x, np.ones((2, 2)))])
    with pytest.raises(L.ShapeError):
        g.backward(x)  # loss must be 1 x 1
    with pytest.raises(L.Error, match="no gradient"):
        g.backward(s).at(y)


@pytest.mark.parametrize("key", sorted(GP_PARAMS))
@pytest.mark.parametrize("plan", [False, True])
def test_make_gp_on_device_tape_matches_reference(key, plan):
    """The reference's make_gp graph (dl/models.hpp:115-135) built node by node
    on the device tape: NLL and every leaf gradient vs its Graph::backward."""
    x, y = GP[key + "/x"], GP[key + "/y"]
    g = TP.Graph()
    m = TP.make_gp(g, x, y, *GP_PARAMS[key])
    if plan:
        g.set_use_memory_plan(True)
        g.forward()
    out = GP[key + "/out"]
    assert abs(host(g.value(m["loss"]))[0, 0] - out[0]) / max(1, abs(out[0])) < 1e-10
    gs = g.backward(m["loss"])
    got = [host(gs.at(m[k]))[0, 0] for k in ("log_sigma2", "log_ell2", "log_lam")]
    assert rel(np.array(got), out[1:]) < 1e-9
    assert rel(host(gs.at(m["x"])), GP[key + "/xbar"]) < 1e-9
    assert rel(host(gs.at(m["y"])).reshape(-1), GP[key + "/ybar"].reshape(-1)) < 1e-9
    assert g.planned_reuse_count() == PLAN[key]


def test_plan_on_off_bitwise_and_saves_memory():
    r = O.rng(5)
    x, y = r.standard_normal((512, 4)), r.standard_normal((512, 1))
    res = []
    for plan in (False, True):
        g = TP.Graph()
        m = TP.make_gp(g, x, y, 1.1, 0.9, 0.2)
        g.set_use_memory_plan(plan)
        g.forward()
        peak = g.peak_bytes
        gs = g.backward(m["loss"])
        res.append((host(g.value(m["loss"])), [host(gs.at(m[k])) for k in ("x", "y", "log_sigma2", "log_ell2",
                                                                              "log_lam")], peak))
    (l0, g0, p0), (l1, g1, p1) = res
    assert np.array_equal(l0, l1)
    assert all(np.array_equal(a, b) for a, b in zip(g0, g1))
    assert p1 < p0, (p0, p1)


@pytest.mark.parametrize("name", ["h2d2T5", "h4d3T20", "h3d5T10"])
def test_kalman_graph_on_device_tape(name):
    """build_kalman_nll (dl/models.hpp:285-337) on the device tape vs the
    reference's make_kalman + Graph::backward, with and without the plan."""
    p = [KG[f"{name}/in/{k}"] for k in ("a", "b", "sh", "sv", "mu0", "s0", "obs")]
    for plan in (False, True):
        g = TP.Graph()
        leaves = [g.leaf(v, k) for v, k in zip(p[:6], ("A", "B", "S_h", "S_v", "mu0", "S0"))]
        obs = [g.leaf(p[6][t].reshape(-1, 1), f"v{t}") for t in range(p[6].shape[0])]
        nll, _, _ = TP.build_kalman_nll(g, *leaves, obs)
        assert g.planned_reuse_count() == PLAN["kalman:" + name]
        if plan:
            g.set_use_memory_plan(True)
            g.forward()
        want = float(KG[f"{name}/nll"])
        assert abs(host(g.value(nll))[0, 0] - want) / max(1, abs(want)) < 1e-11
        gs = g.backward(nll)
        for leaf, k in zip(leaves, ("a", "b", "sh", "sv", "mu0", "s0")):
            assert rel(host(gs.at(leaf)), KG[f"{name}/grad/{k}"]) < 1e-10, k
        ob = np.stack([host(gs.at(o)).reshape(-1) for o in obs])
        assert rel(ob, KG[f"{name}/grad/obs"]) < 1e-10


def test_every_node_pullback_by_finite_differences():
    """One graph touching every node kind; central differences on device."""
    r = O.rng(11)
    base = [O.random_spd(6, r), r.standard_normal((4, 6)), r.standard_normal((6, 1))]

    def build(a_val, b_val, c_val):
        g = TP.Graph()
        a, b, c = g.leaf(a_val, "a"), g.leaf(b_val, "b"), g.leaf(c_val, "c")
        l = g.potrf(a)
        w = g.potri(l)
        t = g.trmm(l, g.trsm(l, c, False, False, True), False, True, True, 0.7)
        q, ll = g.gelqf(b)
        u, lam = g.syevd(g.add(a, g.syrk(b, True, 0.1)))
        uu, sv, vv = g.gesvd(b)
        terms = [g.sum(g.square(t)),
                 g.sum(g.log(g.extract_diag(l))),
                 g.scale_const(g.sum(g.mul(w, w)), 0.01),
                 g.sum(g.abs(g.tril_mask(ll))),
                 g.sum(g.exp(g.scale_const(lam, 0.01))),
                 g.sum(g.sqrt(g.add_const(g.square(sv), 1.0))),
                 g.sum(g.mul(g.gemm2(uu, b), q)),
                 g.sum(g.sum_rows(g.mul(vv, b))),
                 g.sum(g.sum_rows(g.mul(u, g.sub(a, g.make_diag(c))))),
                 g.div_scalar(g.sum(g.tile_cols(c, 3)), g.add_const(g.sum(g.square(c)), 1.0)),
                 g.mul_scalar(g.sum(g.tile_rows(c, 2)), g.sum(g.make_diag(c))),
                 g.sum(g.neg(g.triu_mask(g.gemm2(g.concat_cols(uu, b), g.concat_cols(uu, b), True, False))))]
        s = terms[0]
        for tt in terms[1:]:
            s = g.add(s, tt)
        return g, (a, b, c), s

    g, leaves, s = build(*base)
    gs = g.backward(s)
    eps = 1e-6
    for li in range(3):
        an = host(gs.at(leaves[li]))
        for ix in list(np.ndindex(*base[li].shape))[:12]:
            vals = []
            for sg in (1.0, -1.0):
                xs = [v.copy() for v in base]
                xs[li][ix] += sg * eps
                if li == 0 and ix[0] != ix[1]:  # keep A symmetric: perturb the mirrored entry too
                    xs[0][ix[::-1]] += sg * eps
                gg, _, ss = build(*xs)
                vals.append(host(gg.value(ss))[0, 0])
            fd = (vals[0] - vals[1]) / (2 * eps)
            want = an[ix] + (an[ix[::-1]] if li == 0 and ix[0] != ix[1] else 0.0)
            assert abs(fd - want) < 2e-5 * max(1.0, abs(fd)), (li, ix, fd, want)
