"""Batched Kalman filter NLL + gradient (csrc/kalman.cu, dla_kalman_nll_fwdbwd)
against the REAL reference's make_kalman + Graph::backward (committed golden
vectors, tests/golden/make_golden_kalman.py) and the pinned oracle
restatement (oracle_impl.h o_kalman) on seeded batches."""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1710_08717_b200 import kalman as K  # noqa: E402
from paper_1710_08717_b200 import linalg as L  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "kalman_ref.npz"))
NAMES = ("a", "b", "sh", "sv", "mu0", "s0", "obs")
TOL = 1e-11  # f64: relative to max(1, |reference|); per-op rounding differs from the tape's loop orders


def dev(x, dt=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)


def rel(a, b):
    return np.abs(a - b).max() / max(1.0, np.abs(b).max())


def run(model, batch_params, obs, dt=torch.float64):
    h, d = model[0].shape[-1], model[1].shape[-2]
    B, T = obs.shape[0], obs.shape[1]
    m = K.KalmanNLL(h, d, T, B, "cuda", dt)
    nll, grads, obsbar = m.step(*[dev(p, dt) for p in model], dev(obs, dt))
    return (nll.cpu().numpy(), {k: v.cpu().numpy() for k, v in grads.items()}, obsbar.cpu().numpy())


@pytest.mark.parametrize("name", [str(c) for c in GOLD["cases"]])
def test_kalman_matches_reference_golden(name):
    p = [GOLD[f"{name}/in/{k}"] for k in NAMES]
    nll, grads, obsbar = run(p[:6], False, p[6][None])
    want = float(GOLD[f"{name}/nll"])
    assert abs(nll[0] - want) / max(1.0, abs(want)) < TOL
    for k in NAMES[:6]:
        assert rel(grads[k], GOLD[f"{name}/grad/{k}"]) < TOL, k
    assert rel(obsbar[0], GOLD[f"{name}/grad/obs"]) < TOL


def test_kalman_random_walk_kat():
    # proj/tests/test_models.cpp:187-197
    one, zero = np.ones((1, 1)), np.zeros((1, 1))
    nll, _, _ = run([one, one, one, one, zero, one], False, np.zeros((1, 2, 1)))
    assert abs(nll[0] - 2.6425960226263948) < 1e-12 * 2.65


@pytest.mark.parametrize("h,d,T,B", [(2, 2, 7, 5), (8, 8, 40, 33), (5, 3, 25, 7), (32, 16, 6, 3)])
def test_kalman_batch_per_sequence_params(h, d, T, B):
    r = O.rng(7 + h + d)
    m = O.random_kalman(r, h, d, T, batch=B)
    nll, grads, obsbar = run(list(m[:6]), True, m[6])
    for b in range(B):
        on, og = O.kalman_port(*[x[b] for x in m])
        assert abs(nll[b] - on) / max(1.0, abs(on)) < TOL
        for k, w in zip(NAMES[:6], og[:6]):
            assert rel(grads[k][b], w) < TOL, (b, k)
        assert rel(obsbar[b], og[6]) < TOL


def test_kalman_shared_model_sums_gradients():
    """One model over many sequences (param_stride 0): per-sequence NLLs and
    the gradient of the summed NLL (the tape's shared-leaf accumulation)."""
    r = O.rng(99)
    h, d, T, B = 4, 2, 30, 17
    model = list(O.random_kalman(r, h, d, T))[:6]
    obs = r.standard_normal((B, T, d))
    nll, grads, _ = run(model, False, obs)
    tot = {k: np.zeros_like(v) for k, v in zip(NAMES[:6], model)}
    for b in range(B):
        on, og = O.kalman_port(*model, obs[b])
        assert abs(nll[b] - on) / max(1.0, abs(on)) < TOL
        for k, w in zip(NAMES[:6], og[:6]):
            tot[k] += w
    for k in NAMES[:6]:
        assert rel(grads[k], tot[k]) < TOL, k


def test_kalman_f32():
    r = O.rng(5)
    m = O.random_kalman(r, 3, 2, 12, batch=4)
    nll, grads, _ = run(list(m[:6]), True, m[6], torch.float32)
    for b in range(4):
        on, og = O.kalman_port(*[x[b] for x in m])
        assert abs(nll[b] - on) / max(1.0, abs(on)) < 1e-4
        for k, w in zip(NAMES[:6], og[:6]):
            assert rel(grads[k][b], w) < 2e-3, (b, k)


def test_kalman_not_spd_and_shapes():
    r = O.rng(3)
    m = [x.copy() for x in O.random_kalman(r, 2, 2, 5, batch=3)]
    m[3][1] = -np.eye(2) * 1e3  # sequence 1: S_v makes the step-0 innovation covariance indefinite
    h, d, T, B = 2, 2, 5, 3
    km = K.KalmanNLL(h, d, T, B)
    with pytest.raises(L.NotPositiveDefiniteError) as e:
        km.step(*[dev(x) for x in m[:6]], dev(m[6]))
    assert e.value.batch_index == 1 and e.value.step == 0
    with pytest.raises(L.ShapeError):
        K.KalmanNLL(2, 2, 0)
    with pytest.raises(L.ShapeError):
        km.step(*[dev(x) for x in m[:5]], dev(m[5][:, :1, :]), dev(m[6]))
    with pytest.raises(L.ShapeError):  # blocks beyond the kernel's 32 x 32 design
        K.KalmanNLL(33, 2, 4).step(*[dev(x) for x in O.random_kalman(r, 33, 2, 4)[:6]],
                                    dev(np.zeros((1, 4, 2))))


_GENERIC = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import oracle as O
from paper_1710_08717_b200 import kalman as K
h, d, T, B = (int(v) for v in sys.argv[2:6])
m = O.random_kalman(O.rng(5), h, d, T, batch=B)
dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in m]
nll, grads, obsbar = K.KalmanNLL(h, d, T, B).step(*dev)
np.savez(sys.argv[6], nll=nll.cpu().numpy(), obsbar=obsbar.cpu().numpy(),
         **{k: v.cpu().numpy() for k, v in grads.items()})
"""


@pytest.mark.parametrize("h,d", [(8, 8), (4, 4), (8, 4)])
def test_kalman_specialised_bitwise_equals_runtime_size_kernel(tmp_path, h, d):
    # the compile-time-size kernels (k_kalman<T, 32, H, D>) keep the runtime-size
    # kernel's operation order: results are bitwise identical
    import subprocess
    import sys
    T, B = 30, 40
    root = os.path.dirname(HERE)
    outs = {}
    for spec in ("0", "1"):
        f = str(tmp_path / f"k{spec}.npz")
        env = dict(os.environ, DLA_KALMAN_SPECIALISE=spec)
        subprocess.run([sys.executable, "-c", _GENERIC, root, str(h), str(d), str(T), str(B), f], check=True,
                       env=env, timeout=300)
        outs[spec] = np.load(f)
    for k in outs["0"].files:
        assert np.array_equal(outs["0"][k], outs["1"][k]), k
