"""The non-default potrf schedules (DLA_POTRF_MODE, read once per process):
1 = recursive split, 2 = blocked look-ahead (default), 3 = persistent tile
dataflow.  Each runs in a subprocess against numpy's Cholesky and the same
failure semantics as the default path (dl/cholesky.hpp:49-53)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, torch
from oracle import oracle as O
from paper_1710_08717_b200 import linalg as L
r = O.rng(31)
for n, B in [(300, 2), (256, 1), (513, 1), (130, 3)]:
    a = O.random_spd(n, r, batch=B)
    got = L.potrf(torch.from_numpy(a).cuda()).cpu().numpy()
    want = np.linalg.cholesky(a)
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err < 1e-12, (n, err)
    assert np.all(np.triu(got, 1) == 0)
a = O.random_spd(300, r, batch=2)
a[1, 200, 200] = -1e6
x = torch.from_numpy(a).cuda()
try:
    L.potrf_inplace(x)
    raise SystemExit("no error raised")
except L.NotPositiveDefiniteError as e:
    assert e.batch_index == 1 and e.step == 200, (e.batch_index, e.step)
# GP driver: dla_gp_potrf_inv_f64 under this schedule (no blocked hook point
# in mode 1/3: the early half of L^-1 forms after the factorization) equals
# potrf + dla_potrf_bwd_begin_f64 bitwise
from paper_1710_08717_b200 import gp
xg = torch.from_numpy(r.standard_normal((1, 1024, 8))).cuda()
yg = torch.from_numpy(r.standard_normal((1, 1024, 1))).cuda()
outs = []
for early in (False, True):
    gp._EARLY = early
    g = gp.GPNLL(1024, 8, 1, "cuda")
    outs.append([t.clone() for t in g.step(xg, yg, 1.0, 1.0, 0.1)])
    g.check()
assert all(torch.equal(u, v) for u, v in zip(*outs))
print("ok")
"""


@pytest.mark.parametrize("mode", ["1", "3", "tma"])
def test_potrf_schedule(mode):
    # "tma": the default look-ahead with its trailing updates on the TMA-fed
    # update kernel (syrk_tma.cu, DLA_POTRF_SYRK_TMA=1)
    extra = {"DLA_POTRF_SYRK_TMA": "1"} if mode == "tma" else {"DLA_POTRF_MODE": mode}
    env = dict(os.environ, PYTHONPATH=ROOT, **extra)
    p = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout + p.stderr
