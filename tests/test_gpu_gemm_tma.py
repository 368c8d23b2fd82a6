"""The TMA-fed persistent fp64 GEMM (csrc/gemm_tma.cu) on every operand
layout, masks, triangular operands, batches, ragged edges and alpha / beta.

DLA_GEMM_TMA is read once per process: the checks run in subprocesses with
DLA_GEMM_TMA=2 (the TMA kernel for every f64 product with m, n, k >= 256,
whatever its tile count) against torch's fp64 matmul, the CPU oracle's potrf
pullback, and the generic-kernel run of the same GP step (DLA_GEMM_TMA=0)."""
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
import itertools, sys
import numpy as np, torch
from oracle import oracle as O
from paper_1710_08717_b200 import linalg as L
from paper_1710_08717_b200 import gp
r = O.rng(77)
port = O.port()
# (1) plain products, every transposition, ragged edges, batch, alpha / beta
for (m, n, k), B in [((520, 600, 700), 2), ((256, 256, 256), 1), ((1000, 300, 257), 1), ((384, 1030, 512), 3)]:
    for ta, tb in itertools.product([0, 1], repeat=2):
        a = torch.from_numpy(r.standard_normal((B,) + ((k, m) if ta else (m, k)))).cuda()
        b = torch.from_numpy(r.standard_normal((B,) + ((n, k) if tb else (k, n)))).cuda()
        c0 = torch.from_numpy(r.standard_normal((B, m, n))).cuda()
        c = c0.clone()
        L.gemm_into(c, a, b, ta, tb, 1.5, 0.5)
        oa = a.transpose(-1, -2) if ta else a
        ob = b.transpose(-1, -2) if tb else b
        want = 1.5 * (oa @ ob) + 0.5 * c0
        err = ((c - want).abs().max() / want.abs().max()).item()
        assert err < 1e-13, (m, n, k, ta, tb, err)
# (2) the potrf pullback's triangular products (P' = tril(L^T Lbar), W = P' L^-1,
#     Z = L^-T W) at inverse-path sizes, lower and upper, batched
for n, B in [(512, 2), (1024, 1), (768, 1)]:
    a = O.random_spd(n, r, batch=B)
    for lower in (1, 0):
        l = L.potrf(torch.from_numpy(a).cuda(), lower)
        lb = torch.from_numpy(r.standard_normal((B, n, n))).cuda()
        lb = lb.tril() if lower else lb.triu()
        got = L.potrf_backward(lb, l, lower).cpu().numpy()
        for s in range(B):
            want = port.potrf_bwd(lb[s].cpu().numpy(), l[s].cpu().numpy(), lower)
            err = np.abs(got[s] - want).max() / np.abs(want).max()
            assert err < 1e-10, (n, lower, s, err)
        assert np.array_equal(got, np.swapaxes(got, 1, 2))
# (3) the GP step (its products through the TMA kernel) against the stored
#     generic-kernel result of the same inputs
x = torch.from_numpy(r.standard_normal((1, 1024, 8))).cuda()
y = torch.from_numpy(r.standard_normal((1, 1024, 1))).cuda()
g = gp.GPNLL(1024, 8, 1, "cuda")
out = [t.clone().cpu() for t in g.step(x, y, 1.0, 1.0, 0.1)]
g.check()
torch.save(out, sys.argv[1])
print("ok")
"""


def _run(env_val, path, bn=None):
    env = dict(os.environ, PYTHONPATH=ROOT, DLA_GEMM_TMA=env_val)
    if bn:
        env["DLA_GEMM_TMA_BN"] = bn  # force the tile width (default: 64 triangular / masked, 128 plain)
    p = subprocess.run([sys.executable, "-c", SCRIPT, path], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout + p.stderr


@pytest.mark.parametrize("bn", [None, "128", "64"])
def test_gemm_tma_products_and_pullbacks(tmp_path, bn):
    _run("2", str(tmp_path / "tma.pt"), bn)
    _run("0", str(tmp_path / "generic.pt"))
    a = torch.load(tmp_path / "tma.pt")
    b = torch.load(tmp_path / "generic.pt")
    for u, v in zip(a, b):
        assert torch.allclose(u, v, rtol=1e-11, atol=1e-11), (u, v)
