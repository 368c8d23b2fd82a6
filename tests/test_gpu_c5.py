"""C5 batched marginal-likelihood chain (potrf + potri + trmm + gemm2 +
sumlogdiag, forward and backward) on the GPU vs the CPU oracle's per-op
pullbacks on the same inputs."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1710_08717_b200.c5 import MarginalLikelihoods  # noqa: E402
from tests.test_shard_gloo import c5_item_oracle, make_problem  # noqa: E402


@pytest.mark.parametrize("n", [6, 64, 128])
def test_c5_chain_matches_oracle(port, n):
    batch, theta = 5, math.log(0.3)
    s, y = make_problem(batch, n, seed=n)
    m = MarginalLikelihoods(batch, n)
    out = m.step(torch.from_numpy(s).cuda(), torch.from_numpy(y).cuda(), theta)
    m.check()
    want = np.zeros(2)
    for i in range(batch):
        want += np.array(c5_item_oracle(port, s[i], y[i], theta))
    got = out.cpu().numpy()
    assert abs(got[0] - want[0]) / abs(want[0]) < 1e-11
    assert abs(got[1] - want[1]) / max(1, abs(want[1])) < 1e-9


def test_c5_shards_sum_to_full_batch():
    # bench.py --gpus N shards the C5 batch into contiguous ranges and all-reduces
    # [loss, dloss/dtheta]; on one GPU the per-shard results must sum to the
    # whole-batch result (rtol 1e-12), with the same global inputs per item.
    from paper_1710_08717_b200.shard import shard_range
    from tools.bench_configs import c5_inputs
    total, n, theta = 8192, 128, math.log(0.3)
    s, y = c5_inputs(torch, 0, total, n)
    full = MarginalLikelihoods(total, n).step(s, y, theta).clone()
    for world in (2, 4):
        acc = torch.zeros(2, dtype=torch.float64, device="cuda")
        for rank in range(world):
            lo, hi = shard_range(total, rank, world)
            ss, yy = c5_inputs(torch, lo, hi, n)
            assert torch.equal(ss, s[lo:hi]) and torch.equal(yy, y[lo:hi])  # same global items
            acc += MarginalLikelihoods(hi - lo, n).step(ss, yy, theta)
        assert torch.allclose(acc, full, rtol=1e-12, atol=0)
