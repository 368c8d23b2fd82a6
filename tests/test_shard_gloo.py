"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 path:
contiguous batch sharding + the single all-reduce of (loss, dloss/dtheta) of
the C5 marginal-likelihood workload.  Per-rank compute here is the CPU oracle
(test infrastructure) evaluating the same graph as paper_1710_08717_b200.c5;
the sharding / reduction code under test is the product's shard module."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1710_08717_b200.shard import allreduce_loss_grad, shard_range

LOG_2PI = 1.8378770664093454835606594728112353


def c5_item_oracle(port, s, y, theta):
    """phi and dphi/dtheta of one item through the oracle's per-op pullbacks."""
    from oracle import oracle as O
    return O.c5_item(port, s, y, theta)


def make_problem(batch, n, seed=3):
    from oracle import oracle as O
    r = O.rng(seed)
    return O.random_spd(n, r, batch=batch), r.standard_normal((batch, n, 1))


def _worker(rank, world, port_no, batch, n, theta, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    port = O.port()
    s, y = make_problem(batch, n)
    lo, hi = shard_range(batch, rank, world)
    acc = torch.zeros(2, dtype=torch.float64)
    for i in range(lo, hi):
        phi, g = c5_item_oracle(port, s[i], y[i], theta)
        acc += torch.tensor([phi, g], dtype=torch.float64)
    allreduce_loss_grad(acc)
    q.put((rank, lo, hi, acc.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_shard_range_partitions_exactly():
    for batch in (0, 1, 7, 64, 65536):
        for world in (1, 2, 3, 8):
            rs = [shard_range(batch, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == batch
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_two_rank_allreduce_matches_single_process(port):
    batch, n, theta = 7, 6, math.log(0.3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pn = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, pn, batch, n, theta, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s, y = make_problem(batch, n)
    want = np.zeros(2)
    for i in range(batch):
        want += np.array(c5_item_oracle(port, s[i], y[i], theta))
    covered = sorted((lo, hi) for _, lo, hi, _ in res)
    assert covered == [(0, 4), (4, 7)]
    for _, _, _, got in res:
        np.testing.assert_allclose(got, want, rtol=1e-12)
    # FD check of the hyperparameter gradient of the summed loss
    h = 1e-6
    fp = sum(c5_item_oracle(port, s[i], y[i], theta + h)[0] for i in range(batch))
    fm = sum(c5_item_oracle(port, s[i], y[i], theta - h)[0] for i in range(batch))
    assert abs((fp - fm) / (2 * h) - want[1]) / max(1, abs(want[1])) < 1e-6
