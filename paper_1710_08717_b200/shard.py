"""Batch sharding across GPUs (one process per GPU) and the single collective
of the GP/BLR use cases.

The reference has one batch loop, ``for_each_slice`` (dl/matrix.hpp:217-240),
which deals slice b to thread b mod T inside one process.  Here a batch is
split into contiguous per-rank ranges (host pointer offsets only, no data
movement between GPUs); every rank runs the batched kernels on its range; the
only exchange is one all-reduce of the summed scalar loss and the
hyperparameter gradient (a few dozen bytes) — NCCL over NVLink on B200,
gloo on CPU for the multi-process tests.
"""
from __future__ import annotations

import torch


def shard_range(batch: int, rank: int, world: int):
    """Contiguous [start, end) of a batch for `rank` (sizes differ by <= 1)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def allreduce_loss_grad(loss_grad: torch.Tensor) -> torch.Tensor:
    """Sum [loss, grad...] over ranks in place (no-op without a process group).

    ``loss_grad`` is a 1-D float64 tensor on the rank's device (CUDA for NCCL,
    CPU for gloo).  Deterministic for a fixed world size."""
    dist = torch.distributed
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(loss_grad, op=dist.ReduceOp.SUM)
    return loss_grad
