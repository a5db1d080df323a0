"""Read sharding for multi-GPU runs (one process per GPU, torch.distributed).

Reads are the unit of work: a read's hits depend only on the read and the whole
reference, so every rank maps its own contiguous share
of the reads against its own replica of the reference and nothing crosses
ranks on the data path. The collective layer only carries the barrier and the
max-over-ranks timing; hit counts can be all-gathered for reporting.
"""
from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of n reads for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n, world_size)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def max_over_ranks(values, dist=None, device="cpu"):
    """Element-wise max of a list of floats over all ranks (identity without dist)."""
    if dist is None or not dist.is_initialized():
        return list(values)
    import torch

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(values, dist=None, device="cpu"):
    if dist is None or not dist.is_initialized():
        return list(values)
    import torch

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()


def weak_scaling_value(units_per_rank: int, steps: int, world_size: int, max_ms: float) -> float:
    """Whole-job throughput: every rank's units over the slowest rank's time."""
    return units_per_rank * steps * world_size / (max_ms / 1e3)
