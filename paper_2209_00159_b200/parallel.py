"""Multi-GPU plumbing: independent units sharded over ranks.

Queues and replay scenarios are independent ("different models
and their replicas can use Orloj in parallel"), so the data path has no
exchange.  The only collective is the final integer sum of the replay counters
(one all-reduce of [buckets x 7] int64 over NCCL / NVLink); integer sums make
the result independent of the shard count.
"""
from __future__ import annotations

import numpy as np
import torch


def shard_blocks(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n units for `rank` (score / pick queues)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def shard_round_robin(group_ids, rank: int, world: int) -> np.ndarray:
    """Indices u with group_ids[u] % world == rank (replay: round-robin over seed
    groups so every rank gets every family and SLO bucket)."""
    g = np.asarray(group_ids)
    return np.nonzero(g % world == rank)[0]


def allreduce_counters(per_bucket: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the int64 counter table over all ranks in place (NCCL on CUDA
    tensors, gloo on CPU tensors); a no-op without an initialised process group."""
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.all_reduce(per_bucket, op=torch.distributed.ReduceOp.SUM, group=group)
    return per_bucket


def finish_rate(per_bucket: torch.Tensor) -> torch.Tensor:
    """finished / total per bucket."""
    c = per_bucket.double()
    return c[:, 1] / c[:, 0].clamp(min=1)


def goodput(per_bucket: torch.Tensor) -> torch.Tensor:
    """finished requests per tick of span, per bucket."""
    c = per_bucket.double()
    return c[:, 1] / c[:, 6].clamp(min=1)
