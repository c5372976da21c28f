"""Data-parallel plumbing around libhydro (one process per GPU, torch.distributed).

The eddy shards naturally: tuples are independent, so each rank owns contiguous id ranges and runs
its own eddy; the only exchange is the per-batch statistics delta, all-reduced by NCCL inside
libhydro before every fold.  These helpers hold the host-side parts that are not in
the C library: the shard assignment, the NCCL unique-id broadcast and max-over-ranks timing.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def shard_ids(tuples_per_rank: int, rank: int, world: int, step: int = 0) -> Tuple[int, int]:
    """Weak scaling: step s gives rank r the contiguous ids [(s*world + r) * n, (s*world + r + 1) * n).

    Concatenating the ranks' ranges in rank order (and steps in order) reproduces the global input
    order, so the union of the ranks' result rows in that order equals the 1-GPU result.
    """
    start = (step * world + rank) * tuples_per_rank
    return start, start + tuples_per_rank


def split_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Strong scaling: contiguous [a, b) share of n ids for rank r (sizes differ by at most 1)."""
    return (n * rank) // world, (n * (rank + 1)) // world


def broadcast_unique_id(dist, rank: int, make_uid: Callable[[], bytes]) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id (hydro_nccl_unique_id); every rank receives it."""
    obj = [make_uid() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(value: float, dist=None, device: Optional[str] = None) -> float:
    """Timing rule: the job's time is the slowest rank's (all-reduce MAX)."""
    if dist is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(values, dist=None, device: Optional[str] = None):
    """Element-wise integer sum (the statistics merge libhydro performs with ncclAllReduce)."""
    if dist is None:
        return list(values)
    import torch

    t = torch.tensor(list(values), dtype=torch.int64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()
