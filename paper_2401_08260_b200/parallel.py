"""Slice-parallel multi-GPU driver (north_star): rank r of G takes the contiguous slice range
[r P / G, (r+1) P / G); each rank computes its (1/P)-scaled partial of Alg. 1's average on its own
replica of x, y, w, and ONE all-reduce SUM of the M-length partial sums combines them.  Directions depend only
on (seed, p), so the result is independent of G up to the summation order.

The compute function is injected: ``sks_sum`` on a CUDA device (NCCL process group), or any callable with the
same contract in CPU tests (gloo)."""
from __future__ import annotations

from typing import Callable, Tuple


def slice_range(rank: int, world: int, P: int) -> Tuple[int, int]:
    """[p_begin, p_end) of rank `rank` (contiguous, sizes differ by at most one)."""
    if not (0 <= rank < world) or world <= 0 or P <= 0:
        raise ValueError("bad rank/world/P")
    return rank * P // world, (rank + 1) * P // world


def distributed_sliced_sum(compute: Callable[[int, int], "object"], P: int, group=None):
    """Run ``compute(p_begin, p_end) -> partial s`` (a torch tensor, already scaled by 1/P) for this rank's slice
    range and all-reduce (SUM) the partials in place.  Returns the full estimate on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    p0, p1 = slice_range(rank, world, P)
    s = compute(p0, p1)
    if world > 1:
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    return s
