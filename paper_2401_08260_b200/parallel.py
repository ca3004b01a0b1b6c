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


# ---------------------------------------------------------------------------------------------------------------
# Point-parallel driver for the large-N Fourier path (include/sks.h, sks_exchange_fn).  Slice ranges stop scaling
# where N, M >> P: the direction-independent operand pass over all points is replicated on every rank and a rank
# with fewer than 128 slices leaves tensor-core tile rows idle.  The fast Fourier summation is linear in the
# sources up to the grids and pointwise in the targets after them, so rank r takes the point rows
# [r n / G, (r+1) n / G) of x, w and of y with ALL slices; the ranks meet three times inside the call: rank 0's
# centre mu (d doubles), the maxima of 8 norm words, and the sum of each slice batch's grids (P_batch x n_cap
# floats) -- all small against the point data.  Every pass over the points is divided by G.


def point_range(rank: int, world: int, n: int) -> Tuple[int, int]:
    """[begin, end) of the point rows of rank `rank` (contiguous, sizes differ by at most one)."""
    if not (0 <= rank < world) or world <= 0 or n <= 0:
        raise ValueError("bad rank/world/n")
    return rank * n // world, (rank + 1) * n // world


def make_exchange(workspace, group=None):
    """The sks_exchange_fn of a torch.distributed group for a call whose workspace is the CUDA uint8 tensor
    `workspace`: (callback, keepalive).  Collectives run on views of the workspace (dev_ptr lies inside it), on the
    current stream -- the stream the call is given.  Host-side failures are reported through the return code."""
    import torch
    import torch.distributed as dist

    from . import _lib

    base = workspace.data_ptr()
    src = dist.get_global_rank(group, 0) if group is not None else 0
    errors = []

    def cb(_user, op, dev_ptr, count, _stream):
        try:
            off = int(dev_ptr) - base
            size = {_lib.XCHG_BCAST_F64: 8, _lib.XCHG_MAX_I32: 4, _lib.XCHG_SUM_F32: 4}[op]
            if off < 0 or off + count * size > workspace.numel():
                raise ValueError("exchange buffer outside the workspace")
            raw = workspace[off:off + count * size]
            if op == _lib.XCHG_BCAST_F64:
                dist.broadcast(raw.view(torch.float64), src=src, group=group)
            elif op == _lib.XCHG_MAX_I32:
                dist.all_reduce(raw.view(torch.int32), op=dist.ReduceOp.MAX, group=group)
            else:
                dist.all_reduce(raw.view(torch.float32), op=dist.ReduceOp.SUM, group=group)
            return 0
        except Exception as e:  # noqa: BLE001  (a Python exception must not unwind through the C caller)
            errors.append(e)
            return 1

    fn = _lib.EXCHANGE_FN(cb)
    return fn, errors


def point_sharded_sum(sks_sum, sks_workspace_size, x_local, y_local, w_local, kind: str, scale: float, P: int,
                      seed: int, group=None, **opts):
    """s for this rank's targets y_local from ALL ranks' sources (every rank passes its own rows).  `sks_sum` and
    `sks_workspace_size` are the binding's functions (injected, as in distributed_sliced_sum)."""
    import torch

    N, d = x_local.shape
    ws = torch.empty(max(256, sks_workspace_size(N, y_local.shape[0], d, kind, scale, P, **opts)), dtype=torch.uint8,
                     device=x_local.device)
    fn, errors = make_exchange(ws, group)
    try:
        return sks_sum(x_local, y_local, w_local, kind, scale, P, seed, workspace=ws, exchange=fn, **opts)
    except Exception:
        if errors:
            raise errors[0]
        raise
