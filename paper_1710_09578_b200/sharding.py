"""Column sharding of a transform over the GPUs of one node.

Columns of a (rows, K) block are independent (every structured operator acts
on each column separately, reference core.py:128-149), so the multi-GPU
decomposition is a partition of the columns into contiguous slices, one per
rank (one process per GPU, torch.distributed for the plumbing).  The data path
has no collective: each rank transforms its slice with its own device plan.
Collectives appear only outside the hot path — the max-over-ranks timing
reduction of the benchmark and the optional gather of results.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np


def column_slices(ncols: int, world: int) -> list[tuple[int, int]]:
    """Contiguous [start, stop) column slices of near-equal size, one per rank."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    base, extra = divmod(int(ncols), int(world))
    out, start = [], 0
    for r in range(world):
        stop = start + base + (1 if r < extra else 0)
        out.append((start, stop))
        start = stop
    return out


def local_columns(x, rank: int, world: int):
    """This rank's column slice of a (rows, K) block (a contiguous copy)."""
    a, b = column_slices(x.shape[1], world)[rank]
    part = x[:, a:b]
    if hasattr(part, "contiguous"):
        return part.contiguous()
    return np.ascontiguousarray(part)


def shard_apply(apply_fn: Callable, x, rank: int, world: int):
    """Apply a column-wise operator to this rank's slice only (no collective)."""
    return apply_fn(local_columns(x, rank, world))


def gather_columns(local, group=None, sizes: Sequence[int] | None = None):
    """Reassemble the full block from every rank's slice (torch.distributed
    all_gather; slices may differ in width by one column)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = local if isinstance(local, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(local))
    widths = torch.tensor([t.shape[1]], dtype=torch.int64, device=t.device)
    all_w = [torch.zeros_like(widths) for _ in range(world)]
    dist.all_gather(all_w, widths, group=group)
    wmax = int(max(int(w.item()) for w in all_w))
    pad = torch.zeros((t.shape[0], wmax), dtype=t.dtype, device=t.device)
    pad[:, : t.shape[1]] = t
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    parts = [b[:, : int(w.item())] for b, w in zip(bufs, all_w)]
    out = torch.cat(parts, dim=1)
    return out if isinstance(local, torch.Tensor) else out.numpy()


def max_over_ranks(value: float, group=None, device=None) -> float:
    """The slowest rank's time (multi-GPU throughput is limited by it)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
