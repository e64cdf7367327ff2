"""Multi-GPU plumbing for the batched path: one process per GPU.

The batched configurations shard naturally by matrix: every
rank owns a contiguous slice of the batch and runs the single-GPU pipeline
on it -- there is no collective on the data path.  Collectives appear only
(a) to time a step as the max over ranks and (b) optionally to gather the
results on every rank.  Everything here works with any torch.distributed
backend (nccl on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Sequence

import numpy as np


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous equal-count shard [lo, hi) of `total` items for `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    base, extra = divmod(int(total), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def cost_balanced_bounds(costs: Sequence[float], world: int) -> list[tuple[int, int]]:
    """Contiguous shards with near-equal total cost (product count k + 2s per
    matrix): cut the prefix sum at the world quantiles.  Every shard boundary
    is within one matrix's cost of the ideal split."""
    c = np.asarray(costs, dtype=np.float64)
    if world <= 0:
        raise ValueError("world must be positive")
    pref = np.concatenate([[0.0], np.cumsum(c)])
    total = pref[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        i = int(np.searchsorted(pref, target, side="left"))
        i = min(max(i, cuts[-1]), len(c))
        if i > 0 and abs(pref[i - 1] - target) < abs(pref[i] - target):
            i -= 1
        cuts.append(max(i, cuts[-1]))
    cuts.append(len(c))
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a scalar over the ranks (the step time of a multi-GPU run)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def gather_shards(local, group=None):
    """All-gather variable-length shards along dim 0 (pads to the longest
    shard, then trims); returns the concatenation in rank order."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return local
    world = dist.get_world_size(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)


def cos_sin_sharded(a_full, precision=None, *, group=None, gather=True):
    """cos/sin of a batch spread over the ranks of `group`: each rank computes
    its contiguous shard on its own GPU (cos_sin_batched), and with
    gather=True every rank receives the full results.  Returns
    (cos, sin, k, s) -- full or this rank's shard."""
    import torch.distributed as dist

    from .api import cos_sin_batched
    from .records import Precision
    precision = precision or Precision.DOUBLE
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_bounds(a_full.shape[0], world, rank)
    rep = cos_sin_batched(a_full[lo:hi], precision)
    if not gather:
        return rep.cos_part, rep.sin_part, rep.k, rep.s
    return (gather_shards(rep.cos_part, group), gather_shards(rep.sin_part, group),
            gather_shards(rep.k, group), gather_shards(rep.s, group))
