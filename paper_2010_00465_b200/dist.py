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


def batch_costs(a_full, family=None, precision=None, t=None):
    """Per-matrix product counts k + 2s of a batch, for load balancing only
    (the results always use the device's own selection): induced 1-norms
    (column sums) on whatever device holds the batch, then the library's
    host-twin selection (csm_select_host, driver.py:64-88)."""
    import torch

    from .api import select_batch
    from .records import Precision, SchemeFamily
    family = family or SchemeFamily.COS_SIN_TAYLOR
    precision = precision or Precision.DOUBLE
    x = a_full if isinstance(a_full, torch.Tensor) else torch.from_numpy(np.asarray(a_full))
    if x.shape[0] == 0:
        return np.zeros(0)
    if x.shape[-1] == 0:
        return np.zeros(x.shape[0])
    nrm = x.abs().to(torch.float64).sum(dim=-2).amax(dim=-1).cpu().numpy()
    if t is not None:
        tv = np.broadcast_to(np.asarray(t.cpu() if isinstance(t, torch.Tensor) else t,
                                        dtype=np.float64).reshape(-1), nrm.shape)
        nrm = tv * tv * nrm
    k, sc, st = select_batch(nrm, family, precision)
    return np.where(st == 0, k + 2 * sc, 0).astype(np.float64)


def _rank_device():
    import torch
    return torch.device("cuda", torch.cuda.current_device())


def _sharded(a_full, t, precision, group, gather, balance, device, compute):
    import torch
    import torch.distributed as dist

    from .records import Precision, SchemeFamily
    precision = precision or Precision.DOUBLE
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    host_numpy = not isinstance(a_full, torch.Tensor)
    B = int(a_full.shape[0])
    if balance == "cost":
        fam = SchemeFamily.WAVE_KERNEL if t is not None else SchemeFamily.COS_SIN_TAYLOR
        lo, hi = cost_balanced_bounds(batch_costs(a_full, fam, precision, t), world)[rank]
    elif balance == "count":
        lo, hi = shard_bounds(B, world, rank)
    else:
        raise ValueError(f"balance must be 'cost' or 'count', got {balance!r}")
    dev = torch.device(device) if device is not None else _rank_device()
    shard = a_full[lo:hi]
    shard = (torch.from_numpy(np.ascontiguousarray(shard)) if host_numpy else shard).to(dev)
    t_shard = None
    if t is not None:
        tv = t if isinstance(t, torch.Tensor) else torch.as_tensor(
            np.asarray(t, dtype=np.float64).reshape(-1))
        if tv.numel() == 1:
            tv = tv.reshape(1).expand(B)
        t_shard = tv[lo:hi].to(device=dev, dtype=torch.float64)
    rep = compute(shard, t_shard, precision)
    out = [rep.cos_part, rep.sin_part,
           torch.as_tensor(rep.k, device=dev), torch.as_tensor(rep.s, device=dev)]
    if gather:
        out = [gather_shards(x, group) for x in out]
    if host_numpy:
        out = [x.cpu().numpy() for x in out]
    return tuple(out)


def cos_sin_sharded(a_full, precision=None, *, group=None, gather=True, balance="cost",
                    device=None):
    """cos/sin of a batch (B, n, n) replicated on every rank of `group`:
    each rank computes one contiguous shard on its own GPU (cos_sin_batched)
    with no collective on the data path.  balance='cost' cuts the batch at
    equal total product count k + 2s (batch_costs), 'count' at equal matrix
    count.  With gather=True every rank receives the full results (one
    all-gather per output).  Returns (cos, sin, k, s) -- full or this
    rank's shard -- as numpy arrays for numpy input, else tensors on the
    rank's device."""
    from .api import cos_sin_batched
    return _sharded(a_full, None, precision, group, gather, balance, device,
                    lambda x, _t, p: cos_sin_batched(x, p))


def wave_cos_sin_sharded(a_full, t, precision=None, *, group=None, gather=True,
                         balance="cost", device=None):
    """The wave pair c(t^2 A), s(t, A) of a batch sharded like
    cos_sin_sharded (t: one scalar or one value per matrix)."""
    from .api import wave_cos_sin_batched
    return _sharded(a_full, t, precision, group, gather, balance, device,
                    lambda x, tt, p: wave_cos_sin_batched(x, tt, p))
