"""Multi-process (world_size 2, gloo, CPU) tests of the sharding plumbing the
multi-GPU bench and cos_sin_sharded use.  The GPU compute itself is not run
here (there is no CPU fallback); the shard/gather/timing logic is."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_00465_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        total = 11
        lo, hi = pdist.shard_bounds(total, world, rank)
        full = torch.arange(total * 4, dtype=torch.float64).reshape(total, 2, 2)
        local = full[lo:hi] * 2.0  # stand-in for the per-rank result
        gathered = pdist.gather_shards(local)
        ok_gather = torch.equal(gathered, full * 2.0)
        mx = pdist.max_over_ranks(float(rank + 1))
        sm = pdist.sum_over_ranks(float(hi - lo))
        q.put((rank, ok_gather, mx, sm, (lo, hi)))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover_exactly():
    for total in (0, 1, 7, 16384, 16385):
        for world in (1, 2, 3, 8):
            b = [pdist.shard_bounds(total, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == total
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in b]
            assert max(sizes) - min(sizes) <= 1


def test_cost_balanced_bounds():
    rng = np.random.default_rng(0)
    costs = rng.integers(3, 20, 4096).astype(float)
    for world in (2, 4, 8):
        b = pdist.cost_balanced_bounds(costs, world)
        assert b[0][0] == 0 and b[-1][1] == len(costs)
        loads = [costs[l:h].sum() for l, h in b]
        assert max(loads) - min(loads) <= 2 * costs.max()


@pytest.mark.timeout(120)
def test_two_rank_gather_and_timing():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=90) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
    assert all(r[1] for r in res), "gathered shards differ from the full batch"
    assert all(r[2] == 2.0 for r in res)        # max over ranks
    assert all(r[3] == 11.0 for r in res)       # shard sizes sum to the batch
    assert res[0][4] == (0, 6) and res[1][4] == (6, 11)
