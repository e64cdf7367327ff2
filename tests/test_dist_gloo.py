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


def _fake_batched(x, t, precision):
    """CPU test double of the per-rank GPU computation: the oracle per
    matrix (the real call needs a device; the plumbing around it is what is
    tested here)."""
    from types import SimpleNamespace

    from oracle import cossin_oracle as orc
    cs, ss, ks, scs = [], [], [], []
    for i in range(x.shape[0]):
        a = x[i].numpy()
        c, s, k, sc = (orc.cos_sin(a) if t is None else orc.wave_cos_sin(a, float(t[i])))
        cs.append(c), ss.append(s), ks.append(k), scs.append(sc)
    n = x.shape[-1]
    cos = torch.from_numpy(np.array(cs).reshape(-1, n, n))
    sin = torch.from_numpy(np.array(ss).reshape(-1, n, n))
    return SimpleNamespace(cos_part=cos, sin_part=sin, k=np.array(ks, dtype=np.int32),
                           s=np.array(scs, dtype=np.int32))


def _sharded_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_00465_b200 import api
        from tests._util import cfg2_like, laplacian_wave
        api.cos_sin_batched = lambda x, p: _fake_batched(x, None, p)
        api.wave_cos_sin_batched = lambda x, t, p: _fake_batched(x, t, p)
        a = cfg2_like(np.random.default_rng(3), 13, n=8)
        c, s, k, sc = pdist.cos_sin_sharded(a, device="cpu")  # numpy in -> numpy out
        costs = pdist.batch_costs(a)
        lo, hi = pdist.cost_balanced_bounds(costs, world)[rank]
        cl, sl, kl, scl = pdist.cos_sin_sharded(torch.from_numpy(a), device="cpu",
                                               gather=False)
        aw, tw = laplacian_wave(np.random.default_rng(4), 5, 6)
        wc, ws, wk, wsc = pdist.wave_cos_sin_sharded(aw, tw, device="cpu", balance="count")
        q.put((rank, type(c).__name__, c, s, k, sc, (lo, hi), costs[lo:hi].sum(),
               int(kl.numel()), type(cl).__name__, wc, ws, wk, wsc))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_two_rank_cos_sin_sharded():
    """cos_sin_sharded / wave_cos_sin_sharded at world 2 over gloo with a CPU
    test double for the per-rank GPU call: cost-balanced shards, gathered
    results equal the per-matrix oracle in batch order, numpy in -> numpy
    out, tensor in -> tensor out, gather=False -> this rank's shard."""
    from oracle import cossin_oracle as orc
    from tests._util import cfg2_like, laplacian_wave
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=150) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=30)
    a = cfg2_like(np.random.default_rng(3), 13, n=8)
    aw, tw = laplacian_wave(np.random.default_rng(4), 5, 6)
    for r in res:
        assert r[1] == "ndarray" and r[9] == "Tensor"
        for i in range(13):
            c, s, k, sc = orc.cos_sin(a[i])
            assert np.array_equal(r[2][i], c) and np.array_equal(r[3][i], s)
            assert (r[4][i], r[5][i]) == (k, sc)
        for i in range(5):
            c, s, k, sc = orc.wave_cos_sin(aw[i], float(tw[i]))
            assert np.array_equal(r[10][i], c) and np.array_equal(r[11][i], s)
            assert (r[12][i], r[13][i]) == (k, sc)
    (lo0, hi0), (lo1, hi1) = res[0][6], res[1][6]
    assert lo0 == 0 and hi0 == lo1 and hi1 == 13
    assert res[0][8] == hi0 - lo0 and res[1][8] == hi1 - lo1
    costs = np.array([res[0][7], res[1][7]])
    assert abs(costs[0] - costs[1]) <= 2 * 40  # within one matrix's cost
