"""Block-row distributed chain (configs[4] path).

CPU: world_size 2 over gloo, with a torch-CPU TEST DOUBLE of the slab
product (the library's op programs, gathers, operand caching, commuting of
the sine product and doubling bookkeeping all run for real); the assembled
result is checked against the oracle.  GPU: world_size 1 through the real
sm_100a slab kernel against the oracle and the single-GPU path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cossin_oracle as orc
from tests._util import rel1


def np_slab_op(op, slab, M, n, row0, rhs_full, in0, s, dbl_step, cos_rows,
               sin_rows, scratch, stream):
    """Test double of csm_slab_op: the same op semantics in torch float64."""
    def slot(i):
        return in0 if i == 0 else slab[i]
    acc = slot(op.lhs) @ rhs_full
    eye = torch.eye(n, dtype=torch.float64)[row0:row0 + M]
    outs = []
    final_now = (s == 0) if dbl_step < 0 else (s == dbl_step + 1)
    for sl, scale, final, terms in op.outs:
        v = torch.zeros((M, n), dtype=torch.float64)
        for src, c in terms:
            x = acc if src == -1 else eye if src == -2 else (
                outs[-3 - src] if src <= -3 else slot(src))
            v = v + c * x
        if scale == 2:
            v = v * 2.0 ** -s
        elif scale == 3:
            v = v * 2.0 ** (-2 * s)
        slab[sl] = v
        outs.append(v)
        if final and final_now:
            (cos_rows if final == 1 else sin_rows).copy_(v)


def np_slab_op_pair(ops, slab, M, n, row0, rhs_full, in0, s, dbl_step, cos_rows, sin_rows,
                    scratch, stream):
    """Test double of csm_slab_op_pair: the two doubling ops in turn (they
    read S and C and write other slots, so the order does not matter)."""
    for op in ops:
        np_slab_op(op, slab, M, n, row0, rhs_full, in0, s, dbl_step, cos_rows, sin_rows,
                   scratch, stream)


def np_slab_op_peer(op, slab, M, n, row0, rhs_slabs, in0, s, dbl_step, cos_rows,
                    sin_rows, scratch, stream):
    """Test double of csm_slab_op_peer: row block j of the right operand
    comes from rank j's slab (no gathered copy exists)."""
    rhs = torch.cat([x[op.rhs] for x in rhs_slabs], dim=0)
    np_slab_op(op, slab, M, n, row0, rhs, in0, s, dbl_step, cos_rows, sin_rows, scratch,
               stream)


def test_peer_mode_virtual_ranks_cpu():
    """Peer mode's step/barrier structure with 4 lock-stepped virtual ranks
    and test doubles: no gathers, every rank's rows of cos/sin correct."""
    from paper_2010_00465_b200 import distchain
    old = (distchain.slab_op, distchain.slab_op_peer, distchain.select)
    distchain.slab_op, distchain.slab_op_peer, distchain.select = (
        np_slab_op, np_slab_op_peer, _np_select)
    try:
        n = 256
        g = np.random.default_rng(1).standard_normal((n, n))
        a = torch.from_numpy(8.0 * (g + g.T) / (2.0 * np.sqrt(n)))
        c, s, st = distchain.cos_sin_virtual_ranks(a, 4)
    finally:
        distchain.slab_op, distchain.slab_op_peer, distchain.select = old
    rc, rs, k, sc = orc.cos_sin(a.numpy())
    assert (st.k, st.s, st.gathers) == (k, sc, 0)
    assert st.products == k + 2 * sc
    assert rel1(c.numpy(), rc) <= 1e-12
    assert rel1(s.numpy(), rs) <= 1e-12


def _np_select(a, precision):
    return orc.select(orc.norm1(a.numpy()))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_00465_b200 import distchain
        distchain.slab_op = np_slab_op
        distchain.slab_op_pair = np_slab_op_pair
        distchain.select = _np_select
        g = np.random.default_rng(0).standard_normal((n, n))
        a = torch.from_numpy(20.0 * (g + g.T) / (2.0 * np.sqrt(n)))
        c, s, st = distchain.cos_sin_distributed(a)
        q.put((rank, c.numpy(), s.numpy(), st.k, st.s, st.gathers, st.products))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_block_row_two_ranks_gloo():
    n, world = 128, 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=150) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=30)
    g = np.random.default_rng(0).standard_normal((n, n))
    a = 20.0 * (g + g.T) / (2.0 * np.sqrt(n))
    c_ref, s_ref, k, s = orc.cos_sin(a)
    for rank, c, sn, kk, ss, gathers, prods in res:
        assert (kk, ss) == (k, s)
        assert rel1(c, c_ref) <= 1e-12 and rel1(sn, s_ref) <= 1e-12
        # products: k + 2s.  Gathers for k = 7: A never (replicated), y once
        # (cached for y2 y), c4, mid, cos (reused by the first doubling step),
        # the sine product as sc A, then one C per later doubling: 3 + s.
        assert prods == k + 2 * s
        if k == 7:
            assert gathers == 3 + s if s else gathers == 4
    assert np.array_equal(res[0][1], res[1][1])


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_block_row_single_gpu_against_oracle(cuda):
    from paper_2010_00465_b200 import distchain
    import paper_2010_00465_b200 as csm
    n = 1024
    g = np.random.default_rng(0).standard_normal((n, n))
    a = 20.0 * (g + g.T) / (2.0 * np.sqrt(n))
    c, s, st = distchain.cos_sin_distributed(torch.from_numpy(a).to(cuda))
    c_ref, s_ref, k, sc = orc.cos_sin(a)
    assert (st.k, st.s) == (k, sc)
    single = csm.cos_sin(a)
    # noise gate as in test_large_symmetric_against_oracle_noise_floor
    assert rel1(c.cpu().numpy(), c_ref) <= 2e-11
    assert rel1(s.cpu().numpy(), s_ref) <= 2e-11
    assert rel1(c.cpu().numpy(), single.result.cos_part) <= 2e-11


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_peer_mode_virtual_ranks_gpu(cuda, world):
    """csm_slab_op_peer with the right operand split over `world` slabs (all
    on this GPU): bit-identical to the gather-mode chain, and the oracle."""
    from paper_2010_00465_b200 import distchain
    n = 512
    g = np.random.default_rng(3).standard_normal((n, n))
    a_np = 20.0 * (g + g.T) / (2.0 * np.sqrt(n))
    a = torch.from_numpy(a_np).cuda()
    c, s, st = distchain.cos_sin_virtual_ranks(a, world)
    c1, s1, st1 = distchain.cos_sin_distributed(a)
    assert (st.k, st.s) == (st1.k, st1.s) and st.gathers == 0
    assert torch.equal(c, c1) and torch.equal(s, s1)
    rc, rs, k, sc = orc.cos_sin(a_np)
    assert rel1(c.cpu().numpy(), rc) <= 1e-10


@pytest.mark.gpu
def test_peer_mode_symmetric_memory_single_rank(cuda):
    """cos_sin_distributed_peer through torch symmetric memory (NCCL, one
    rank, in a subprocess): allocation, rendezvous, device barriers and
    the peer-pointer product; bit-identical to the gather-mode chain."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "peer_smoke.py")],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert "peer == gather: True True" in out.stdout, out.stdout + out.stderr[-2000:]


# -- the C driver (csm_dist_cos_sin, csrc/distchain.cu) ----------------------

def _cfg5_like(n, seed=0):
    g = np.random.default_rng(seed).standard_normal((n, n))
    return 20.0 * (g + g.T) / (2.0 * np.sqrt(n))


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_c_driver_world1_bitwise_python_driver(cuda):
    """csm_dist_cos_sin at W = 1 (no communicator) runs the same products
    as the Python gather-mode driver: bit-identical outputs, same (k, s),
    gathers and product count."""
    from paper_2010_00465_b200 import distchain
    a = torch.from_numpy(_cfg5_like(1024)).to(cuda)
    c, s, st = distchain.cos_sin_distributed_c(a)
    c1, s1, st1 = distchain.cos_sin_distributed(a, driver="python")
    assert (st.k, st.s) == (st1.k, st1.s)
    assert st.products == st1.products == st.k + 2 * st.s
    assert st.gathers == 0  # W = 1 reads the slab itself
    assert torch.equal(c, c1) and torch.equal(s, s1)


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_c_driver_nccl_forced_gathers_world1(cuda):
    """The NCCL path of the C driver on one GPU: a one-rank communicator
    (csm_nccl_get_unique_id / csm_nccl_comm_init_rank) and every non-A
    right operand all-gathered by ncclAllGather into the gather pool, with
    the cache of distchain.py (same gather count): bit-identical."""
    from paper_2010_00465_b200 import distchain
    a = torch.from_numpy(_cfg5_like(1024, seed=1)).to(cuda)
    c, s, st = distchain.cos_sin_distributed_c(a, force_gather=True)
    c1, s1, st1 = distchain.cos_sin_distributed(a, driver="python")
    assert st.gathers == st1.gathers > 0
    assert torch.equal(c, c1) and torch.equal(s, s1)


@pytest.mark.gpu
@pytest.mark.timeout(900)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_c_driver_virtual_ranks_k_split(cuda, world):
    """W virtual ranks on this GPU (csm_dist_cos_sin_virtual): every first
    gather of an operand is overlapped with the K-split product (own rows
    first, then the rest plus the partial sum).  Same schedule (gathers,
    products) as the Python driver; outputs within the reference's own
    noise of the oracle and of the unsplit chain."""
    from paper_2010_00465_b200 import distchain
    from tests._util import permuted_noise
    n = 1024
    a_np = _cfg5_like(n, seed=2)
    a = torch.from_numpy(a_np).to(cuda)
    c, s, st = distchain.cos_sin_virtual_gather(a, world)
    c1, s1, st1 = distchain.cos_sin_distributed(a, driver="python")
    assert (st.k, st.s, st.gathers, st.products) == (st1.k, st1.s, st1.gathers, st1.products)
    (rc, rs, k, sc), noise = permuted_noise(orc.cos_sin, a_np, np.random.default_rng(3))
    assert (st.k, st.s) == (k, sc)
    gate = max(1e-12, 4.0 * noise)
    assert rel1(c.cpu().numpy(), rc) <= gate and rel1(s.cpu().numpy(), rs) <= gate
    assert rel1(c.cpu().numpy(), c1.cpu().numpy()) <= gate
    # K-split changes only the summation order: symmetric input, symmetric cos
    assert float((c - c.T).abs().max() / c.abs().max()) <= 1e-12


@pytest.mark.gpu
def test_c_driver_errors(cuda):
    import ctypes

    from paper_2010_00465_b200 import _lib, distchain
    with pytest.raises(ValueError):
        distchain.cos_sin_virtual_gather(torch.zeros((64, 64), device=cuda), 2)  # not f64
    with pytest.raises(RuntimeError, match="multiple of 64"):
        distchain.cos_sin_virtual_gather(torch.zeros((192, 192), dtype=torch.float64,
                                                     device=cuda), 2)
    bad = torch.from_numpy(_cfg5_like(128)).to(cuda)
    bad[3, 5] = float("nan")
    import paper_2010_00465_b200 as csm
    with pytest.raises(csm.MatrixInputError):
        distchain.cos_sin_distributed_c(bad)
    L = _lib.lib()
    k = ctypes.c_int32()
    rc = L.csm_dist_cos_sin(0, ctypes.c_void_p(bad.data_ptr()), None, None, 128, None, 1,
                            ctypes.byref(k), ctypes.byref(k), ctypes.byref(k), None, 0, None)
    assert rc == _lib.ERR_ARG  # CSM_DIST_FORCE_GATHER without a communicator
