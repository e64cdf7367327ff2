"""Block-row distributed cos/sin of ONE large matrix (configs[4]: 8192^2).

SURVEY.md 8e: the matrix is split by rows over the W ranks (M = n / W rows
each, one process per GPU).  Every product of the chain is

    out_rows = L_rows @ R_full,

so the only exchange is an all-gather of the current right operand over
NVLink (NCCL, through torch.distributed) -- or, in peer mode, no gather at
all: the slabs live in torch symmetric memory and csm_slab_op_peer streams
the right operand's row blocks straight from the owning GPUs inside the
GEMM (cos_sin_distributed_peer below).  Polynomials in A commute, which
removes gathers: the input A is replicated on every rank, so A A and the
final sine product (computed as sc A instead of A sc) need none, and a
gathered operand is cached until its slot is overwritten -- the degree-12
chain then gathers y, c4, mid, cos and one C per doubling step (5 + s).

The products and their fused linear combinations run in the sm_100a library
(csm_slab_op); the chain programs come from the library too
(csm_chain_program / csm_doubling_program), so this driver only schedules
gathers and launches.  Selection uses the full replicated matrix on every
rank (bit-exact norm, driver.py:64-88).
"""
from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

from . import _lib
from .records import Precision, _PREC_CODE

NSLOT = 9  # CSM_SLAB_SLOTS
_OP_HEAD = struct.Struct("<4i")
_OUT_HEAD = struct.Struct("<4i")
_TERM = struct.Struct("<iid")
MAXT = 8


@dataclass
class OpView:
    """Decoded view of one op descriptor (tiled.cu tk::Op)."""

    raw: bytearray
    lhs: int
    rhs: int
    outs: list  # [(slot, scale, final, [(src, coef), ...])]

    def swapped(self) -> "OpView":
        raw = bytearray(self.raw)
        _OP_HEAD.pack_into(raw, 0, self.rhs, self.lhs, len(self.outs), 0)
        return OpView(raw, self.rhs, self.lhs, self.outs)


def decode_op(raw: bytes) -> OpView:
    lhs, rhs, nout, _ = _OP_HEAD.unpack_from(raw, 0)
    outs = []
    off = _OP_HEAD.size
    per_out = _OUT_HEAD.size + MAXT * _TERM.size
    for q in range(3):
        base = off + q * per_out
        slot, nterms, scale, final = _OUT_HEAD.unpack_from(raw, base)
        terms = [_TERM.unpack_from(raw, base + _OUT_HEAD.size + t * _TERM.size)
                 for t in range(nterms)]
        if q < nout:
            outs.append((slot, scale, final, [(src, c) for src, _, c in terms]))
    return OpView(bytearray(raw), lhs, rhs, outs)


def chain_program(k: int, fold: bool = True):
    """(steps, cos_slot, sin_slot): steps = list of lists of OpView."""
    L = _lib.lib()
    ob = int(L.csm_op_bytes())
    buf = ctypes.create_string_buffer(ob * 16)
    nops = (ctypes.c_int32 * 16)()
    cs, ss = ctypes.c_int32(), ctypes.c_int32()
    nsteps = _lib.check(L.csm_chain_program(_lib.FAMILY_TAYLOR, k, 1 if fold else 0,
                                            buf, 16, nops, 16, ctypes.byref(cs),
                                            ctypes.byref(ss)), "csm_chain_program")
    steps, o = [], 0
    for i in range(nsteps):
        step = []
        for _ in range(nops[i]):
            step.append(decode_op(buf.raw[o * ob:(o + 1) * ob]))
            o += 1
        steps.append(step)
    return steps, cs.value, ss.value


def doubling_program(c0: int, s0: int, c1: int, s1: int):
    L = _lib.lib()
    ob = int(L.csm_op_bytes())
    buf = ctypes.create_string_buffer(ob * 2)
    _lib.check(L.csm_doubling_program(c0, s0, c1, s1, buf), "csm_doubling_program")
    return [decode_op(buf.raw[:ob]), decode_op(buf.raw[ob:2 * ob])]


# -- device primitives (replaceable by test doubles in the CPU tests) --------

def _device_slab_op(op: OpView, slab, M, n, row0, rhs_full, in0, s, dbl_step,
                    cos_rows, sin_rows, scratch, stream):
    import torch
    vp = ctypes.c_void_p
    raw = (ctypes.c_char * len(op.raw)).from_buffer(op.raw)
    _lib.check(_lib.lib().csm_slab_op(
        raw, vp(slab.data_ptr()), M, n, row0, vp(rhs_full.data_ptr()),
        vp(in0.data_ptr()), s, 0.0, dbl_step, vp(cos_rows.data_ptr()),
        vp(sin_rows.data_ptr()), 0, vp(scratch.data_ptr()), scratch.numel(),
        vp(int((stream or torch.cuda.current_stream()).cuda_stream))), "csm_slab_op")
    return int(_lib.lib().csm_last_launch_count())


def _device_slab_op_pair(ops, slab, M, n, row0, rhs_full, in0, s, dbl_step, cos_rows,
                         sin_rows, scratch, stream):
    """The doubling step's two ops (S C, C C) in one csm_slab_op_pair call:
    one launch, and one conversion of C on the Ozaki engine."""
    import torch
    vp = ctypes.c_void_p
    raw = [(ctypes.c_char * len(op.raw)).from_buffer(op.raw) for op in ops]
    _lib.check(_lib.lib().csm_slab_op_pair(
        raw[0], raw[1], vp(slab.data_ptr()), M, n, row0, vp(rhs_full.data_ptr()),
        vp(in0.data_ptr()), s, 0.0, dbl_step, vp(cos_rows.data_ptr()),
        vp(sin_rows.data_ptr()), 0, vp(scratch.data_ptr()), scratch.numel(),
        vp(int((stream or torch.cuda.current_stream()).cuda_stream))), "csm_slab_op_pair")
    return int(_lib.lib().csm_last_launch_count())


def _device_select(a, precision: Precision):
    from .api import norm1, select_batch
    k, s, st = select_batch([norm1(a)], precision=precision)
    if st[0] != 0:
        raise ValueError("norm must be finite and nonnegative")
    return int(k[0]), int(s[0])


def _device_slab_op_peer(op: OpView, slab, M, n, row0, rhs_slabs, in0, s, dbl_step,
                         cos_rows, sin_rows, scratch, stream):
    import torch
    vp = ctypes.c_void_p
    raw = (ctypes.c_char * len(op.raw)).from_buffer(op.raw)
    ptrs = [x if isinstance(x, int) else x.data_ptr() for x in rhs_slabs]
    parts = (ctypes.c_void_p * len(ptrs))(*ptrs)
    _lib.check(_lib.lib().csm_slab_op_peer(
        raw, vp(slab.data_ptr()), M, n, row0, parts, len(rhs_slabs), vp(in0.data_ptr()), s,
        0.0, dbl_step, vp(cos_rows.data_ptr()), vp(sin_rows.data_ptr()), 0,
        vp(scratch.data_ptr()), scratch.numel(),
        vp(int((stream or torch.cuda.current_stream()).cuda_stream))), "csm_slab_op_peer")
    return int(_lib.lib().csm_last_launch_count())


def _slab_scratch_size(M: int, n: int) -> int:
    """Scratch bytes of the slab calls under the calling thread's engine
    (the library checks the size it is given and fails rather than
    overflowing)."""
    L = _lib.lib()
    return int(L.csm_slab_scratch_bytes()) + int(L.csm_slab_engine_bytes(M, n))


def _peer_engine():
    """Peer mode runs every product on the DMMA engine: csm_slab_op_peer is
    DMMA-only, and the products whose right operand is the replicated A (run
    through csm_slab_op) take the same engine, so one chain never mixes
    engines."""
    from .api import engine_scope
    return engine_scope("dmma")


slab_op = _device_slab_op
slab_op_pair = _device_slab_op_pair
slab_op_peer = _device_slab_op_peer
select = _device_select


@dataclass
class DistStats:
    k: int
    s: int
    gathers: int
    products: int
    launches: int = 0  # library kernels launched by the gather-mode products


def _use_c_driver(a, group) -> bool:
    """The C driver (csm_dist_cos_sin, gathers overlapped with the K-split
    products) runs CUDA inputs on the FP64 DMMA engine over NCCL; the
    Python schedule below runs everything else (the Ozaki engine's slab
    products, and the CPU test doubles of the gloo tests)."""
    import torch.distributed as dist

    from .api import get_engine
    if not getattr(a, "is_cuda", False) or get_engine() != "dmma":
        return False
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return True
    return dist.get_backend(group) == "nccl"


def cos_sin_distributed(a, precision: Precision = Precision.DOUBLE, *,
                        group=None, gather_outputs: bool = True, driver: str = "auto"):
    """cos(a), sin(a) for one n x n float64 matrix replicated on every rank
    of `group`, computed block-row over the ranks.  Returns (cos, sin,
    stats): the full matrices if gather_outputs, else this rank's rows.
    driver: 'c' (csm_dist_cos_sin), 'python' (this module's schedule over
    torch.distributed all-gathers and csm_slab_op) or 'auto' (the C driver
    whenever it applies, see _use_c_driver)."""
    import torch
    import torch.distributed as dist
    if driver not in ("auto", "c", "python"):
        raise ValueError(f"driver must be 'auto', 'c' or 'python', got {driver!r}")
    if driver == "c" or (driver == "auto" and slab_op is _device_slab_op
                         and _use_c_driver(a, group)):
        return cos_sin_distributed_c(a, precision, group=group, gather_outputs=gather_outputs)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = int(a.shape[0])
    if a.shape != (n, n) or a.dtype != torch.float64:
        raise ValueError("expected a square float64 tensor")
    if n % (64 * world):
        raise ValueError(f"n={n} must be a multiple of 64 x world ({world})")
    M, row0 = n // world, rank * (n // world)
    a = a.contiguous()
    k, s = select(a, precision)
    steps, cos_slot, sin_slot = chain_program(k, fold=True)
    dev = a.device
    slab = torch.empty((NSLOT, M, n), dtype=torch.float64, device=dev)
    cos_rows = torch.empty((M, n), dtype=torch.float64, device=dev)
    sin_rows = torch.empty_like(cos_rows)
    scratch = None
    if dev.type == "cuda":  # + the Ozaki engine's scratch when it runs the products
        L = _lib.lib()
        scratch = torch.empty(_slab_scratch_size(M, n), dtype=torch.uint8, device=dev)
    in0 = a[row0:row0 + M]
    cache: dict[int, object] = {}
    stats = DistStats(k, s, 0, 0)

    def full(slot: int):
        if slot == 0:
            return a
        if slot not in cache:
            buf = torch.empty((n, n), dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_gather_into_tensor(buf, slab[slot].contiguous(), group=group)
            else:
                buf.copy_(slab[slot])
            cache[slot] = buf
            stats.gathers += 1
        return cache[slot]

    def run(op: OpView, dbl_step: int):
        if op.lhs == 0 and op.rhs != 0:  # A sc = sc A: keep A as the gathered side
            op = op.swapped()
        rf = full(op.rhs)
        launched = slab_op(op, slab, M, n, row0, rf, in0, s, dbl_step, cos_rows, sin_rows,
                           scratch, None)
        stats.products += 1
        stats.launches += launched or 0
        return [o[0] for o in op.outs]

    for step in steps:
        written = []
        for op in step:
            written += run(op, -1)
        for w in written:
            cache.pop(w, None)
    c0, s0 = cos_slot, sin_slot
    free = [i for i in range(1, NSLOT) if i not in (c0, s0)]
    c1, s1 = free[0], free[1]
    for i in range(s):
        ops = doubling_program(c0, s0, c1, s1)
        # both products share the gathered C: one paired call
        launched = slab_op_pair(ops, slab, M, n, row0, full(c0), in0, s, i, cos_rows,
                                sin_rows, scratch, None)
        stats.products += 2
        stats.launches += launched or 0
        for w in [o[0] for op in ops for o in op.outs]:
            cache.pop(w, None)
        c0, s0, c1, s1 = c1, s1, c0, s0
    if not gather_outputs or world == 1:
        return cos_rows, sin_rows, stats
    cfull = torch.empty((n, n), dtype=torch.float64, device=dev)
    sfull = torch.empty_like(cfull)
    dist.all_gather_into_tensor(cfull, cos_rows, group=group)
    dist.all_gather_into_tensor(sfull, sin_rows, group=group)
    return cfull, sfull, stats


# ---------------------------------------------------------------------------
# Peer mode: the all-gather fused into the product (no gathered copies).

def _peer_rank_program(a, precision, rank: int, world: int, slab, rhs_slabs,
                       cos_rows, sin_rows, scratch, stats: DistStats):
    """One rank's chain as a generator that yields at every point where all
    ranks must have finished writing before anyone reads (a cross-rank
    barrier).  A is replicated, so products whose right operand is A (and
    A sc, run as sc A) read it locally; every other right operand is read
    row block by row block from its owner through rhs_slabs."""
    n = int(a.shape[0])
    M, row0 = n // world, rank * (n // world)
    in0 = a[row0:row0 + M]
    k, s = stats.k, stats.s
    steps, cos_slot, sin_slot = chain_program(k, fold=True)

    def run(op: OpView, dbl_step: int):
        if op.lhs == 0 and op.rhs != 0:  # A X = X A: polynomials in A commute
            op = op.swapped()
        if op.rhs == 0:
            launched = slab_op(op, slab, M, n, row0, a, in0, s, dbl_step, cos_rows, sin_rows,
                               scratch, None)
        else:
            launched = slab_op_peer(op, slab, M, n, row0, rhs_slabs, in0, s, dbl_step,
                                    cos_rows, sin_rows, scratch, None)
        if rank == 0:
            stats.products += 1
            stats.launches += launched or 0

    for step in steps:
        for op in step:
            run(op, -1)
        yield
    c0, s0 = cos_slot, sin_slot
    free = [i for i in range(1, NSLOT) if i not in (c0, s0)]
    c1, s1 = free[0], free[1]
    for i in range(s):
        for op in doubling_program(c0, s0, c1, s1):
            run(op, i)
        yield
        c0, s0, c1, s1 = c1, s1, c0, s0


def cos_sin_virtual_ranks(a, world: int, precision: Precision = Precision.DOUBLE):
    """The peer-mode chain with `world` virtual ranks in ONE process (all
    slabs on this device, stepped in lock-step): exercises the multi-part
    right-operand addressing of csm_slab_op_peer and the step/barrier
    structure on a single GPU.  Returns (cos, sin, stats)."""
    import torch
    n = int(a.shape[0])
    if a.shape != (n, n) or a.dtype != torch.float64:
        raise ValueError("expected a square float64 tensor")
    if n % (64 * world):
        raise ValueError(f"n={n} must be a multiple of 64 x world ({world})")
    a = a.contiguous()
    M = n // world
    k, s = select(a, precision)
    dev = a.device
    slabs = [torch.empty((NSLOT, M, n), dtype=torch.float64, device=dev) for _ in range(world)]
    cos = torch.empty((n, n), dtype=torch.float64, device=dev)
    sin = torch.empty_like(cos)
    stats = DistStats(k, s, 0, 0)
    with _peer_engine():
        scratch = None
        if dev.type == "cuda":
            scratch = torch.empty(_slab_scratch_size(M, n), dtype=torch.uint8, device=dev)
        gens = [_peer_rank_program(a, precision, r, world, slabs[r], slabs,
                                   cos[r * M:(r + 1) * M], sin[r * M:(r + 1) * M], scratch,
                                   stats)
                for r in range(world)]
        done = False
        while not done:
            for g in gens:  # one step of every rank, then the (implicit) barrier
                try:
                    next(g)
                except StopIteration:
                    done = True
    return cos, sin, stats


_PEER_CTX: dict = {}


def cos_sin_distributed_peer(a, precision: Precision = Precision.DOUBLE, *, group=None,
                             gather_outputs: bool = True):
    """cos_sin_distributed with the all-gather fused into the product: the
    slabs are allocated in torch symmetric memory (NVLink peer mappings), a
    device-side barrier separates dependent steps, and every product reads
    the remote row blocks of its right operand directly.  One process per
    GPU; needs peer access between the GPUs of the group."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = int(a.shape[0])
    if a.shape != (n, n) or a.dtype != torch.float64:
        raise ValueError("expected a square float64 tensor")
    if n % (64 * world):
        raise ValueError(f"n={n} must be a multiple of 64 x world ({world})")
    a = a.contiguous()
    M = n // world
    k, s = select(a, precision)
    dev = a.device
    grp = group if group is not None else dist.group.WORLD
    key = (n, world, str(dev), grp.group_name)
    ctx = _PEER_CTX.get(key)
    if ctx is None:  # symmetric slabs are allocated and mapped once per shape
        slab = symm_mem.empty((NSLOT, M, n), dtype=torch.float64, device=dev)
        hdl = symm_mem.rendezvous(slab, grp.group_name)
        with _peer_engine():
            scratch = torch.empty(_slab_scratch_size(M, n), dtype=torch.uint8, device=dev)
        ctx = (slab, hdl, [int(p) for p in hdl.buffer_ptrs], scratch)
        _PEER_CTX[key] = ctx
        hdl.barrier(channel=0)  # every peer mapping is live
    slab, hdl, ptrs, scratch = ctx
    cos_rows = torch.empty((M, n), dtype=torch.float64, device=dev)
    sin_rows = torch.empty_like(cos_rows)
    stats = DistStats(k, s, 0, 0)
    hdl.barrier(channel=0)  # no rank still reads the previous call's slabs
    with _peer_engine():
        for _ in _peer_rank_program(a, precision, rank, world, slab, ptrs, cos_rows, sin_rows,
                                    scratch, stats):
            hdl.barrier(channel=0)  # this step's rows are written on every rank
    if not gather_outputs or world == 1:
        return cos_rows, sin_rows, stats
    cfull = torch.empty((n, n), dtype=torch.float64, device=dev)
    sfull = torch.empty_like(cfull)
    dist.all_gather_into_tensor(cfull, cos_rows, group=group)
    dist.all_gather_into_tensor(sfull, sin_rows, group=group)
    return cfull, sfull, stats


# ---------------------------------------------------------------------------
# The C driver (csm_dist_cos_sin, csrc/distchain.cu): the same schedule run
# from C++ over an NCCL communicator, with every first gather of an operand
# overlapped with the rank's own-rows part of its product (K-split).

_NCCL_COMMS: dict = {}


def nccl_comm(group=None):
    """An NCCL communicator (ncclComm_t) over the ranks of `group` for the C
    driver: rank 0 makes the unique id (csm_nccl_get_unique_id),
    torch.distributed broadcasts its 128 bytes, every rank joins
    (csm_nccl_comm_init_rank).  Cached per group; None at world 1."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    grp = group if group is not None else dist.group.WORLD
    key = grp.group_name
    if key not in _NCCL_COMMS:
        L = _lib.lib()
        uid = ctypes.create_string_buffer(128)
        if dist.get_rank(group) == 0:
            _lib.check(L.csm_nccl_get_unique_id(uid), "csm_nccl_get_unique_id")
        box = [uid.raw]
        dist.broadcast_object_list(box, src=dist.get_global_rank(grp, 0), group=group)
        uid = ctypes.create_string_buffer(box[0], 128)
        comm = ctypes.c_void_p()
        _lib.check(L.csm_nccl_comm_init_rank(ctypes.byref(comm), dist.get_world_size(group),
                                             uid, dist.get_rank(group)),
                   "csm_nccl_comm_init_rank")
        _NCCL_COMMS[key] = comm
    return _NCCL_COMMS[key]


_DIST_FORCE_GATHER = 1  # CSM_DIST_FORCE_GATHER


def _dist_stats(k, s):
    g, p = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.lib().csm_dist_last_stats(ctypes.byref(g), ctypes.byref(p)),
               "csm_dist_last_stats")
    return DistStats(int(k), int(s), g.value, p.value, int(_lib.lib().csm_last_launch_count()))


def _status_raise(st: int):
    from .api import _status_error
    if st != 0:
        raise _status_error(st, float("nan"))


def cos_sin_distributed_c(a, precision: Precision = Precision.DOUBLE, *, group=None,
                          comm=None, gather_outputs: bool = True, force_gather: bool = False):
    """cos_sin_distributed through the C driver csm_dist_cos_sin: `a`
    replicated on every rank (CUDA float64, n a multiple of 64 W), the
    communicator from nccl_comm(group) unless given.  force_gather makes
    even W = 1 gather through NCCL (tests the NCCL path on one GPU).
    Returns (cos, sin, stats) like cos_sin_distributed."""
    import torch
    import torch.distributed as dist
    n = int(a.shape[0])
    if a.shape != (n, n) or a.dtype != torch.float64 or not a.is_cuda:
        raise ValueError("expected a square float64 CUDA tensor")
    if comm is None:
        comm = nccl_comm(group)
        if comm is None and force_gather:  # a one-rank communicator
            L = _lib.lib()
            uid = ctypes.create_string_buffer(128)
            _lib.check(L.csm_nccl_get_unique_id(uid), "csm_nccl_get_unique_id")
            comm = ctypes.c_void_p()
            _lib.check(L.csm_nccl_comm_init_rank(ctypes.byref(comm), 1, uid, 0),
                       "csm_nccl_comm_init_rank")
            _NCCL_COMMS.setdefault("__single__", comm)
            comm = _NCCL_COMMS["__single__"]
    world = dist.get_world_size(group) if (comm is not None and dist.is_initialized()) else 1
    flags = _DIST_FORCE_GATHER if force_gather else 0
    a = a.contiguous()
    M = n // world
    L = _lib.lib()
    dev = a.device
    cos_rows = torch.empty((M, n), dtype=torch.float64, device=dev)
    sin_rows = torch.empty_like(cos_rows)
    ws_bytes = int(L.csm_dist_workspace_size(n, world, flags))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    k, s, st = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    vp = ctypes.c_void_p
    _lib.check(L.csm_dist_cos_sin(_PREC_CODE[precision], vp(a.data_ptr()),
                                  vp(cos_rows.data_ptr()), vp(sin_rows.data_ptr()), n, comm,
                                  flags, ctypes.byref(k), ctypes.byref(s), ctypes.byref(st),
                                  vp(ws.data_ptr()), ws_bytes,
                                  vp(int(torch.cuda.current_stream().cuda_stream))),
               "csm_dist_cos_sin")
    _status_raise(st.value)
    stats = _dist_stats(k.value, s.value)
    if not gather_outputs or world == 1:
        return cos_rows, sin_rows, stats
    cfull = torch.empty((n, n), dtype=torch.float64, device=dev)
    sfull = torch.empty_like(cfull)
    dist.all_gather_into_tensor(cfull, cos_rows, group=group)
    dist.all_gather_into_tensor(sfull, sin_rows, group=group)
    return cfull, sfull, stats


def cos_sin_virtual_gather(a, world: int, precision: Precision = Precision.DOUBLE):
    """The C driver's schedule for `world` virtual ranks on this GPU
    (csm_dist_cos_sin_virtual): K-split products, the gather cache and
    the all-gathers (as device copies) of the multi-GPU run, on one device.
    Returns (cos, sin, stats)."""
    import torch
    n = int(a.shape[0])
    if a.shape != (n, n) or a.dtype != torch.float64 or not a.is_cuda:
        raise ValueError("expected a square float64 CUDA tensor")
    a = a.contiguous()
    L = _lib.lib()
    cos = torch.empty((n, n), dtype=torch.float64, device=a.device)
    sin = torch.empty_like(cos)
    ws_bytes = world * int(L.csm_dist_workspace_size(n, world, _DIST_FORCE_GATHER))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=a.device)
    k, s, st = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    vp = ctypes.c_void_p
    _lib.check(L.csm_dist_cos_sin_virtual(_PREC_CODE[precision], vp(a.data_ptr()),
                                          vp(cos.data_ptr()), vp(sin.data_ptr()), n, world,
                                          ctypes.byref(k), ctypes.byref(s), ctypes.byref(st),
                                          vp(ws.data_ptr()), ws_bytes,
                                          vp(int(torch.cuda.current_stream().cuda_stream))),
               "csm_dist_cos_sin_virtual")
    _status_raise(st.value)
    return cos, sin, _dist_stats(k.value, s.value)
