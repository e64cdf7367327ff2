"""Per-op local error of the block-row chain (world 1) on one matrix: every
GPU slab op is replayed on a CPU copy of its inputs (the torch test double
of tests/test_distchain.py) and the op's outputs are compared."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2010_00465_b200 as csm
from paper_2010_00465_b200 import distchain
from tests._util import rel1
from tests.test_distchain import np_slab_op
from tests.test_gpu_guard import _cases

n = int(sys.argv[1])
nm = sys.argv[2]
eng = sys.argv[3] if len(sys.argv) > 3 else "auto"
names, a = _cases(n)
x = torch.from_numpy(a[names.index(nm)]).cuda()
dev_op, dev_pair = distchain.slab_op, distchain.slab_op_pair
count = [0]


def traced(ops, slab, M, nn, row0, rhs, in0, s, dbl, co, so, scratch, stream):
    snap = slab.cpu().clone()
    cos_c, sin_c = co.cpu().clone(), so.cpu().clone()
    if len(ops) == 1:
        r = dev_op(ops[0], slab, M, nn, row0, rhs, in0, s, dbl, co, so, scratch, stream)
    else:
        r = dev_pair(ops, slab, M, nn, row0, rhs, in0, s, dbl, co, so, scratch, stream)
    torch.cuda.synchronize()
    for op in ops:
        np_slab_op(op, snap, M, nn, row0, rhs.cpu(), in0.cpu(), s, dbl, cos_c, sin_c, None, None)
    for op in ops:
        for o in op.outs:
            e = rel1(slab[o[0]].cpu().numpy(), snap[o[0]].numpy())
            print(f"op {count[0]:2d} dbl {dbl:2d} lhs {op.lhs} rhs {op.rhs} -> slot {o[0]}: "
                  f"rel err {e:.2e}  ||out|| {float(snap[o[0]].abs().sum(0).max()):.2e}", flush=True)
        count[0] += 1
    return r


distchain.slab_op = lambda op, *rest: traced([op], *rest)
distchain.slab_op_pair = lambda ops, *rest: traced(ops, *rest)
with csm.engine_scope(eng):
    distchain.cos_sin_distributed(x)
