"""One product L R through csm_slab_op (world 1, slab = the whole matrix)
on each engine, against an extended-precision reference, next to the
guard's a-priori bound E (oz_guard).  Diagnoses the Ozaki engine on badly
scaled operands."""
import ctypes
import math
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2010_00465_b200 as csm
from paper_2010_00465_b200 import _lib, distchain
from oracle import cossin_oracle as orc
from tests.test_gpu_guard import _cases


def P_of(K, nm=16):
    mods = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193][:nm]
    return int(math.floor((sum(math.log2(m) for m in mods) - 2 - math.log2(K)) / 2))


def bound(L, R):
    n = L.shape[1]
    P = P_of(n)
    rm, cm = np.abs(L).max(1), np.abs(R).max(0)
    d = np.where(rm > 0, np.ldexp(1.0, np.frexp(rm)[1] - P - 1), 0.0)
    f = np.where(cm > 0, np.ldexp(1.0, np.frexp(cm)[1] - P - 1), 0.0)
    return (d.sum() * np.abs(R).sum(0) + f * (np.abs(L).sum() + n * d.sum())).max()


def product(L, R, eng):
    n = L.shape[0]
    steps, _, _ = distchain.chain_program(3, fold=False)
    op = steps[0][0]  # slot 1 = slot0 @ slot0 (no scaling)
    dev = torch.device("cuda")
    Lt = torch.from_numpy(L).to(dev)
    Rt = torch.from_numpy(R).to(dev)
    slab = torch.zeros((9, n, n), dtype=torch.float64, device=dev)
    co = torch.empty((n, n), dtype=torch.float64, device=dev)
    so = torch.empty_like(co)
    with csm.engine_scope(eng):
        scratch = torch.empty(distchain._slab_scratch_size(n, n), dtype=torch.uint8, device=dev)
        distchain._device_slab_op(op, slab, n, n, 0, Rt, Lt, 0, -1, co, so, scratch, None)
    torch.cuda.synchronize()
    return slab[1].cpu().numpy()


def ext_ref(L, R):
    Ll, Rl = L.astype(np.longdouble), R.astype(np.longdouble)
    return Ll @ Rl


n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
names, a = _cases(n)
for nm in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["graded1e+08@1000"]):
    x = a[names.index(nm)]
    k, s = orc.select(orc.norm1(x))
    X = x * 2.0 ** -s
    pairs = [("X X", X, X)]
    y = X @ X
    pairs.append(("y y", y, y))
    for lab, L, R in pairs:
        ref = ext_ref(L, R)
        cn = float(np.abs(ref).sum(0).max())
        E = bound(L, R)
        line = f"{nm} {lab}: ||C|| {cn:.3e} E/||C|| {E / cn:.3e} n u {n * 2.0**-53:.3e}"
        for eng in ("dmma", "ozaki-unguarded", "ozaki"):
            c = product(L, R, eng)
            err = float(np.abs(c.astype(np.longdouble) - ref).sum(0).max()) / cn
            line += f" | {eng} {err:.3e}"
        print(line, flush=True)
