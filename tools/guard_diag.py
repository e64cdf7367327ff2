"""Diagnostic: errors of each product engine on the badly scaled guard cases
(tests/test_gpu_guard.py) against the oracle, its permuted-order noise and
the double-double truth (verify.reference_cos_sin)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc
from tests._util import rel1
from tests.test_gpu_guard import _cases

n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
names, a = _cases(n)
sel = [i for i, nm in enumerate(names) if only is None or any(o in nm for o in only)]
a = a[sel]
names = [names[i] for i in sel]
res = {}
for eng in ("auto", "dmma", "ozaki-unguarded"):
    with csm.engine_scope(eng):
        res[eng] = csm.cos_sin_batched(a)
truth = csm.verify.reference_cos_sin_batched(a) if hasattr(csm.verify, "reference_cos_sin_batched") else None
rng = np.random.default_rng(99)
for i, nm in enumerate(names):
    c, s, k, sc = orc.cos_sin(a[i])
    perm = rng.permutation(n)
    inv = np.argsort(perm)
    cp, sp, _, _ = orc.cos_sin(a[i][np.ix_(perm, perm)])
    noise = rel1(cp[np.ix_(inv, inv)], c)
    line = f"{nm:20s} k={k} s={sc} noise={noise:.2e}"
    if truth is not None:
        tc = truth[0][i]
        line += f" oracle-vs-truth={rel1(c, tc):.2e}"
    for eng, r in res.items():
        line += f" | {eng}: ora {rel1(r.cos_part[i], c):.2e}"
        if truth is not None:
            line += f" tru {rel1(r.cos_part[i], tc):.2e}"
    print(line, flush=True)
