"""Whole chain on one badly scaled matrix: batched API vs block-row (slab)
path at world 1, per engine, against the oracle."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2010_00465_b200 as csm
from paper_2010_00465_b200 import distchain
from oracle import cossin_oracle as orc
from tests._util import rel1
from tests.test_gpu_guard import _cases

n = int(sys.argv[1])
names, a = _cases(n)
for nm in sys.argv[2].split(","):
    x = a[names.index(nm)]
    c, s, k, sc = orc.cos_sin(x)
    line = f"{nm} k={k} s={sc}"
    for eng in ("dmma", "ozaki-unguarded", "auto"):
        with csm.engine_scope(eng):
            r = csm.cos_sin_batched(x[None])
            cb = r.cos_part[0]
            cd, sd, st = distchain.cos_sin_distributed(torch.from_numpy(x).cuda())
        line += f" | {eng}: batched {rel1(cb, c):.2e} slab {rel1(cd.cpu().numpy(), c):.2e}"
    print(line, flush=True)
