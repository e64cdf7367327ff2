"""Taylor vs Pade-8 head-to-head on the GPU: matrices/s and
product-equivalents for the same seeded batch.  python tools/bench_pade.py"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2010_00465_b200 as csm
from tests._util import cfg2_like


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


rows = []
for n, B in ((64, 16384), (128, 4096), (256, 1024), (512, 128)):
    a = torch.from_numpy(cfg2_like(np.random.default_rng(7), B, n=n)).cuda()
    t = csm.cos_sin_batched(a, raise_on_error=False)
    p = csm.pade_cos_sin_batched(a, raise_on_error=False)
    torch.cuda.synchronize()
    tk = (t.k + 2 * t.s).double().mean().item()
    pk = (5 + 7 / 3 + 2 * p.s.double()).mean().item()
    ms_t = timed(lambda: csm.cos_sin_batched(a, raise_on_error=False))
    ms_p = timed(lambda: csm.pade_cos_sin_batched(a, raise_on_error=False))
    row = {"n": n, "batch": B, "taylor_mat_s": B / ms_t * 1e3, "pade_mat_s": B / ms_p * 1e3,
           "taylor_mean_cost": tk, "pade_mean_cost": pk, "speedup_taylor_over_pade": ms_p / ms_t}
    rows.append(row)
    print(json.dumps(row), flush=True)
