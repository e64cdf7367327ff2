"""Scratch check of the Ozaki engine against the DMMA engine and the oracle:
python tools/oz_check.py [n ...].  For each n: a small cfg2-like batch
(parity: relative 1-norm vs the oracle, both engines), then a timing batch
(~1 GiB of input) through each engine."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc
from tests._util import cfg2_like, rel1

ns = [int(x) for x in sys.argv[1:]] or [256, 512, 1024]
for n in ns:
    a = cfg2_like(np.random.default_rng(1), 6, n=n)
    ref = [orc.cos_sin(a[i]) for i in range(a.shape[0])]
    for eng in ("dmma", "ozaki"):
        csm.set_engine(eng)
        rep = csm.cos_sin_batched(torch.from_numpy(a).cuda())
        torch.cuda.synchronize()
        worst = 0.0
        for i in range(a.shape[0]):
            c, s, k, sc = ref[i]
            assert (int(rep.k[i]), int(rep.s[i])) == (k, sc)
            cg = rep.cos_part[i].cpu().numpy()
            sg = rep.sin_part[i].cpu().numpy()
            worst = max(worst, rel1(cg, c), rel1(sg, s))
        print(f"n={n} {eng}: worst rel 1-norm vs oracle {worst:.2e}", flush=True)
    B = max(8, (1 << 30) // (n * n * 8))
    a = torch.from_numpy(cfg2_like(np.random.default_rng(0), B, n=n)).cuda()
    for eng in ("dmma", "ozaki"):
        csm.set_engine(eng)
        rep = csm.cos_sin_batched(a)
        torch.cuda.synchronize()
        k = rep.k.cpu().numpy().astype(np.int64)
        s = rep.s.cpu().numpy().astype(np.int64)
        flops = float((2.0 * n ** 3 * (k + 2 * s)).sum())
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            csm.cos_sin_batched(a, raise_on_error=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = min(ts)
        print(f"n={n} B={B} {eng}: {ms:.2f} ms  {B / ms * 1e3:.0f} mat/s  "
              f"{flops / ms / 1e9:.1f} TFLOP/s fp64-equiv  ({flops / ms / 1e9 / 36.95:.2f} x DMMA peak)",
              flush=True)
    del a
    torch.cuda.empty_cache()
csm.set_engine("dmma")
