"""Diagnose self-selecting vs K0 path differences at n < 64 (test inputs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_00465_b200 as csm
from tests._util import cfg2_like
for n in (37, 1):
    rng = np.random.default_rng(700 + n)
    big = cfg2_like(rng, 160, n=n)
    big[3, 0, 0] = np.nan
    big[5] *= 1e306
    idx = [0, 1, 2, 3, 4, 5, 77, 159]
    for a in (big, big.astype(np.float32)):
        prec = csm.Precision.DOUBLE if a.dtype == np.float64 else csm.Precision.SINGLE
        full = csm.cos_sin_batched(torch.from_numpy(a).cuda(), prec, raise_on_error=False)
        sub = csm.cos_sin_batched(torch.from_numpy(a[idx]).cuda(), prec, raise_on_error=False)
        for j, i in enumerate(idx):
            fc = full.cos_part[i].cpu().numpy(); sc = sub.cos_part[j].cpu().numpy()
            print(n, a.dtype, i, int(full.status[i]), int(sub.status[j]), int(full.k[i]), int(sub.k[j]),
                  int(full.s[i]), int(sub.s[j]), 'equal', np.array_equal(fc, sc),
                  'nan full/sub', int(np.isnan(fc).sum()), int(np.isnan(sc).sum()),
                  'maxdiff', float(np.nanmax(np.abs(fc - sc))) if fc.size else 0)
