"""Small cases for compute-sanitizer runs (one tool per gpurun call, per
/opt/skills/guides/B200_PROFILING.md): K1 (n <= 64, persistent, bulk-copy
prefetch), K1c (4-CTA cluster, DSMEM + cluster barriers), the tiled chain
(n > 128, DMMA) and the Ozaki-II int8 tcgen05 product (n = 768).
usage: python tools/sanitize_cases.py k1 k1c tiled ozaki"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2010_00465_b200 as csm  # noqa: E402
from tests._util import cfg2_like  # noqa: E402

rng = np.random.default_rng(0)
cases = sys.argv[1:] or ["k1", "k1c", "tiled", "ozaki"]
for c in cases:
    if c == "k1":  # more matrices than SMs: every CTA prefetches a next matrix
        rep = csm.cos_sin_batched(cfg2_like(rng, 300, n=64))
        w = csm.wave_cos_sin_batched(cfg2_like(rng, 200, n=40, hi=0.5), 0.3)
    elif c == "k1c":
        rep = csm.cos_sin_batched(cfg2_like(rng, 80, n=128))
        w = csm.wave_cos_sin_batched(cfg2_like(rng, 40, n=96, hi=0.5), 0.3)
    elif c == "tiled":
        rep = csm.cos_sin_batched(cfg2_like(rng, 6, n=160))
        p = csm.pade_cos_sin_batched(cfg2_like(rng, 3, n=200))
    elif c == "ozaki":
        g = rng.standard_normal((768, 768))
        with csm.engine_scope("ozaki"):
            r = csm.cos_sin(g * (2.0 / np.abs(g).sum(axis=0).max()))
    else:
        raise SystemExit(f"unknown case {c}")
    print(c, "ok", flush=True)
