"""Scratch A/B of the Ozaki int8 GEMM tile walk (CSM_OZ_GX) at one n: python tools/oz_gx_probe.py N BATCH."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2010_00465_b200 as csm
from tests._util import cfg2_like
n, B = int(sys.argv[1]), int(sys.argv[2])
a = torch.from_numpy(cfg2_like(np.random.default_rng(0), B, n=n, lo=0.5, hi=1.5)).cuda()
csm.set_engine("ozaki")
csm.cos_sin_batched(a); torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); csm.cos_sin_batched(a, raise_on_error=False); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"n={n} B={B} gx={os.environ.get('CSM_OZ_GX','default')}: {min(ts):.2f} ms", flush=True)
