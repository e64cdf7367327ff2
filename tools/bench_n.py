"""Scratch timing of the batched fp64 path at one n (not the bench contract):
python tools/bench_n.py N [batch]."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2010_00465_b200 as csm
from tests._util import cfg2_like

n = int(sys.argv[1])
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
a = torch.from_numpy(cfg2_like(np.random.default_rng(0), B, n=n)).cuda()
rep = csm.cos_sin_batched(a)
torch.cuda.synchronize()
k = rep.k.cpu().numpy().astype(np.int64)
s = rep.s.cpu().numpy().astype(np.int64)
flops = float((2.0 * n ** 3 * (k + 2 * s)).sum())
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    csm.cos_sin_batched(a, raise_on_error=False)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
print(f"n={n} B={B} lib={os.environ.get('CSM_LIB_PATH', 'default')} fused_max="
      f"{os.environ.get('CSM_FUSED_MAX', '128')}: {ms:.3f} ms {B / ms * 1e3:.0f} mat/s "
      f"{flops / ms / 1e9:.2f} TFLOP/s frac={flops / ms / 1e9 / 36.95:.3f}", flush=True)
