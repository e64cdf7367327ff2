"""GPU timeline of one batched call (torch.profiler, CUDA activity): kernel
time by name and the idle gaps between kernels.  python tools/timeline.py cfg"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from collections import defaultdict
import numpy as np
import torch
import paper_2010_00465_b200 as csm
from tests._util import cfg2_like, cfg3_like

which = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
method = sys.argv[2] if len(sys.argv) > 2 else "taylor"
rng = np.random.default_rng(0)
if which == "cfg3":
    a = torch.from_numpy(cfg3_like(rng, 4096)).cuda(); prec = csm.Precision.SINGLE
elif which == "cfg2":
    a = torch.from_numpy(cfg2_like(rng, 16384)).cuda(); prec = csm.Precision.DOUBLE
else:
    n = int(which); a = torch.from_numpy(cfg2_like(rng, max(1, 2 ** 21 // n ** 2 * 8), n=n)).cuda(); prec = csm.Precision.DOUBLE
run = csm.cos_sin_batched if method == "taylor" else csm.pade_cos_sin_batched
for _ in range(2):
    run(a, prec, raise_on_error=False)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    run(a, prec, raise_on_error=False)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    agg[e.name[:60]][0] += 1
    agg[e.name[:60]][1] += (e.time_range.end - e.time_range.start) / 1e3
t0, t1 = ev[0].time_range.start, ev[-1].time_range.end
busy = sum(v[1] for v in agg.values())
gaps = []
for x, y in zip(ev, ev[1:]):
    g = (y.time_range.start - x.time_range.end) / 1e3
    if g > 0.02:
        gaps.append((round(g, 3), x.name[:30], y.name[:30]))
print(f"{which}: span {(t1 - t0) / 1e3:.3f} ms, kernels {busy:.3f} ms")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
    print(f"  {v[1]:8.3f} ms {v[0]:5d}x  {k}")
print("  largest gaps (ms):", sorted(gaps, reverse=True)[:8])
