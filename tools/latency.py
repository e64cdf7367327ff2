"""Small-batch latency: one cos_sin_batched call vs BatchPlan.run vs a CUDA
graph replay (python tools/latency.py)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2010_00465_b200 as csm
from paper_2010_00465_b200.plan import BatchPlan
from tests._util import cfg2_like

for n, B in ((64, 1), (64, 16), (128, 4)):
    a = torch.from_numpy(cfg2_like(np.random.default_rng(0), B, n=n)).cuda()
    plan = BatchPlan(B, n)
    plan.capture(a)

    def per_call(fn, reps=200):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / reps * 1e6

    u_api = per_call(lambda: csm.cos_sin_batched(a, raise_on_error=False))
    u_run = per_call(lambda: plan.run(a))
    u_graph = per_call(plan.replay)
    print(f"n={n} batch={B}: api {u_api:.1f} us, plan.run {u_run:.1f} us, graph replay {u_graph:.1f} us")
