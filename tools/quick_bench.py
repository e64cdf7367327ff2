"""Scratch timing of the batched path (not the bench contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_00465_b200 as csm
from tests._util import cfg2_like, cfg3_like

def run(name, a, prec, reps=5, n=64):
    ad = torch.from_numpy(a).cuda()
    rep = csm.cos_sin_batched(ad, prec)
    torch.cuda.synchronize()
    k = rep.k.cpu().numpy().astype(np.int64); s = rep.s.cpu().numpy().astype(np.int64)
    flops = float((2.0 * n**3 * (k + 2 * s)).sum())
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); csm.cos_sin_batched(ad, prec, raise_on_error=False); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"{name}: {ms:.3f} ms  {a.shape[0]/ms*1e3:.0f} mat/s  {flops/ms/1e9:.2f} TFLOP/s  mean k+2s={np.mean(k+2*s):.3f}", flush=True)

rng = np.random.default_rng(0)
run("cfg2 16384x64 f64", cfg2_like(rng, 16384), csm.Precision.DOUBLE)
run("cfg3-ish 512x256 f32", cfg3_like(rng, 512), csm.Precision.SINGLE, n=256)
run("256 f64 x512", cfg2_like(rng, 512, n=256), csm.Precision.DOUBLE, n=256)
