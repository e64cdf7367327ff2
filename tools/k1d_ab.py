"""A/B timing of K1d vs K1 on cfg2 (run with CSM_K1D=0 / 1): CUDA-event time of
cos_sin_batched on a resident batch, matrices/s and TFLOP/s."""
import os, sys, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2010_00465_b200 as csm
from paper_2010_00465_b200 import _lib
from tests._util import cfg2_like
B = int(os.environ.get("AB_B", "16384")); N = int(os.environ.get("AB_N", "64"))
WAVE = os.environ.get("AB_WAVE", "0") == "1"
if WAVE:  # the wave family on Laplacian-like inputs (cfg4's distribution at order N)
    from tests._util import laplacian_wave
    a_np, t_np = laplacian_wave(np.random.default_rng(0), B, N)
    a = torch.from_numpy(a_np).cuda(); t = torch.from_numpy(t_np).cuda()
    run = lambda: csm.wave_cos_sin_batched(a, t)
else:
    a = torch.from_numpy(cfg2_like(np.random.default_rng(0), B, n=N)).cuda()
    run = lambda: csm.cos_sin_batched(a)
r = run(); torch.cuda.synchronize()
prod = float((r.k + 2 * r.s).sum().item())
L = _lib.lib()
L.csm_profile_enable(1)
for _ in range(3): run()
torch.cuda.synchronize()
tot = ctypes.c_double(); cnt = ctypes.c_int64()
L.csm_profile_collect(ctypes.byref(tot), ctypes.byref(cnt))
reps = 10
for _ in range(reps): run()
torch.cuda.synchronize()
L.csm_profile_collect(ctypes.byref(tot), ctypes.byref(cnt))
ms = tot.value / max(cnt.value, 1)
peak = ctypes.c_double()
print(f"{'wave ' if WAVE else ''}CSM_K1D={os.environ.get('CSM_K1D','1')} n={N} B={B} kernel {ms:.4f} ms  {B/ms*1e3/1e6:.3f} M mat/s  {2*N**3*prod/ms*1e3/1e12:.2f} TFLOP/s (intervals {cnt.value})")
