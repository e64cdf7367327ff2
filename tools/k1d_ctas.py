"""Per-CTA start/end times of K1d (trace build): load balance across the 296
CTAs and the pairing of CTAs on SMs.  Build: python tools/trace_fused.py --build"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CSM_LIB_PATH"] = os.path.join(ROOT, "tools", "libcossin_trace.so")
import numpy as np, torch
from paper_2010_00465_b200 import _lib
import paper_2010_00465_b200 as csm
from tests._util import cfg2_like
L = _lib.lib()
a = torch.from_numpy(cfg2_like(np.random.default_rng(0), 16384, n=64)).cuda()
for _ in range(3):
    r = csm.cos_sin_batched(a); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
L.csm_trace_k1d_ctas(buf)
t = np.array(buf[:], dtype=np.uint64).reshape(1024, 4)[:296].astype(np.int64)
t0 = t[:, 1].min()
start = (t[:, 1] - t0) / 1e3; end = (t[:, 2] - t0) / 1e3
print(f"CTAs 296: start max {start.max():.1f} us; end min {end.min():.1f} median {np.median(end):.1f} max {end.max():.1f} us")
sm = t[:, 0]
pairs = {}
for c in range(296): pairs.setdefault(int(sm[c]), []).append(c)
print("CTAs per SM:", sorted(set(len(v) for v in pairs.values())))
print("example pairs:", [pairs[k] for k in sorted(pairs)[:6]])
sm_end = np.array([max(end[c] for c in v) for v in pairs.values()])
print(f"per-SM end: min {sm_end.min():.1f} median {np.median(sm_end):.1f} max {sm_end.max():.1f}")
order = np.argsort(end)
print("earliest CTAs:", [(int(c), round(float(end[c]), 1)) for c in order[:6]])
print("latest CTAs:", [(int(c), round(float(end[c]), 1)) for c in order[-6:]])
cost = (r.k + 2 * r.s).cpu().numpy()
print("total products", cost.sum(), "per CTA mean", cost.sum() / 296)
