"""Phase trace of fused64 (CTA 0): build a -DCSM_TRACE copy of the library,
run cfg2, print per-phase cycle statistics."""
import ctypes, os, subprocess, sys
from collections import defaultdict
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
so = os.path.join(ROOT, "tools", "libcossin_trace.so")
if os.environ.get("TRACE_SO"):
    so = os.path.join(ROOT, "tools", os.environ["TRACE_SO"])
if "--build" in sys.argv:
    extra = [a for a in sys.argv[1:] if a.startswith("-D")]
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           "-Xcompiler", "-fPIC", "-shared", "-DCSM_TRACE", *extra, "-o", so,
                           os.path.join(ROOT, "paper_2010_00465_b200/csrc/cossin_b200.cu")])
    sys.exit(0)
os.environ["CSM_LIB_PATH"] = so  # load the traced copy
import numpy as np, torch
from paper_2010_00465_b200 import _lib
import paper_2010_00465_b200 as csm
from tests._util import cfg2_like
L = _lib.lib(); L.csm_trace_dump.restype = ctypes.c_int
N = int(os.environ.get("TRACE_N", "64")); B = int(os.environ.get("TRACE_B", "16384"))
a = torch.from_numpy(cfg2_like(np.random.default_rng(0), B, n=N)).cuda()
csm.cos_sin_batched(a); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 65536)(); L.csm_trace_dump(buf, 65536)
csm.cos_sin_batched(a); torch.cuda.synchronize()
n = L.csm_trace_dump(buf, 65536)
ev = [(int(buf[i]) & 255, int(buf[i]) >> 8) for i in range(n)]
# phases
stats = defaultdict(list); last = None; mats = 0; ks = defaultdict(int)
for tag, v in ev:
    if tag == 9:
        ks[(v >> 4, v & 15)] += 1; mats += 1; continue
    if last is not None:
        stats[(last[0], tag)].append(v - last[1])
    last = (tag, v)
t0 = ev[0][1]; t1 = ev[-1][1]
print(f"events={n} matrices={mats} cycles={t1-t0} per-matrix={(t1-t0)/max(mats,1):.0f}")
for key in sorted(stats, key=lambda k: -sum(stats[k])):
    v = stats[key]
    print(f"{key[0]}->{key[1]}: n={len(v):5d} mean={np.mean(v):8.1f} total={sum(v)/(t1-t0)*100:5.1f}%")
print(sorted(ks.items()))
# per-epilogue-type breakdown: step index within chain -> (k, step)
cur_k = None; step = 0; per = defaultdict(list); t2 = t3 = None
for tag, v in ev:
    if tag == 9:
        cur_k = (v >> 4, v & 15); step = 0; continue
    if tag == 2: t2 = v
    if tag == 3: t3 = v
    if tag == 4 and t2 is not None and t3 is not None:
        per[(cur_k[0], step)].append((t3 - t2, v - t3)); step += 1
for key in sorted(per):
    a = np.array(per[key])
    print(f"k={key[0]} step={key[1]}: n={len(a):4d} issue={a[:,0].mean():7.0f} drain+epi={a[:,1].mean():7.0f}")
