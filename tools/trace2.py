"""Two-thread trace (group 0 leader and group 1 leader) of fused64, CTA 0.
Prints a merged timeline excerpt and per-group phase stats."""
import ctypes, os, subprocess, sys
from collections import defaultdict
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
libs = {tid: os.path.join(ROOT, "tools", f"libcossin_trace_t{tid}.so") for tid in (0, 256)}
if "--build" in sys.argv:
    for tid, so in libs.items():
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "-Xcompiler", "-fPIC", "-shared", "-DCSM_TRACE", f"-DCSM_TRACE_TID={tid}", "-o", so,
                               os.path.join(ROOT, "paper_2010_00465_b200/csrc/cossin_b200.cu")])
    sys.exit(0)
tid = int(sys.argv[1])
os.environ["CSM_LIB_PATH"] = libs[tid]
import numpy as np, torch
from paper_2010_00465_b200 import _lib
import paper_2010_00465_b200 as csm
from tests._util import cfg2_like
L = _lib.lib(); L.csm_trace_dump.restype = ctypes.c_int
a = torch.from_numpy(cfg2_like(np.random.default_rng(0), 16384)).cuda()
csm.cos_sin_batched(a); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 65536)(); L.csm_trace_dump(buf, 65536)
csm.cos_sin_batched(a); torch.cuda.synchronize()
n = L.csm_trace_dump(buf, 65536)
np.save(os.path.join(ROOT, "gpurun_out", f"trace_t{tid}.npy"), np.array([buf[i] for i in range(n)], dtype=np.uint64))
print("saved", n)
