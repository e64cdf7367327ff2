"""Build tools/libcossin_debug.so: the library with the device-side bounds
checks of CSM_DCHECK enabled (-DCSM_DEBUG_CHECKS).  compute-sanitizer is
closed on this pool; the GPU suite is run against this build instead:
    CSM_LIB_PATH=tools/libcossin_debug.so python -m pytest tests -m gpu"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(ROOT, "tools", "libcossin_debug.so")
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
       "-Xcompiler", "-fPIC", "-shared", "-DCSM_DEBUG_CHECKS", "-o", out,
       os.path.join(ROOT, "paper_2010_00465_b200", "csrc", "cossin_b200.cu")]
sys.exit(subprocess.call(cmd))
