"""Time the GPU double-double reference path (csrc/ddref.cu).

Reports per-product time of csm_dd_matmul at several n, the FP64 pipe
rate it implies (33 DADD/DMUL per k step and output element, each counted
as one FP64 instruction -- an FMA-counted peak of P TFLOP/s issues P/2 T
instr/s), and one reference_cos_sin call.  Usage:
    python tools/ddref_bench.py [n ...]
"""
import ctypes
import json
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2010_00465_b200 import _lib, verify as V  # noqa: E402

OPS_PER_STEP = 33


def main():
    ns = [int(v) for v in sys.argv[1:]] or [256, 1024, 2048, 4096]
    L = _lib.lib()
    peak = ctypes.c_double()
    _lib.check(L.csm_fp64_peak(20000, ctypes.byref(peak), None), "peak")
    out = {"fp64_peak_tflops": peak.value, "rows": []}
    for n in ns:
        B = max(1, (2048 // n) ** 3 // 8) if n < 2048 else 1
        x = torch.randn(B, n, n, dtype=torch.float64, device="cuda")
        y = torch.randn_like(x)
        xl = x * 1e-17
        yl = y * 1e-17
        V.dd_matmul(x, xl, y, yl)
        torch.cuda.synchronize()
        reps = 3
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            V.dd_matmul(x, xl, y, yl)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        instr = OPS_PER_STEP * float(n) ** 3 * B
        rate = instr / (ms * 1e-3) / 1e12
        row = {"n": n, "batch": B, "ms_per_call": ms, "ms_per_product": ms / B,
               "fp64_instr_T_per_s": rate,
               "frac_of_fp64_issue_peak": rate / (peak.value / 2)}
        if n <= 2048:
            a = torch.randn(n, n, dtype=torch.float64, device="cuda")
            a *= 4.0 / a.abs().sum(0).max()
            torch.cuda.synchronize()
            t = time.perf_counter()
            V.reference_cos_sin(a)
            torch.cuda.synchronize()
            row["reference_cos_sin_s"] = time.perf_counter() - t
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
