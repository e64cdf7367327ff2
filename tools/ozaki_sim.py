"""Numerics check for an Ozaki-style fp64 GEMM from int8 slices (row / column
power-of-two scaling, S signed 7-bit slices, levels i+j <= S+1 summed exactly
in integers): error against an extended-precision product vs plain fp64."""
import numpy as np
def split(M, S, axis):
    # per-row (axis=1) or per-column (axis=0) power-of-2 scaling, S signed slices of 7 bits
    amax = np.abs(M).max(axis=axis, keepdims=True)
    e = np.ceil(np.log2(np.where(amax > 0, amax, 1.0)))
    R = M / 2.0**e   # |R| <= 1
    sl = []
    for j in range(S):
        R = R * 128.0
        q = np.trunc(R)  # in [-127, 127]... use round-to-nearest-ish trunc
        sl.append(q.astype(np.int64))
        R = R - q
    return sl, e
def ozaki(A, B, S):
    As, ea = split(A, S, 1)
    Bs, eb = split(B, S, 0)
    n = A.shape[0]
    C = np.zeros((n, n))
    for lvl in range(2, S + 2):   # level = i + j (1-based)
        acc = np.zeros((n, n), dtype=np.int64)
        for i in range(1, lvl):
            j = lvl - i
            if j > S: continue
            acc += As[i-1] @ Bs[j-1]
        C += acc.astype(np.float64) * 2.0**(-7 * lvl)
    return C * 2.0**ea * 2.0**eb
rng = np.random.default_rng(0)
n = 64
from numpy.linalg import norm
for trial, scale in ((0, 1.0), (1, 1e3)):
    A = rng.standard_normal((n, n)) * (10.0 ** rng.uniform(-3, 3, (n, n)) if trial else 1.0)
    B = rng.standard_normal((n, n))
    exact = (A.astype(np.longdouble) @ B.astype(np.longdouble))
    ref = A @ B
    for S in (6, 7, 8, 9):
        C = ozaki(A, B, S)
        e_oz = float(np.abs(C - exact).max() / np.abs(exact).max())
        e_ref = float(np.abs(ref - exact).max() / np.abs(exact).max())
        print(trial, S, "ozaki err %.2e  fp64 err %.2e  gemms %d" % (e_oz, e_ref, S*(S+1)//2))
