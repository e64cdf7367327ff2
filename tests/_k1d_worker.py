"""Worker of tests/test_gpu_k1d.py: runs the seeded K1d cases in this process
(whose CSM_K1D the parent sets: 1 = K1d, 0 = K1) and saves outputs to an npz,
so that the parent can compare the two kernels bit for bit."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def cases():
    """name -> (batch array, raise_on_error).  Batches > 148 so the call takes
    the scheduled path (K0 + K1 / K1d), not the self-selecting K1."""
    from tests._util import cfg2_like
    rng = np.random.default_rng(20250)
    out = {}
    out["cfg2_like_64"] = cfg2_like(rng, 1500, n=64)            # every k, s = 0..6
    out["deep_64"] = cfg2_like(rng, 400, n=64, lo=2.0, hi=3.3)  # s up to ~10
    out["tiny_64"] = cfg2_like(rng, 300, n=64, lo=-9.0, hi=-3.0)  # k = 3, s = 0
    out["n37"] = cfg2_like(rng, 700, n=37)
    out["n5"] = cfg2_like(rng, 900, n=5)
    out["n63"] = cfg2_like(rng, 333, n=63)
    out["f32_64"] = cfg2_like(rng, 600, n=64).astype(np.float32)
    out["f32_20"] = cfg2_like(rng, 600, n=20).astype(np.float32)
    bad = cfg2_like(rng, 500, n=64)
    bad[7, 3, 4] = np.nan
    bad[123, 0, 0] = np.inf
    bad[499, 63, 63] = np.nan
    out["nonfinite_64"] = bad
    return out


def main(path):
    import paper_2010_00465_b200 as csm
    res = {}
    for name, a in cases().items():
        r = csm.cos_sin_batched(a, raise_on_error=False)
        res[name + "/c"] = np.asarray(r.cos_part)
        res[name + "/s"] = np.asarray(r.sin_part)
        res[name + "/k"] = np.asarray(r.k)
        res[name + "/sx"] = np.asarray(r.s)
        res[name + "/st"] = np.asarray(r.status)
    np.savez(path, **res)


if __name__ == "__main__":
    main(sys.argv[1])
