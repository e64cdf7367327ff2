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
    # the scaling epilogues' multiply paths and the 2**-s fallbacks: products
    # that underflow to subnormals / zero (tiny norms), s in the hundreds and
    # beyond 1022 (huge norms: intermediate overflow to inf / NaN, as the
    # reference's own arithmetic gives), and batches mixing both
    tiny = cfg2_like(rng, 200, n=64, lo=-200.0, hi=-150.0)
    huge = cfg2_like(rng, 200, n=64, lo=100.0, hi=307.0)
    out["subnormal_64"] = tiny
    out["huge_64"] = huge
    mixed = np.concatenate([tiny[:60], huge[:60], cfg2_like(rng, 80, n=64)])
    out["mixed_extreme_64"] = mixed[rng.permutation(mixed.shape[0])]
    out["huge_n30"] = cfg2_like(rng, 160, n=30, lo=200.0, hi=300.0)
    # batch sizes around the persistent grid (296 CTAs, two per SM)
    for count in (149, 295, 296, 297, 593):
        out[f"edge_{count}"] = cfg2_like(rng, count, n=64)
    bad = cfg2_like(rng, 500, n=64)
    bad[7, 3, 4] = np.nan
    bad[123, 0, 0] = np.inf
    bad[499, 63, 63] = np.nan
    out["nonfinite_64"] = bad
    return out


def wave_cases():
    """name -> (batch, t): the wave family (driver.py:126-146) on K1d."""
    from tests._util import cfg2_like, laplacian_wave
    rng = np.random.default_rng(20251)
    out = {}
    out["wave_lap_64"] = laplacian_wave(rng, 900, 64)        # every k, s = 0..6
    out["wave_lap_48"] = laplacian_wave(rng, 500, 48)
    a = cfg2_like(rng, 700, n=64, lo=-2.0, hi=3.0)
    out["wave_gauss_64"] = (a, 10.0 ** rng.uniform(-2.0, 0.5, 700))
    a = cfg2_like(rng, 400, n=21, lo=-1.0, hi=2.0)
    out["wave_gauss_21"] = (a, 10.0 ** rng.uniform(-3.0, 1.0, 400))
    a32, t32 = laplacian_wave(rng, 300, 64)
    out["wave_f32_64"] = (a32.astype(np.float32), t32)
    bad, tb = laplacian_wave(rng, 200, 64)
    bad[3, 5, 5] = np.nan
    bad[199, 0, 63] = np.inf
    out["wave_nonfinite_64"] = (bad, tb)
    return out


def main(path):
    import paper_2010_00465_b200 as csm
    res = {}
    for name, (a, t) in wave_cases().items():
        r = csm.wave_cos_sin_batched(a, t, raise_on_error=False)
        res[name + "/c"] = np.asarray(r.cos_part)
        res[name + "/s"] = np.asarray(r.sin_part)
        res[name + "/k"] = np.asarray(r.k)
        res[name + "/sx"] = np.asarray(r.s)
        res[name + "/st"] = np.asarray(r.status)
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
