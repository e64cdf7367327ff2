"""Oracle side of tests/test_gpu_fullsize.py's cfg4 check, in a module that
imports only numpy and the oracle, so the spawned pool workers start light
(no torch, no CUDA library)."""
import numpy as np


def cfg4_parts(count=512, n=512):
    """oracle.cpu_pool._gen('cfg4', 0, count, n) without materialising the
    whole batch: a[i] = lap + diag(v[i]) (same draws, same order)."""
    rng = np.random.default_rng(0)
    lap = (np.diag(2.0 * np.ones(n)) - np.diag(np.ones(n - 1), 1)
           - np.diag(np.ones(n - 1), -1)) * float((n + 1) ** 2)
    v = rng.uniform(0.0, 10.0, (count, n))
    return lap, v, 10.0 ** rng.uniform(-4.0, -1.0, count)


def cfg4_worker(args):
    """Oracle side of one chunk of cfg4: per matrix (k, s, gpu-vs-oracle
    errors, the oracle's permuted-order noise, and both distances to the
    eigendecomposition answer)."""
    lo, hi, c_path, s_path, seed = args
    import numpy as np

    from oracle import cossin_oracle as orc
    from tests._util import permuted_noise, rel1
    lap, v_all, t_all = cfg4_parts()
    cg = np.load(c_path, mmap_mode="r")
    sg = np.load(s_path, mmap_mode="r")
    rng = np.random.default_rng(seed)
    out = []
    for i in range(lo, hi):
        a, t = lap + np.diag(v_all[i]), float(t_all[i])
        (c, s, k, sc), noise = permuted_noise(lambda x: orc.wave_cos_sin(x, t), a, rng)
        lam, v = np.linalg.eigh(a)
        w = np.sqrt(lam)
        ce = (v * np.cos(t * w)) @ v.T
        se = (v * (np.sin(t * w) / w)) @ v.T
        out.append((i, k, sc, rel1(cg[i], c), rel1(sg[i], s), noise,
                    rel1(cg[i], ce), rel1(c, ce), rel1(sg[i], se), rel1(s, se)))
    return out
