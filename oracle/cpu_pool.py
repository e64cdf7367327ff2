"""CPU baseline runner -- TEST/BENCH INFRASTRUCTURE ONLY.

Times the oracle (the numpy restatement of the reference's cos_sin /
wave_cos_sin, oracle/cossin_oracle.py) on the host cores: a process pool
of P workers, one BLAS thread each (the fair throughput configuration for
small matrices, where Python overhead dominates).  Used only
by bench.py's cpu_baseline leg and its --impl reference arm.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time


def _gen(kind: str, seed: int, count: int, n: int):
    import numpy as np
    rng = np.random.default_rng(seed)
    if kind == "cfg2":
        g = rng.standard_normal((count, n, n))
        tgt = 10.0 ** rng.uniform(-3.0, 2.0, count)
        nrm = np.abs(g).sum(axis=1).max(axis=1)
        return g * (tgt / nrm)[:, None, None], None
    if kind == "cfg3":
        g = rng.uniform(-1.0, 1.0, (count, n, n))
        tgt = 10.0 ** rng.uniform(-2.0, np.log10(50.0), count)
        nrm = np.abs(g).sum(axis=1).max(axis=1)
        return (g * (tgt / nrm)[:, None, None]).astype(np.float32), None
    if kind == "cfg4":
        lap = (np.diag(2.0 * np.ones(n)) - np.diag(np.ones(n - 1), 1)
               - np.diag(np.ones(n - 1), -1)) * float((n + 1) ** 2)
        v = rng.uniform(0.0, 10.0, (count, n))
        a = lap[None] + v[:, :, None] * np.eye(n)[None]
        return a, 10.0 ** rng.uniform(-4.0, -1.0, count)
    raise ValueError(kind)


def _work(args):
    kind, seed, count, n, min_seconds = args
    from oracle import cossin_oracle as orc
    a, t = _gen(kind, seed, count, n)
    done = 0
    t0 = time.perf_counter()
    while True:
        for i in range(count):
            if kind == "cfg4":
                orc.wave_cos_sin(a[i], float(t[i]), "double")
            elif kind == "cfg3":
                orc.cos_sin(a[i].astype("float64"), "single")
            else:
                orc.cos_sin(a[i], "double")
            done += 1
        el = time.perf_counter() - t0
        if el >= min_seconds:
            return done, el


def run_pool(kind: str, n: int, per_worker: int, workers: int | None = None,
             min_seconds: float = 10.0, seed: int = 1000):
    """Returns (matrices_per_second, workers, matrices_done, seconds)."""
    workers = workers or os.cpu_count() or 1
    old = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS",
                                          "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in old:
        os.environ[k] = "1"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    old_pp = os.environ.get("PYTHONPATH")
    os.environ["PYTHONPATH"] = root + (os.pathsep + old_pp if old_pp else "")
    try:
        ctx = mp.get_context("spawn")
        with ctx.Pool(workers) as pool:
            res = pool.map(_work, [(kind, seed + w, per_worker, n, min_seconds)
                                   for w in range(workers)])
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        if old_pp is None:
            os.environ.pop("PYTHONPATH", None)
        else:
            os.environ["PYTHONPATH"] = old_pp
    done = sum(r[0] for r in res)
    secs = max(r[1] for r in res)
    rate = sum(r[0] / r[1] for r in res)  # workers run concurrently
    return rate, workers, done, secs
