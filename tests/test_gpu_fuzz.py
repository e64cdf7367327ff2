"""Seeded fuzz over every dispatch path: random n (1..300), batch sizes,
families, dtypes and norm ranges through the batched API, each matrix
checked against the oracle ((k, s) bit-exact, 1e-12 / 1e-5 outputs)."""
import numpy as np
import pytest

import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc
from tests._util import pair_close

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(600)
def test_fuzz_dispatch_paths(cuda):
    rng = np.random.default_rng(20260101)
    cases = 0
    for trial in range(80):
        n = int(rng.choice([1, 2, 5, 31, 63, 64, 65, 97, 127, 128, 129, 191, 256, 300]))
        batch = int(rng.integers(1, 7 if n > 128 else 40))
        wave = bool(rng.integers(0, 2))
        f32 = bool(rng.integers(0, 4) == 0)
        lo, hi = sorted(rng.uniform(-4, 2.3, 2))
        g = rng.standard_normal((batch, n, n))
        if wave:
            g = g @ np.swapaxes(g, 1, 2) / n + 0.1 * np.eye(n)
        nrm = np.abs(g).sum(axis=1).max(axis=1)
        a = g * (10.0 ** rng.uniform(lo, hi, batch) / nrm)[:, None, None]
        prec = "single" if f32 else "double"
        if f32:
            a = a.astype(np.float32)
        t = 10.0 ** rng.uniform(-1.0, 0.3, batch)
        if wave:
            rep = csm.wave_cos_sin_batched(a, t, csm.Precision(prec))
        else:
            rep = csm.cos_sin_batched(a, csm.Precision(prec))
        tol = 1e-5 if f32 else 1e-12
        for i in range(batch):
            ai = a[i].astype(np.float64) if f32 else a[i]
            if wave:
                c, s, k, sc = orc.wave_cos_sin(ai, t[i], prec)
            else:
                c, s, k, sc = orc.cos_sin(ai, prec)
            assert (int(rep.k[i]), int(rep.s[i])) == (k, sc), (trial, n, i)
            assert pair_close(rep.cos_part[i], c, s, tol)[0], (trial, n, wave, f32, i)
            if orc.norm1(s) > 0:
                assert pair_close(rep.sin_part[i], s, c, tol)[0], (trial, n, wave, f32, i)
            cases += 1
    assert cases > 400
