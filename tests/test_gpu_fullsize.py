"""Parity at the full sizes of BASELINE configs[3] (cfg4: 512 wave pairs of
512 x 512) and configs[4] (cfg5: one 8192 x 8192 symmetric matrix), the
inputs bench.py times (bench.make_inputs, seed 0).

Gate: (k, s) bit-exact; each output within max(1e-12,
4 x the reference's own rounding noise on that input), the noise being the
oracle's distance to itself on P A P^T with P undone (every GEMM summed in
another order, tests/_util.permuted_noise).  At these sizes and scalings
(s up to 12) the reference's noise exceeds 1e-12, so a flat 1e-12 would
reject the reference against itself.  The third number compares both
against an independent truth: the eigendecomposition for the SPD wave
inputs, the double-double GPU oracle (verify.reference_cos_sin, bitwise
equal to the reference's own verify.py:480-521 on its goldens) for cfg5.
"""
import os

import numpy as np
import pytest

import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc
from tests._util import permuted_noise, rel1

pytestmark = pytest.mark.gpu

TOL64 = 1e-12


from tests._fullsize_worker import cfg4_parts as _cfg4_parts, cfg4_worker as _cfg4_worker  # noqa: E402


@pytest.mark.timeout(1500)
def test_full_cfg4_against_oracle(cuda, tmp_path):
    """All 512 x 512^2 wave pairs of configs[3] against the oracle (and the
    eigendecomposition), each at its own noise-floor gate."""
    import multiprocessing as mp

    from oracle.cpu_pool import _gen
    a, t = _gen("cfg4", 0, 512, 512)
    lap, v, t2 = _cfg4_parts()
    assert np.array_equal(t, t2) and np.array_equal(a[511], lap + np.diag(v[511]))
    rep = csm.wave_cos_sin_batched(a, t)
    del a
    c_path, s_path = str(tmp_path / "c.npy"), str(tmp_path / "s.npy")
    np.save(c_path, np.asarray(rep.cos_part))
    np.save(s_path, np.asarray(rep.sin_part))
    ks, ss = np.asarray(rep.k), np.asarray(rep.s)
    workers = min(16, os.cpu_count() or 1)
    bounds = np.linspace(0, 512, 4 * workers + 1).astype(int)
    jobs = [(int(lo), int(hi), c_path, s_path, 7 + j)
            for j, (lo, hi) in enumerate(zip(bounds[:-1], bounds[1:]))]
    # spawned workers inherit the environment at exec time: one BLAS thread
    # each (set before numpy loads in them), and the repo on their path
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    keys = ("PYTHONPATH", "OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")
    saved = {k: os.environ.get(k) for k in keys}
    os.environ["PYTHONPATH"] = root + (os.pathsep + saved["PYTHONPATH"]
                                       if saved["PYTHONPATH"] else "")
    for k in keys[1:]:
        os.environ[k] = "1"
    try:
        with mp.get_context("spawn").Pool(workers) as pool:
            rows = [r for part in pool.map(_cfg4_worker, jobs) for r in part]
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert len(rows) == 512
    worst = 0.0
    for (i, k, sc, ec, es, noise, gce, oce, gse, ose) in rows:
        assert (int(ks[i]), int(ss[i])) == (k, sc), i
        gate = max(TOL64, 4.0 * noise)
        assert ec <= gate and es <= gate, (i, sc, ec, es, noise)
        # third number: no further from the eigendecomposition than the
        # reference itself
        assert gce <= 4.0 * oce + 1e-14, (i, gce, oce)
        assert gse <= 4.0 * ose + 1e-14, (i, gse, ose)
        worst = max(worst, ec / gate, es / gate)
    assert int(ss.max()) >= 9  # the configs' t range reaches deep scaling
    print(f"cfg4: 512 matrices, s in [{int(ss.min())}, {int(ss.max())}], "
          f"worst error / gate {worst:.3f}")


@pytest.fixture(scope="module")
def cfg5_reference():
    """configs[4] input (bench.make_inputs('cfg5', seed 0)), the oracle's
    answer, its permuted-order noise and the double-double truth."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2010_00465_b200 import verify
    n = 8192
    g = np.random.default_rng(0).standard_normal((n, n))
    a = 20.0 * (g + g.T) / (2.0 * np.sqrt(n))
    del g
    (c, s, k, sc), noise = permuted_noise(orc.cos_sin, a, np.random.default_rng(8))
    truth = verify.reference_cos_sin(a)
    return dict(a=a, c=c, s=s, k=k, sc=sc, noise=noise,
                tc=np.asarray(truth.cos_part), ts=np.asarray(truth.sin_part))


def _check_cfg5(ref, got_c, got_s, k, sc):
    assert (k, sc) == (ref["k"], ref["sc"])
    gate = max(TOL64, 4.0 * ref["noise"])
    ec, es = rel1(got_c, ref["c"]), rel1(got_s, ref["s"])
    assert ec <= gate and es <= gate, (ec, es, ref["noise"])
    for got, orc_out, tr in ((got_c, ref["c"], ref["tc"]), (got_s, ref["s"], ref["ts"])):
        assert rel1(got, tr) <= 4.0 * rel1(orc_out, tr) + 1e-15, (rel1(got, tr),
                                                                  rel1(orc_out, tr))
    return ec, es


@pytest.mark.timeout(1500)
@pytest.mark.parametrize("engine", ["dmma", "auto"])
def test_full_cfg5_single_gpu(cuda, cfg5_reference, engine):
    """configs[4] at 8192^2 on one GPU through the drop-in cos_sin, on the
    default FP64 DMMA engine and on the guarded Ozaki-II engine."""
    ref = cfg5_reference
    with csm.engine_scope(engine):
        rep = csm.cos_sin(ref["a"])
    _check_cfg5(ref, rep.result.cos_part, rep.result.sin_part,
                rep.scheme_used.k_products, rep.scaling_exponent)


@pytest.mark.timeout(1500)
def test_full_cfg5_block_row_world1(cuda, cfg5_reference):
    """configs[4] through the block-row distributed chain (distchain) at
    world 1: the multi-GPU code path, one slab."""
    import torch

    from paper_2010_00465_b200 import distchain
    ref = cfg5_reference
    c, s, st = distchain.cos_sin_distributed(torch.from_numpy(ref["a"]).to(cuda))
    _check_cfg5(ref, c.cpu().numpy(), s.cpu().numpy(), st.k, st.s)
