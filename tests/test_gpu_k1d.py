"""K1d (two CTAs per SM, csrc/fused64d.cu) against K1 (csrc/fused64.cu) and the
oracle.  K1d restates K1's arithmetic operation for operation, so its outputs
must equal K1's BIT FOR BIT on every matrix; K1 itself is checked against the
oracle by test_gpu_parity.py, and the cfg2-like case is checked here again
through K1d (driver.py:108-123, schemes.py:264-395)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests import _k1d_worker
from tests._util import rel1

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, k1d):
    out = str(tmp_path / f"k1d_{k1d}.npz")
    env = dict(os.environ, CSM_K1D=str(k1d))
    subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_k1d_worker.py"), out],
                   check=True, env=env, cwd=ROOT, timeout=900)
    return np.load(out)


@pytest.fixture(scope="module")
def k1_outputs(tmp_path_factory, cuda):
    return _run(tmp_path_factory.mktemp("k1"), 0)


@pytest.fixture(scope="module")
def both(tmp_path_factory, k1_outputs):
    """(outputs of K1d, outputs of K1) on the same seeded batches."""
    return _run(tmp_path_factory.mktemp("k1d"), 1), k1_outputs


def test_k1d_bitwise_equals_k1(both):
    new, old = both
    assert sorted(new.files) == sorted(old.files)
    for key in new.files:
        a, b = new[key], old[key]
        assert a.shape == b.shape and a.dtype == b.dtype, key
        # NaN-filled outputs of rejected matrices compare equal as bits
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (
            key, int((a.view(np.uint8) != b.view(np.uint8)).sum()))


def test_k1d_covers_every_chain_and_deep_scaling(both):
    new, _ = both
    k = new["cfg2_like_64/k"]
    assert set(np.unique(k)) == {3, 4, 6, 7}
    assert new["deep_64/sx"].max() >= 8
    assert new["tiny_64/sx"].max() == 0
    st = new["nonfinite_64/st"]
    assert st[7] == 1 and st[123] == 1 and st[499] == 1 and st.sum() == 3
    assert np.isnan(new["nonfinite_64/c"][7]).all() and np.isnan(new["nonfinite_64/s"][499]).all()
    # the extreme cases reach the fallbacks: s beyond 511 (2**-2s no longer a
    # normal number: f * f), and tiny inputs whose y = A A is subnormal or zero
    assert new["huge_64/sx"].max() > 900 and new["huge_64/sx"].min() < 511
    assert new["subnormal_64/sx"].max() == 0
    assert (new["subnormal_64/st"] == 0).all()
    assert (new["huge_64/st"] == 0).sum() > 150  # (a few inputs overflow to inf: rejected)


def test_k1d_wave_family(both):
    """The wave chains on K1d: every k, scaling, and against the oracle."""
    from oracle import cossin_oracle as orc
    new, _ = both
    assert set(np.unique(new["wave_lap_64/k"])) == {3, 4, 5}
    assert new["wave_lap_64/sx"].max() >= 3 and new["wave_lap_64/sx"].min() == 0
    st = new["wave_nonfinite_64/st"]
    assert st[3] == 1 and st[199] == 1 and st.sum() == 2
    cases = _k1d_worker.wave_cases()
    rng = np.random.default_rng(6)
    for name, tol in (("wave_lap_64", 1e-12), ("wave_gauss_21", 1e-12), ("wave_f32_64", 1e-5)):
        a, t = cases[name]
        for i in rng.choice(a.shape[0], 16, replace=False):
            c, s, k, sc = orc.wave_cos_sin(a[i].astype(np.float64), float(t[i]))
            assert (k, sc) == (int(new[name + "/k"][i]), int(new[name + "/sx"][i])), (name, i)
            assert rel1(new[name + "/c"][i], c) <= tol, (name, i, k, sc)
            assert rel1(new[name + "/s"][i], s) <= tol, (name, i, k, sc)


def test_k1d_against_oracle(both):
    from oracle import cossin_oracle as orc
    new, _ = both
    cases = _k1d_worker.cases()
    rng = np.random.default_rng(5)
    # (deep scaling is covered by the bitwise comparison with K1, whose own
    # noise-floor-gated parity tests are in test_gpu_parity.py)
    for name, tol in (("cfg2_like_64", 1e-12), ("n37", 1e-12), ("n5", 1e-12), ("f32_64", 1e-5)):
        a = cases[name]
        for i in rng.choice(a.shape[0], 24, replace=False):
            c, s, k, sc = orc.cos_sin(a[i].astype(np.float64))
            assert (k, sc) == (int(new[name + "/k"][i]), int(new[name + "/sx"][i])), (name, i)
            assert rel1(new[name + "/c"][i], c) <= tol, (name, i, k, sc)
            assert rel1(new[name + "/s"][i], s) <= tol, (name, i, k, sc)
