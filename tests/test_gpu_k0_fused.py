"""The fused K0 launch (csrc/k0_select.cu norm_select_kernel: one warp per
matrix computes norm1, finiteness, (k, s) and the schedule's cost histogram)
against the separate norm1 / select / histogram launches (CSM_K0_FUSED=0 in
a subprocess) and against the oracle's selection (matcore.py:100-104,
driver.py:64-88).  Same column sums in the same order, so (k, s), status and
every output bit must be equal."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import cossin_oracle as orc
from tests import _k0_worker

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, fused):
    out = str(tmp_path / f"k0_{fused}.npz")
    env = dict(os.environ, CSM_K0_FUSED=str(fused))
    subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_k0_worker.py"), out],
                   check=True, env=env, cwd=ROOT, timeout=900)
    return np.load(out)


@pytest.fixture(scope="module")
def both(tmp_path_factory, cuda):
    return (_run(tmp_path_factory.mktemp("k0f"), 1), _run(tmp_path_factory.mktemp("k0s"), 0))


def test_fused_k0_bitwise_equals_separate_launches(both):
    new, old = both
    assert sorted(new.files) == sorted(old.files)
    for key in new.files:
        a, b = new[key], old[key]
        assert a.shape == b.shape and a.dtype == b.dtype, key
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (
            key, int((a.view(np.uint8) != b.view(np.uint8)).sum()))


def test_fused_k0_selection_matches_oracle(both):
    new, _ = both
    for name, (a, t) in _k0_worker.cases().items():
        k, s, st = new[f"{name}/k"], new[f"{name}/s"], new[f"{name}/st"]
        if f"{name}/k_unaligned" in new.files:  # the scalar-load variant agrees
            assert np.array_equal(k, new[f"{name}/k_unaligned"]), name
            assert np.array_equal(s, new[f"{name}/s_unaligned"]), name
            assert np.array_equal(st, new[f"{name}/st_unaligned"]), name
        for i in range(a.shape[0]):
            x = a[i]
            if not np.isfinite(x).all():
                assert st[i] == 1, (name, i)
                continue
            norm = orc.norm1(x)  # summed in the input's dtype, like matcore.py:100-104
            if t is not None:
                norm = float(t[i]) * float(t[i]) * norm
            try:
                kk, ss = orc.select(norm, "wave" if t is not None else "taylor", "double")
            except (ValueError, OverflowError):
                assert st[i] != 0, (name, i)
                continue
            assert st[i] == 0 and (int(k[i]), int(s[i])) == (kk, ss), (name, i)


def test_fused_k0_status_cases(both):
    new, _ = both
    st = new["status_64/st"]
    assert st[3] == 1 and st[100] == 1 and st[255] == 1
    assert st[18] == 0 and st[19] == 0 and new["status_64/k"][19] == 3
