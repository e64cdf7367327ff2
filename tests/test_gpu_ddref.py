"""GPU double-double reference values (csm_ddref_cos_sin / csm_dd_matmul)
against the reference's own outputs (tests/golden/ddref.npz, generated from
verify.py:449-521) and the pinned numpy restatement: bit for bit."""
import os

import numpy as np
import pytest

import paper_2010_00465_b200 as csm
from paper_2010_00465_b200 import verify as V
from oracle import cossin_oracle as orc
from oracle import ddref_oracle as ddo
from tests.test_oracle_golden import _bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden(golden_dir):
    return np.load(os.path.join(golden_dir, "ddref.npz"))


def test_dd_matmul_golden_bitwise(cuda, golden):
    for n in (1, 7, 40, 65):
        g = {k: golden[f"mm{n}__{k}"] for k in ("xh", "xl", "yh", "yl", "oh", "ol")}
        oh, ol = V.dd_matmul(g["xh"], g["xl"], g["yh"], g["yl"])
        assert _bits_equal(oh, g["oh"]), n
        assert _bits_equal(ol, g["ol"]), n


def test_reference_cos_sin_golden_bitwise(cuda, golden):
    for name in golden["names"]:
        name = str(name)
        res = V.reference_cos_sin(golden[f"{name}__a"])
        assert res.cost.total_cost == int(golden[f"{name}__cost"]), name
        assert _bits_equal(res.cos_part, golden[f"{name}__cos"]), name
        assert _bits_equal(res.sin_part, golden[f"{name}__sin"]), name


def test_batched_mixed_scaling_matches_oracle(cuda, rng):
    """One call, matrices with different s (per-matrix pass-through in the
    doubling launches), n not a multiple of the 64 tile."""
    n = 96
    norms = [1e-8, 0.7, 35.0]
    a = rng.standard_normal((3, n, n))
    a *= (np.array(norms) / np.abs(a).sum(axis=1).max(axis=1))[:, None, None]
    c, s, sc = V.reference_cos_sin_batched(a)
    for i in range(3):
        rc, rs, rsc = ddo.reference_cos_sin(a[i])
        assert sc[i] == rsc
        assert _bits_equal(c[i], rc), i
        assert _bits_equal(s[i], rs), i
    assert sc[0] == 0 and sc[2] > sc[1] > 0


def test_overflow_and_shape_errors(cuda):
    with pytest.raises(OverflowError):
        V.reference_cos_sin(np.array([[1e308, 0.0], [1e308, 0.0]]))
    with pytest.raises(csm.MatrixInputError):
        V.reference_cos_sin(np.zeros((2, 3)))


def test_fast_path_accuracy_against_ddref(cuda, rng):
    """The product path's cos/sin against the double-double values: the
    accuracy the reference's verify module reports, at n = 256."""
    n = 256
    a = rng.standard_normal((n, n))
    a *= 3.0 / orc.norm1(a)
    rep = csm.cos_sin(a)
    ref = V.reference_cos_sin(a)
    for got, want in ((rep.result.cos_part, ref.cos_part),
                      (rep.result.sin_part, ref.sin_part)):
        err = np.linalg.norm(got - want, 2) / np.linalg.norm(want, 2)
        assert err < 1e-13
