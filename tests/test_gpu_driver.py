"""The reference's driver-level tests (pkg/tests/test_driver.py:85-230),
restated against the GPU path: same inputs, same assertions, same
tolerances (the rng fixture uses the reference suite's seed)."""
import math
from fractions import Fraction

import numpy as np
import pytest

import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc

pytestmark = pytest.mark.gpu
TAY = csm.TAYLOR_TABLE[csm.Precision.DOUBLE]


def test_cos_sin_zero_matrix(cuda):
    r = csm.cos_sin(np.zeros((3, 3)))
    assert np.array_equal(r.result.cos_part, np.eye(3))
    assert np.array_equal(r.result.sin_part, np.zeros((3, 3)))
    assert r.scaling_exponent == 0 and r.total_products == Fraction(3)


def test_cos_sin_pi_diagonal(cuda):
    r = csm.cos_sin(np.diag([math.pi, math.pi]))
    assert (r.scheme_used.k_products, r.scaling_exponent) == (7, 1)
    assert r.total_products == Fraction(9)
    assert np.max(np.abs(r.result.cos_part + np.eye(2))) <= 1e-13
    assert np.max(np.abs(r.result.sin_part)) <= 1e-13


def test_cost_law_total_is_k_plus_2s(cuda, rng):
    for target in (0.004, 0.07, 0.6, 2.0, 55.0, 900.0):
        a = rng.standard_normal((5, 5))
        a *= target / orc.norm1(a)
        r = csm.cos_sin(a)
        scheme, s = csm.select_scheme(orc.norm1(a), TAY)
        assert r.scheme_used == scheme and r.scaling_exponent == s
        assert r.total_products == Fraction(scheme.k_products) + 2 * s


def test_pade_cost_law(cuda, rng):
    a = rng.standard_normal((4, 4))
    a *= 2.0 / orc.norm1(a)
    r = csm.pade_cos_sin(a)
    assert r.total_products == Fraction(22, 3) + 2 * r.scaling_exponent


def test_scalar_accuracy_through_doubling(cuda):
    r = csm.cos_sin(np.array([[2.7]]))
    assert r.scaling_exponent >= 1
    assert r.result.cos_part[0, 0] == pytest.approx(math.cos(2.7), abs=1e-15)
    assert r.result.sin_part[0, 0] == pytest.approx(math.sin(2.7), abs=1e-15)


def test_pythagorean_identity(cuda, rng):
    b = rng.standard_normal((8, 8))
    a = b + b.T
    a *= 50.0 / orc.norm1(a)
    r = csm.cos_sin(a)
    c, s = r.result.cos_part, r.result.sin_part
    assert orc.norm1(c @ c + s @ s - np.eye(8)) <= 1e-12


def test_wave_diagonal_example(cuda):
    r = csm.wave_cos_sin(np.diag([4.0, 4.0]), 2.0)
    assert (r.scheme_used.k_products, r.scaling_exponent) == (5, 3)
    assert np.max(np.abs(r.result.c_part - math.cos(4.0) * np.eye(2))) <= 1e-13
    assert np.max(np.abs(r.result.s_part - (math.sin(4.0) / 2.0) * np.eye(2))) <= 1e-13


def test_wave_small_norm_unscaled(cuda):
    r = csm.wave_cos_sin(np.diag([0.25, 0.01]), 1.0)
    assert r.scaling_exponent == 0
    assert r.result.c_part[0, 0] == pytest.approx(math.cos(0.5), abs=1e-15)
    assert r.result.s_part[0, 0] == pytest.approx(math.sin(0.5) / 0.5, abs=1e-15)


def test_pade_small_norm_unscaled(cuda):
    r = csm.pade_cos_sin(np.diag([0.1, -0.1]))
    assert r.scaling_exponent == 0 and r.total_products == Fraction(22, 3)
    assert r.result.cos_part[0, 0] == pytest.approx(math.cos(0.1), abs=1e-15)


def test_taylor_beats_pade_on_products(cuda, rng):
    a = rng.standard_normal((6, 6))
    a *= 2.0 / orc.norm1(a)
    assert csm.cos_sin(a).total_products < csm.pade_cos_sin(a).total_products


def test_single_precision_selection(cuda, rng):
    a = rng.standard_normal((4, 4))
    a *= 0.15 / orc.norm1(a)
    single = csm.cos_sin(a, csm.Precision.SINGLE)
    double = csm.cos_sin(a, csm.Precision.DOUBLE)
    assert single.scaling_exponent <= double.scaling_exponent
    assert single.total_products <= double.total_products
    assert np.max(np.abs(single.result.cos_part - double.result.cos_part)) <= 1e-7


def test_wave_rejects_bad_input(cuda):
    with pytest.raises(csm.MatrixInputError):
        csm.wave_cos_sin(np.zeros((2, 3)), 1.0)
    with pytest.raises(csm.MatrixInputError):
        csm.wave_cos_sin(np.array([[math.nan]]), 1.0)


def test_empty_matrices_like_the_reference(cuda):
    """0 x 0 inputs behave as in the reference: cos_sin / reference values /
    taylor_sin9 return empty results, pade_cos_sin raises (its pivot test is
    0 <= 0, matcore.py:141-147)."""
    from paper_2010_00465_b200 import verify
    e = np.zeros((0, 0))
    r = csm.cos_sin(e)
    assert r.result.cos_part.shape == (0, 0) and r.total_products == Fraction(3)
    ref = verify.reference_cos_sin(e)
    assert ref.cos_part.shape == (0, 0) and ref.cost.total_cost == 7
    assert csm.taylor_sin9(e, csm.CostLedger()).shape == (0, 0)
    with pytest.raises(csm.SingularMatrixError):
        csm.pade_cos_sin(e)
