"""The reference's scheme-layer tests (pkg/tests/test_schemes.py) run against
the device scheme cores: product budgets, bitwise zero-matrix identities,
diagonal reduction with exact-zero off-diagonals, scalar closed forms,
the hyperbolic continuation of the wave kernels, result shapes and the
scheme-id validation.  Same inputs and tolerances as the reference's own
tests (line numbers cited per test)."""
import math
from fractions import Fraction

import numpy as np
import pytest

import paper_2010_00465_b200 as csm

pytestmark = pytest.mark.gpu

TAYLOR_KS = (3, 4, 6, 7)
WAVE_KS = (3, 4, 5)


def _taylor(k):
    return csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, k)


def _wave(k):
    return csm.SchemeId(csm.SchemeFamily.WAVE_KERNEL, k)


@pytest.mark.parametrize("k", TAYLOR_KS)
def test_taylor_product_budget(cuda, k):  # test_schemes.py:36-41
    ledger = csm.CostLedger()
    csm.taylor_cos_sin(np.zeros((3, 3)), _taylor(k), ledger)
    assert ledger.total_cost == Fraction(k)


@pytest.mark.parametrize("k", WAVE_KS)
def test_wave_product_budget(cuda, k):  # :44-48
    ledger = csm.CostLedger()
    csm.wave_kernels(np.zeros((3, 3)), 0.5, _wave(k), ledger)
    assert ledger.total_cost == Fraction(k)


def test_standalone_sine_budgets(cuda):  # :51-60
    ledger = csm.CostLedger()
    csm.taylor_sin9(np.zeros((2, 2)), ledger)
    assert ledger.total_cost == Fraction(5)
    ledger = csm.CostLedger()
    csm.wave_sin34(np.zeros((2, 2)), 1.0, ledger)
    assert ledger.total_cost == Fraction(2)


@pytest.mark.parametrize("k", TAYLOR_KS)
def test_taylor_zero_matrix(cuda, k):  # :69-73
    out = csm.taylor_cos_sin(np.zeros((4, 4)), _taylor(k), csm.CostLedger())
    assert np.array_equal(out.cos_part, np.eye(4))
    assert np.array_equal(out.sin_part, np.zeros((4, 4)))


@pytest.mark.parametrize("k", WAVE_KS)
def test_wave_zero_matrix(cuda, k):  # :76-81: s(t, 0) is the sinc limit t I
    """c(0) = I bitwise for every k, s(t, 0) = t I bitwise for k = 3, 4.  For
    k = 5 the reference's s = t (z_0 I + ... + z_11 cos) sums its twelve
    coefficients to exactly 1 only in its own operation order (matcore.lin,
    one rounding per term); the fused FMA epilogue rounds differently and
    lands within one ulp of t."""
    out = csm.wave_kernels(np.zeros((4, 4)), 0.7, _wave(k), csm.CostLedger())
    assert np.array_equal(out.c_part, np.eye(4))
    if k < 5:
        assert np.array_equal(out.s_part, 0.7 * np.eye(4))
    else:
        assert np.all(out.s_part[~np.eye(4, dtype=bool)] == 0.0)
        assert np.all(np.abs(np.diag(out.s_part) - 0.7) <= np.spacing(0.7))


@pytest.mark.parametrize("k", WAVE_KS)
def test_wave_zero_time(cuda, k, rng):  # :84-89
    out = csm.wave_kernels(rng.standard_normal((3, 3)), 0.0, _wave(k), csm.CostLedger())
    assert np.array_equal(out.c_part, np.eye(3))
    assert np.array_equal(out.s_part, np.zeros((3, 3)))


@pytest.mark.parametrize("k", TAYLOR_KS)
def test_taylor_diagonal_reduction(cuda, k):  # :98-110
    d = np.diag([0.1, -0.3, 0.55])
    out = csm.taylor_cos_sin(d, _taylor(k), csm.CostLedger())
    off = ~np.eye(3, dtype=bool)
    assert np.all(out.cos_part[off] == 0.0)
    assert np.all(out.sin_part[off] == 0.0)
    if k >= 6:
        for i, x in enumerate(np.diag(d)):
            assert out.cos_part[i, i] == pytest.approx(math.cos(x), abs=1e-15)
            assert out.sin_part[i, i] == pytest.approx(math.sin(x), abs=1e-15)


def test_sin9_scalar_accuracy(cuda):  # :113-119
    d = np.diag([0.1, -0.05])
    got = csm.taylor_sin9(d, csm.CostLedger())
    assert got[0, 0] == pytest.approx(math.sin(0.1), abs=1e-15)
    assert got[1, 1] == pytest.approx(math.sin(-0.05), abs=1e-15)


def test_wave_scalar_values(cuda):  # :122-132
    a = np.diag([0.25, 4.0])
    t = 0.5
    out = csm.wave_kernels(a, t, _wave(5), csm.CostLedger())
    for i, x in enumerate(np.diag(a)):
        w = math.sqrt(x)
        assert out.c_part[i, i] == pytest.approx(math.cos(t * w), abs=1e-14)
        assert out.s_part[i, i] == pytest.approx(math.sin(t * w) / w, abs=1e-14)


def test_wave_hyperbolic_continuation(cuda):  # :135-141: cosh / sinh for a < 0
    w = 0.7
    a = np.diag([-(w * w)])
    out = csm.wave_kernels(a, 1.0, _wave(5), csm.CostLedger())
    assert out.c_part[0, 0] == pytest.approx(math.cosh(w), abs=1e-14)
    assert out.s_part[0, 0] == pytest.approx(math.sinh(w) / w, abs=1e-14)


def test_wave_hyperbolic_through_the_driver(cuda):
    """The same continuation through wave_cos_sin with scaling (s > 0) and
    on the tiled (n > 128) and K1 paths: cosh / sinh of a diagonal with
    negative entries."""
    for n in (5, 160):
        w = np.linspace(0.2, 3.0, n)
        a = np.diag(-(w * w))
        r = csm.wave_cos_sin(a, 2.0)
        assert r.scaling_exponent > 0
        np.testing.assert_allclose(np.diag(r.result.c_part), np.cosh(2.0 * w), rtol=1e-13)
        np.testing.assert_allclose(np.diag(r.result.s_part), np.sinh(2.0 * w) / w, rtol=1e-13)
        off = ~np.eye(n, dtype=bool)
        assert np.all(r.result.c_part[off] == 0.0) and np.all(r.result.s_part[off] == 0.0)


def test_result_shapes(cuda, rng):  # :181-188
    a = 0.1 * rng.standard_normal((4, 4))
    out = csm.taylor_cos_sin(a, _taylor(6), csm.CostLedger())
    assert out.cos_part.shape == (4, 4) and out.sin_part.shape == (4, 4)
    wout = csm.wave_kernels(a, 0.3, _wave(4), csm.CostLedger())
    assert wout.c_part.shape == (4, 4) and wout.s_part.shape == (4, 4)


def test_scheme_family_checks(cuda):  # schemes.py:384-385, :420-421
    with pytest.raises(ValueError):
        csm.taylor_cos_sin(np.eye(2), _wave(4), csm.CostLedger())
    with pytest.raises(ValueError):
        csm.wave_kernels(np.eye(2), 1.0, _taylor(4), csm.CostLedger())
    with pytest.raises(ValueError):
        csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, 5)
