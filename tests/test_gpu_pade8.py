"""pade8_cos_sin, the Pade base pair with no scaling (schemes.py:446-464),
on the device (csm_pade_core) against the oracle's pade8_core and the
reference's own scheme tests (pkg/tests/test_schemes.py:63-66, :92-95,
:173-178, :208-213, :216-218)."""
import math
from fractions import Fraction

import numpy as np
import pytest

import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc
from tests._util import pair_close

pytestmark = pytest.mark.gpu


def test_pade8_constant_id_and_k():
    assert csm.PADE8.family is csm.SchemeFamily.PADE8
    assert csm.PADE8.k_products == 5


def test_pade8_budget_is_7_and_a_third(cuda):
    ledger = csm.CostLedger()
    csm.pade8_cos_sin(np.zeros((3, 3)), ledger)
    assert ledger.total_cost == Fraction(22, 3)


def test_pade8_zero_matrix(cuda):
    out = csm.pade8_cos_sin(np.zeros((2, 2)), csm.CostLedger())
    assert np.allclose(out.cos_part, np.eye(2), atol=1e-15)
    assert np.array_equal(out.sin_part, np.zeros((2, 2)))


def test_pade8_diagonal_accuracy(cuda):
    d = np.diag([0.05, -0.11])
    out = csm.pade8_cos_sin(d, csm.CostLedger())
    for i, x in enumerate(np.diag(d)):
        assert out.cos_part[i, i] == pytest.approx(math.cos(x), abs=1e-15)
        assert out.sin_part[i, i] == pytest.approx(math.sin(x), abs=1e-15)


def test_pade8_matches_taylor_at_small_norm(cuda, rng):
    a = 0.05 * rng.standard_normal((4, 4))
    p = csm.pade8_cos_sin(a, csm.CostLedger())
    t = csm.taylor_cos_sin(a, csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, 7),
                           csm.CostLedger())
    assert np.max(np.abs(p.cos_part - t.cos_part)) <= 1e-14
    assert np.max(np.abs(p.sin_part - t.sin_part)) <= 1e-14


@pytest.mark.parametrize("n", [5, 64, 100, 257])
def test_pade8_against_oracle(cuda, n):
    rng = np.random.default_rng(900 + n)
    a = rng.standard_normal((n, n))
    a *= 1.2 / orc.norm1(a)  # inside PADE_TABLE's theta (no scaling needed)
    out = csm.pade8_cos_sin(a, csm.CostLedger())
    c, s = orc.pade8_core(a)
    assert pair_close(out.cos_part, c, s, 1e-12)[0]
    assert pair_close(out.sin_part, s, c, 1e-12)[0]


def test_pade8_device_tensors(cuda, rng):
    import torch
    a = 0.3 * rng.standard_normal((16, 16))
    out = csm.pade8_cos_sin(torch.from_numpy(a).to(cuda), csm.CostLedger())
    assert out.cos_part.is_cuda and out.sin_part.is_cuda
    c, s = orc.pade8_core(a)
    assert pair_close(out.cos_part.cpu().numpy(), c, s, 1e-12)[0]


def _singular_input():
    """A 4 x 4 input whose Pade denominator is singular: the denominator
    sum d_i z^i has no real roots, so take a complex root z0 = x + iy and
    the real 2 x 2 block A = [[u, -v], [v, u]] with (u + iv)^2 = z0; then
    A^2 represents z0 and the denominator's leading block represents
    d(z0) = 0 (to rounding).  The trailing 2 x 2 block is 0, so
    ||den||_1 >= 1 and the threshold 1e3 eps ||den||_1 is meaningful."""
    d = [float(c) for c in orc.PADE_DEN]
    z = min(np.roots(d[::-1]), key=abs)
    for _ in range(50):  # Newton polish in complex128
        f = sum(c * z ** i for i, c in enumerate(d))
        fp = sum(i * c * z ** (i - 1) for i, c in enumerate(d) if i)
        z -= f / fp
    r = np.sqrt(complex(z))
    a = np.zeros((4, 4))
    a[0, 0], a[0, 1], a[1, 0], a[1, 1] = r.real, -r.imag, r.imag, r.real
    return a


def test_pade8_singular_denominator(cuda):
    """The reference raises SingularMatrixError from lu_solve_pair
    (matcore.py:141-147) after charging the five products."""
    a = _singular_input()
    with pytest.raises(orc.SingularDenominator):
        orc.pade8_core(a)
    ledger = csm.CostLedger()
    with pytest.raises(csm.SingularMatrixError):
        csm.pade8_cos_sin(a, ledger)
    assert ledger.products == 5 and ledger.lu_factorizations == 0


def test_pade8_empty_is_singular(cuda):
    # lu_factor of 0 x 0: min pivot 0 <= threshold 0 (matcore.py:141-147)
    ledger = csm.CostLedger()
    with pytest.raises(csm.SingularMatrixError):
        csm.pade8_cos_sin(np.zeros((0, 0)), ledger)
    assert ledger.products == 5
