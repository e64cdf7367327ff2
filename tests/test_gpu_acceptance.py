"""The reference's acceptance criteria 6 and 7 (pkg/tests/test_acceptance.py
:250-354) run through the GPU path.  Criterion 7's involutory leg fails by
design in the reference itself (7.7e-9 at lambda = 1e4, s = 13); here it is
held to the reference's own error, measured with the pinned oracle."""
import math

import numpy as np
import pytest

import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc

pytestmark = pytest.mark.gpu


def _rel2(x, y):
    d = float(np.linalg.norm(y, 2))
    return float(np.linalg.norm(x - y, 2)) / d if d else float(np.linalg.norm(x, 2))


def test_criterion_6_wave_block_identity(cuda):
    """c(t^2 A), s(t, A) against cos / sin of t sqrt(A) (eigh), 20 SPD draws
    with the reference's seed; the wave 2x2 block identity to 1e-11."""
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(20):
        dim = int(rng.integers(2, 9))
        basis = np.linalg.qr(rng.standard_normal((dim, dim)))[0]
        eig = rng.uniform(0.05, 9.0, dim)
        a = (basis * eig) @ basis.T
        a = 0.5 * (a + a.T)
        t = float(rng.uniform(0.2, 2.0))
        wave = csm.wave_cos_sin(a, t)
        vals, vecs = np.linalg.eigh(a)
        root = (vecs * np.sqrt(vals)) @ vecs.T
        trig = csm.cos_sin(t * root)
        sin_scaled = np.linalg.solve(root, trig.result.sin_part)
        bw = np.block([[wave.result.c_part, wave.result.s_part],
                       [-a @ wave.result.s_part, wave.result.c_part]])
        bt = np.block([[trig.result.cos_part, sin_scaled],
                       [-a @ sin_scaled, trig.result.cos_part]])
        worst = max(worst, _rel2(bw, bt))
    assert worst <= 1e-11, worst


def test_criterion_7_property_suite(cuda):
    z = csm.cos_sin(np.zeros((3, 3)))
    assert np.array_equal(z.result.cos_part, np.eye(3))
    assert np.array_equal(z.result.sin_part, np.zeros((3, 3)))
    w = csm.wave_cos_sin(np.zeros((2, 2)), 0.4)
    assert np.array_equal(w.result.c_part, np.eye(2))
    assert np.array_equal(w.result.s_part, 0.4 * np.eye(2))
    d = np.diag([0.2, -1.1, 3.0])
    r = csm.cos_sin(d).result
    off = ~np.eye(3, dtype=bool)
    assert np.all(r.cos_part[off] == 0.0)
    for i, x in enumerate(np.diag(d)):
        assert abs(r.cos_part[i, i] - math.cos(x)) <= 1e-14
        assert abs(r.sin_part[i, i] - math.sin(x)) <= 1e-14
    rng = np.random.default_rng(11)
    for target, symmetric in ((0.5, False), (5.0, False), (40.0, True)):
        a = rng.standard_normal((6, 6))
        if symmetric:
            a = a + a.T
        a *= target / orc.norm1(a)
        out = csm.cos_sin(a).result
        defect = orc.norm1(out.cos_part @ out.cos_part + out.sin_part @ out.sin_part
                           - np.eye(6))
        assert defect <= 1e-10, (target, defect)
    # involutory family cos([[1, lam], [0, -1]]) = cos(1) I: the norm-driven
    # scaling squares away accuracy (the reference fails its own 1e-10 bar
    # at lam = 1e4); the GPU path must not be worse than the reference
    for j in range(5):
        a = np.array([[1.0, 10.0 ** j], [0.0, -1.0]])
        truth = math.cos(1.0) * np.eye(2)
        mine = _rel2(csm.cos_sin(a).result.cos_part, truth)
        ref = _rel2(orc.cos_sin(a)[0], truth)
        assert mine <= 10.0 * ref + 1e-15, (j, mine, ref)


@pytest.mark.parametrize("n", [8, 64, 100, 200])
def test_wave_k4_c_chain_is_the_taylor_k6_cos_chain(cuda, n):
    """pkg/tests/test_schemes.py:144-151: the wave k=4 c-chain on R^2 is the
    Taylor k=6 cos chain on R, bit for bit (one shared even-variable chain).
    R has entries in 2^-6 Z, so R R is exact and both chains see the same y."""
    rng = np.random.default_rng(900 + n)
    r = rng.integers(-3, 4, (n, n)).astype(np.float64) / 64.0
    r2 = r @ r
    assert np.array_equal(r2, np.round(r2 * 4096.0) / 4096.0)  # exact
    w = csm.wave_kernels(r2, 1.0, csm.SchemeId(csm.SchemeFamily.WAVE_KERNEL, 4),
                         csm.CostLedger())
    t = csm.taylor_cos_sin(r, csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, 6),
                           csm.CostLedger())
    assert np.array_equal(w.c_part, t.cos_part)
