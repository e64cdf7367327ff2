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


# -- criteria 3-5 on the reference's own acceptance corpus --------------------
# tests/golden/acceptance_corpus.npz: the 500-entry corpus of
# pkg/tests/test_acceptance.py:160-184 (seed 0, classes 162/220/109/9, norms
# in (1e-4, 1e4)) with the reference's own per-entry results
# (scripts/gen_golden.py gen_acceptance).

def _acceptance(golden_dir):
    import os
    d = np.load(os.path.join(golden_dir, "acceptance_corpus.npz"))
    mats, off = [], 0
    for n in d["dims"]:
        mats.append(d["data"][off:off + n * n].reshape(n, n))
        off += n * n
    return d, mats, [str(t) for t in d["tags"]]


def _criterion4_fraction(tags, norms, ec, es):
    """pkg/tests/test_acceptance.py:208-218: entries below 1e-11 in both
    errors, the overscaling rows with norm > 1e6 excluded."""
    included = [i for i in range(len(tags))
                if not (tags[i] == "overscaling" and norms[i] > 1e6)]
    good = [i for i in included if ec[i] < 1e-11 and es[i] < 1e-11]
    return len(good) / len(included), included


@pytest.mark.timeout(900)
def test_criteria_3_to_5_on_the_reference_corpus(cuda, golden_dir):
    """Criteria 3-5 (test_acceptance.py:187-254) with this implementation in
    place of the reference: the ledger law and (k, s) exactly as the
    reference's on all 500 entries (C3), the accuracy fraction of C4 no lower
    than the reference's own 92.4% (the reference fails the 95% gate by design,
    test_output.txt:353-359), and the Taylor-vs-Pade head-to-head (C5)."""
    import math

    from paper_2010_00465_b200 import corpus
    d, mats, tags = _acceptance(golden_dir)
    recs = corpus.run_corpus(mats, tags)
    t = recs[0::2]
    p = recs[1::2]
    n = len(mats)
    # C3: k + 2s (Taylor) and 22/3 + 2s (Pade), bit-exact with the reference
    for i in range(n):
        assert t[i].scaling_s == int(d["t_s"][i]) and t[i].products == float(d["t_prod"][i]), i
        assert p[i].scaling_s == int(d["p_s"][i]), i
        assert abs(p[i].products - float(d["p_prod"][i])) < 1e-12, i
        assert int(round(t[i].products)) - 2 * t[i].scaling_s in (3, 4, 6, 7)
    # C4: the same fraction computation on our errors and on the reference's
    norms = d["norm"]
    mine, inc = _criterion4_fraction(tags, norms, [r.rel_err_cos for r in t],
                                     [r.rel_err_sin for r in t])
    ref, _ = _criterion4_fraction(tags, norms, d["t_ec"], d["t_es"])
    assert abs(ref - 0.9235) < 1e-3  # the fixture reproduces the reference's 92.4%
    assert mine >= ref - 2.0 / len(inc), (mine, ref)
    # per entry: no worse than 10x the reference's error, up to the doubling
    # recursion's conditioning (tests/test_gpu_corpus.py)
    for i in range(n):
        for mine_e, ref_e in ((t[i].rel_err_cos, float(d["t_ec"][i])),
                              (t[i].rel_err_sin, float(d["t_es"][i]))):
            if math.isinf(ref_e):
                continue
            assert mine_e <= 10.0 * ref_e + max(1e-14, 64 * 2.0 ** -53 * 4.0 ** t[i].scaling_s), \
                (i, mine_e, ref_e)
    # C5: Taylor never costs more and is within 10x of Pade on >= 90%
    cheaper = sum(t[i].products <= p[i].products for i in range(n))
    comparable = sum(t[i].rel_err_cos <= 10.0 * p[i].rel_err_cos
                     and t[i].rel_err_sin <= 10.0 * p[i].rel_err_sin for i in range(n))
    assert cheaper >= 0.9 * n and comparable >= 0.9 * n, (cheaper, comparable)
    print(f"C3 ok on {n}; C4 {100 * mine:.1f}% below 1e-11 (reference {100 * ref:.1f}%); "
          f"C5 cheaper {cheaper}/{n}, comparable {comparable}/{n}")
