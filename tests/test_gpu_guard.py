"""The Ozaki engine's accuracy guard on badly scaled operands (the default
engine runs Ozaki-II from padded order 768 up).

Ozaki-II rounds each row of L and each column of R to P bits of that row's
(column's) maximum, so entries far below their row / column maximum lose
accuracy an fp64 GEMM (matcore.py:97) keeps.  oz_guard bounds that error a
priori for every product and reruns the product on DMMA unless the bound
stays below n u ||C||_1.  These tests run the reference gallery's graded
families (Pascal, Frank, Lehmer, Grcar; gallery.py:57-179, rescaled as
:182-183) and graded D B D^-1 at n = 768 and 1024 through the default
engine and compare with the oracle at max(1e-12, 4 x the oracle's own
permuted-order noise) -- the SURVEY.md 8a gate.  The unguarded engine
(CSM_ENGINE_OZAKI_UNGUARDED, experiments only) fails that gate on some of
them, which is what the guard is for."""
import numpy as np
import pytest

import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc
from tests._util import (gallery_frank, gallery_grcar, gallery_lehmer, gallery_pascal_lower,
                         graded, pair_close, permuted_noise, rescaled)

pytestmark = pytest.mark.gpu

TARGETS = (2.0, 50.0, 1000.0)


def _cases(n):
    rng = np.random.default_rng(4000 + n)
    fams = [("pascal_lower", gallery_pascal_lower(n)), ("frank", gallery_frank(n)),
            ("lehmer", gallery_lehmer(n)), ("grcar", gallery_grcar(n))]
    fams += [(f"graded{sp:g}", graded(rng, n, sp)) for sp in (1e4, 1e8, 1e12)]
    names, mats = [], []
    for name, m in fams:
        for t in TARGETS:
            names.append(f"{name}@{t:g}")
            mats.append(rescaled(m, t))
    return names, np.stack(mats)


_ORACLE = {}


def _oracle(n):
    if n not in _ORACLE:
        names, a = _cases(n)
        rng = np.random.default_rng(99)
        refs = [permuted_noise(orc.cos_sin, a[i], rng) for i in range(a.shape[0])]
        _ORACLE[n] = (names, a, refs)
    return _ORACLE[n]


def _errors(rep, refs):
    out = []
    for i, ((c, s, k, sc), noise) in enumerate(refs):
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc)
        gate = max(1e-12, 4.0 * noise)
        okc, ec = pair_close(rep.cos_part[i], c, s, gate)
        oks, es = pair_close(rep.sin_part[i], s, c, gate)
        out.append((okc and oks, max(ec, es), gate))
    return out


@pytest.mark.parametrize("n", [768, 1024])
def test_default_engine_on_badly_scaled_inputs(cuda, n):
    names, a, refs = _oracle(n)
    assert csm.get_engine() == "auto"  # Ozaki-II at these orders
    rep = csm.cos_sin_batched(a)
    bad = [(nm, e, g) for nm, (ok, e, g) in zip(names, _errors(rep, refs)) if not ok]
    assert not bad, bad


@pytest.mark.parametrize("n", [768, 1024])
def test_dmma_engine_on_badly_scaled_inputs(cuda, n):
    names, a, refs = _oracle(n)
    with csm.engine_scope("dmma"):
        rep = csm.cos_sin_batched(a)
    bad = [(nm, e, g) for nm, (ok, e, g) in zip(names, _errors(rep, refs)) if not ok]
    assert not bad, bad


def test_unguarded_engine_fails_where_the_guard_steps_in(cuda):
    """Without the guard the Ozaki rounding shows: Frank at norm 1000
    (k = 6, s = 10) lands orders of magnitude past the gate (a CPU model
    of the rounding gives 3.6e-8 against a 1.4e-13 noise floor)."""
    n = 768
    names, a, refs = _oracle(n)
    i = names.index("frank@1000")
    with csm.engine_scope("ozaki-unguarded"):
        rep = csm.cos_sin_batched(a[i:i + 1])
    (ok, err, gate), = _errors(rep, refs[i:i + 1])
    assert not ok and err > 100 * gate, (err, gate)
    rep = csm.cos_sin_batched(a[i:i + 1])  # guarded default
    (ok, err, gate), = _errors(rep, refs[i:i + 1])
    assert ok, (err, gate)


def test_guard_keeps_well_scaled_products_on_ozaki(cuda):
    """On well-scaled inputs the guard does not fire: the default engine's
    result differs from the DMMA engine's (it IS the Ozaki product), and
    it is bit-identical to the engine without the guard."""
    rng = np.random.default_rng(5)
    g = rng.standard_normal((3, 768, 768))
    a = g * (np.array([0.5, 20.0, 300.0]) / np.abs(g).sum(axis=1).max(axis=1))[:, None, None]
    auto = csm.cos_sin_batched(a)
    with csm.engine_scope("ozaki-unguarded"):
        ung = csm.cos_sin_batched(a)
    with csm.engine_scope("dmma"):
        dm = csm.cos_sin_batched(a)
    assert np.array_equal(auto.cos_part, ung.cos_part)
    assert np.array_equal(auto.sin_part, ung.sin_part)
    assert not np.array_equal(auto.cos_part, dm.cos_part)
