"""Badly scaled operands: the default engine, and the Ozaki engine's
accuracy guard.

Ozaki-II rounds each row of L and each column of R to P bits of that row's
(column's) maximum, so entries far below their row / column maximum lose
accuracy an fp64 GEMM (matcore.py:97) keeps.  oz_guard bounds that error a
priori for every product and reruns the product on DMMA unless the bound
stays below n u ||C||_1 -- a NORM-WISE guarantee per product.

The inputs are the reference gallery's graded families (Pascal, Frank,
Lehmer, Grcar; gallery.py:57-179, rescaled as :182-183) and graded D B D^-1,
at n = 768 and 1024 and 1-norms 2, 50 and 1000 (s up to 10).

* The DEFAULT engine (DMMA, componentwise error like the reference's GEMM)
  matches the oracle on all of them at max(1e-12, 4 x the oracle's own
  permuted-order noise) -- the SURVEY.md 8a gate.
* Per product, the guarded Ozaki engine stays within its bound n u ||C||_1
  on every operand pair of those chains, measured against double-double
  products; without the guard (CSM_ENGINE_OZAKI_UNGUARDED, experiments
  only) Pascal and graded operands break it by orders of magnitude.
* Whole chains on the Ozaki engine: the guard rescues Frank at norm 1000
  (unguarded 3.6e-8 off); graded chains with s = 10 doublings still lose
  accuracy through products that pass the norm-wise test (cos ~ I + small
  graded entries, rounded relative to the diagonal), which is why DMMA is
  the default (K7)."""
import numpy as np
import pytest

import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc
from tests._util import (gallery_frank, gallery_grcar, gallery_lehmer, gallery_pascal_lower,
                         graded, pair_close, permuted_noise, rel1, rescaled)

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
    assert csm.get_engine() == "dmma"  # the default
    rep = csm.cos_sin_batched(a)
    bad = [(nm, e, g) for nm, (ok, e, g) in zip(names, _errors(rep, refs)) if not ok]
    assert not bad, bad


def _slab_product(L, R, engine):
    """One product L R through csm_slab_op (world 1, no scaling)."""
    import torch
    from paper_2010_00465_b200 import distchain
    n = L.shape[0]
    steps, _, _ = distchain.chain_program(3, fold=False)
    op = steps[0][0]  # slot 1 = slot 0 @ right operand
    dev = torch.device("cuda")
    slab = torch.zeros((9, n, n), dtype=torch.float64, device=dev)
    co = torch.empty((n, n), dtype=torch.float64, device=dev)
    so = torch.empty_like(co)
    with csm.engine_scope(engine):
        scratch = torch.empty(distchain._slab_scratch_size(n, n), dtype=torch.uint8, device=dev)
        distchain._device_slab_op(op, slab, n, n, 0, torch.from_numpy(R).to(dev),
                                  torch.from_numpy(L).to(dev), 0, -1, co, so, scratch, None)
    return slab[1].cpu().numpy()


def test_guard_holds_the_per_product_bound(cuda):
    """Every operand pair the chains of the badly scaled cases multiply
    first (A A, y y, and the doubling's C C and S C from the oracle's own
    cos / sin): the guarded Ozaki product is within n u ||C||_1 of the
    double-double product; the unguarded one breaks that bound on Pascal
    and the graded matrices."""
    from paper_2010_00465_b200 import verify
    n = 768
    names, a, refs = _oracle(n)
    u = 2.0 ** -53
    broken = set()
    for i, nm in enumerate(names):
        (c, s, k, sc), _ = refs[i]
        x = a[i] * 2.0 ** -sc
        y = x @ x
        cc = c / np.abs(c).sum(axis=0).max()
        pairs = [("AA", x, x), ("yy", y, y), ("CC", cc, cc), ("SC", s, cc)]
        for lab, L, R in pairs:
            if not np.abs(L).any() or not np.abs(R).any():
                continue
            th, tl = verify.dd_matmul(L, None, R)
            norm = float(np.abs(th).sum(axis=0).max())
            if norm == 0.0:
                continue
            guarded = _slab_product(L, R, "ozaki")
            err = float(np.abs(guarded - th - tl).sum(axis=0).max())
            assert err <= (n + 2) * u * norm, (nm, lab, err / norm)
            unguarded = _slab_product(L, R, "ozaki-unguarded")
            if float(np.abs(unguarded - th - tl).sum(axis=0).max()) > 100 * n * u * norm:
                broken.add(nm.split("@")[0])
    assert {"pascal_lower", "graded1e+08", "graded1e+12"} <= broken, broken


def test_guard_rescues_a_chain(cuda):
    """Frank at norm 1000 (k = 6, s = 10): without the guard the Ozaki chain
    lands 3.6e-8 from the oracle (gate ~5e-13); with it, within the gate."""
    n = 768
    names, a, refs = _oracle(n)
    i = names.index("frank@1000")
    with csm.engine_scope("ozaki-unguarded"):
        rep = csm.cos_sin_batched(a[i:i + 1])
    (ok, err, gate), = _errors(rep, refs[i:i + 1])
    assert not ok and err > 100 * gate, (err, gate)
    with csm.engine_scope("ozaki"):
        rep = csm.cos_sin_batched(a[i:i + 1])
    (ok, err, gate), = _errors(rep, refs[i:i + 1])
    assert ok, (err, gate)


def test_guard_keeps_well_scaled_products_on_ozaki(cuda):
    """On well-scaled inputs the guard does not fire: the guarded result is
    bit-identical to the engine without the guard, differs from the DMMA
    engine's (it IS the Ozaki product), and matches the oracle."""
    rng = np.random.default_rng(5)
    g = rng.standard_normal((3, 768, 768))
    a = g * (np.array([0.5, 20.0, 300.0]) / np.abs(g).sum(axis=1).max(axis=1))[:, None, None]
    with csm.engine_scope("ozaki"):
        oz = csm.cos_sin_batched(a)
    with csm.engine_scope("ozaki-unguarded"):
        ung = csm.cos_sin_batched(a)
    dm = csm.cos_sin_batched(a)
    assert np.array_equal(oz.cos_part, ung.cos_part)
    assert np.array_equal(oz.sin_part, ung.sin_part)
    assert not np.array_equal(oz.cos_part, dm.cos_part)
    prng = np.random.default_rng(7)
    for i in range(a.shape[0]):
        (c, s, _, _), noise = permuted_noise(orc.cos_sin, a[i], prng)
        gate = max(1e-12, 4.0 * noise)  # norm 300: s = 8, the oracle's own noise ~1e-12
        assert rel1(oz.cos_part[i], c) <= gate and rel1(oz.sin_part[i], s) <= gate, (i, gate)
