"""Host C++ twin of select_scheme (driver.py:64-88) against the reference's
golden selections and the oracle, plus the reference's own selection tests
(pkg/tests/test_driver.py:27-71) restated on the drop-in API."""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc

FAM = {"taylor": csm.SchemeFamily.COS_SIN_TAYLOR,
       "wave": csm.SchemeFamily.WAVE_KERNEL, "pade": csm.SchemeFamily.PADE8}
PREC = {"double": csm.Precision.DOUBLE, "single": csm.Precision.SINGLE}


def test_tables_carry_reference_bits(golden_dir):
    import json
    doc = json.load(open(os.path.join(golden_dir, "constants.json")))
    for key, ents in doc["tables"].items():
        fam, prec = key.split("_")
        tab = csm.table_for(FAM[fam], PREC[prec])
        assert [e.scheme.k_products for e in tab.entries] == [e["k"] for e in ents]
        for mine, ref in zip(tab.entries, ents):
            assert mine.theta_cos == float.fromhex(ref["theta_cos"])
            assert mine.theta_sin == float.fromhex(ref["theta_sin"])
            assert mine.cost == Fraction(ref["cost"])


def test_host_twin_matches_reference_golden(golden_dir):
    g = np.load(os.path.join(golden_dir, "selection.npz"))
    for fam in ("taylor", "wave", "pade"):
        for prec in ("double", "single"):
            key = f"{fam}_{prec}"
            k, s, st = csm.select_batch(g[f"{key}_norm"], FAM[fam], PREC[prec])
            assert np.all(st == 0)
            assert np.array_equal(k, g[f"{key}_k"].astype(np.int32)), key
            assert np.array_equal(s, g[f"{key}_s"].astype(np.int32)), key


def test_host_twin_matches_oracle_on_random_norms():
    rng = np.random.default_rng(99)
    norms = np.concatenate([10.0 ** rng.uniform(-8, 12, 200_000),
                            rng.uniform(0, 40, 100_000)])
    for fam in ("taylor", "wave"):
        k, s, st = csm.select_batch(norms, FAM[fam], csm.Precision.DOUBLE)
        want = [orc.select(float(x), fam, "double") for x in norms]
        assert np.array_equal(k, np.array([w[0] for w in want]))
        assert np.array_equal(s, np.array([w[1] for w in want]))


def test_log2_boundary_norms_exhaustive():
    """Norms whose quotient q = norm/theta sits a few ulps above 2^e: the
    glibc log2 rounding trap of driver.py:67."""
    for fam in ("taylor", "wave"):
        for prec in ("double", "single"):
            tab = csm.table_for(FAM[fam], PREC[prec])
            vals = []
            for e in tab.entries:
                for p in range(0, 60):
                    base = math.ldexp(e.theta_eff, p)
                    x = base
                    for _ in range(80):
                        vals.append(x)
                        x = math.nextafter(x, math.inf)
                    vals.append(math.nextafter(base, 0.0))
            k, s, st = csm.select_batch(vals, FAM[fam], PREC[prec])
            for x, kk, ss in zip(vals, k, s):
                assert (kk, ss) == orc.select(x, fam, prec), (fam, prec, x)


def test_select_known_answers():
    tab = csm.TAYLOR_TABLE[csm.Precision.DOUBLE]
    assert [(sch.k_products, s) for sch, s in
            (csm.select_scheme(x, tab) for x in (0.005, 0.0, 10.0))] == \
        [(3, 0), (3, 0), (7, 3)]
    for bad in (-1.0, math.inf, math.nan):
        with pytest.raises(ValueError):
            csm.select_scheme(bad, tab)


def test_select_cost_tie_prefers_fewer_squarings():
    # pkg/tests/test_driver.py:49-63
    tab = csm.ThetaTable(csm.Precision.DOUBLE, (
        csm.ThetaEntry(csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, 3),
                       1.0, 1.0, Fraction(3)),
        csm.ThetaEntry(csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, 4),
                       2.0, 2.0, Fraction(5)),
    ))
    sch, s = csm.select_scheme(4.0, tab)
    assert (sch.k_products, s) == (4, 1)


def test_select_fractional_costs():
    """Pade-style 22/3 costs are compared exactly (Fraction semantics)."""
    tab = csm.ThetaTable(csm.Precision.DOUBLE, (
        csm.ThetaEntry(csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, 3),
                       0.5, 0.5, Fraction(20, 3)),
        csm.ThetaEntry(csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, 4),
                       1.0, 1.0, Fraction(22, 3)),
    ))
    # norm 1.5: entry0 s=2 -> 20/3+4 = 32/3 ; entry1 s=1 -> 22/3+2 = 28/3
    sch, s = csm.select_scheme(1.5, tab)
    assert (sch.k_products, s) == (4, 1)


def test_select_scaling_monotone():
    tab = csm.TAYLOR_TABLE[csm.Precision.DOUBLE]
    prev = 0
    for norm in (0.001, 0.05, 0.3, 1.0, 2.5, 7.0, 31.0, 200.0, 4e3):
        _, s = csm.select_scheme(norm, tab)
        assert s >= prev
        prev = s


def test_overflowing_quotient_raises_overflow():
    tab = csm.TAYLOR_TABLE[csm.Precision.DOUBLE]
    with pytest.raises(OverflowError):
        orc.select(1.7e308)
    with pytest.raises(OverflowError):
        csm.select_scheme(1.7e308, tab)
