"""Pin the CPU oracle against golden vectors produced by the reference itself.

tests/golden/*.npz come from scripts/gen_golden.py, which imports the
reference package (pkg/src/cossinm) in the build container and records its
select_scheme / cos_sin / wave_cos_sin / norm1 outputs.  The oracle must
reproduce (k, s) and norm1 bit for bit, and the matrix outputs to within
a few ulps of BLAS reordering (it runs the same numpy calls, so on the
same machine it is normally bit-exact).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import cossin_oracle as orc


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name), allow_pickle=False)


def rel1(x, ref):
    d = orc.norm1(x - ref)
    r = orc.norm1(ref)
    return d / r if r > 0 else d


def test_constants_match_reference_bits(golden_dir):
    doc = json.load(open(os.path.join(golden_dir, "constants.json")))
    for i in range(1, 9):
        assert orc.X8[i] == float.fromhex(doc["x_deg8"][str(i)]), i
    for i in range(9):
        assert orc.Z8[i] == float.fromhex(doc["z_deg8"][str(i)]), i
    for j in (1, 2, 3, 4):
        for i in range(4):
            assert orc.A12[j][i] == float.fromhex(doc["a_deg12"][f"{i},{j}"])
    for i in range(12):
        assert orc.Z12[i] == float.fromhex(doc["z_deg12"][str(i)]), i
    for key, ents in doc["tables"].items():
        fam, prec = key.split("_")
        mine = orc.THETA[(fam, prec)]
        assert [k for k, _ in mine] == [e["k"] for e in ents]
        assert [th for _, th in mine] == [float.fromhex(e["theta_eff"])
                                          for e in ents]


def test_log2_fix_table_matches_libm(golden_dir):
    """The fix-up table the device uses reproduces math.log2 + ceil."""
    doc = json.load(open(os.path.join(golden_dir, "constants.json")))
    fix = doc["log2_fix"]
    rng = np.random.default_rng(5)
    for e in list(range(0, 80)) + list(rng.integers(80, 1023, 40)):
        e = int(e)
        J = fix[e]
        for j in sorted({0, 1, 2, J, J + 1, J + 2, max(J - 1, 0)}):
            q = math.ldexp(1.0 + j * 2.0 ** -52, e)
            want = math.ceil(math.log2(q))
            got = e if (j == 0 or j <= J) else e + 1
            assert got == want, (e, j, J)


def test_selection_matches_reference(golden_dir):
    g = _load(golden_dir, "selection.npz")
    for fam in ("taylor", "wave"):
        for prec in ("double", "single"):
            key = f"{fam}_{prec}"
            norms, ks, ss = g[f"{key}_norm"], g[f"{key}_k"], g[f"{key}_s"]
            for x, k, s in zip(norms, ks, ss):
                assert orc.select(float(x), fam, prec) == (int(k), int(s)), x


def test_select_known_answers():
    # pkg/tests/test_driver.py:27-40, :97-104
    assert orc.select(0.005) == (3, 0)
    assert orc.select(0.0) == (3, 0)
    assert orc.select(10.0) == (7, 3)
    assert orc.select(math.pi) == (7, 1)
    for bad in (-1.0, math.inf, math.nan):
        with pytest.raises(ValueError):
            orc.select(bad)


def test_norm1_bits(golden_dir):
    g = _load(golden_dir, "norm1.npz")
    i = 0
    while f"a{i}" in g:
        a = g[f"a{i}"]
        assert orc.norm1(a) == float(g[f"n{i}"])
        assert orc.norm1_sequential(a) == float(g[f"n{i}"])
        i += 1


def test_trig_outputs_match_reference(golden_dir):
    g = _load(golden_dir, "trig.npz")
    for entry in g["names"]:
        name, prec = str(entry).split("|")
        a = g[f"{name}__a"]
        c, s, k, sc = orc.cos_sin(a, prec)
        assert (k, sc) == tuple(int(v) for v in g[f"{name}__ks"]), name
        assert rel1(c, g[f"{name}__cos"]) <= 1e-14, name
        assert rel1(s, g[f"{name}__sin"]) <= 1e-14 or orc.norm1(s) < 1e-300


def test_wave_outputs_match_reference(golden_dir):
    g = _load(golden_dir, "wave.npz")
    for entry in g["names"]:
        name, prec = str(entry).split("|")
        a, t = g[f"{name}__a"], float(g[f"{name}__t"])
        c, s, k, sc = orc.wave_cos_sin(a, t, prec)
        assert (k, sc) == tuple(int(v) for v in g[f"{name}__ks"]), name
        assert rel1(c, g[f"{name}__c"]) <= 1e-14, name
        assert rel1(s, g[f"{name}__s"]) <= 1e-14 or orc.norm1(s) < 1e-300


def test_bitwise_identities():
    # pkg/tests/test_schemes.py:69-110 restated through the driver
    c, s, k, sc = orc.cos_sin(np.zeros((3, 3)))
    assert np.array_equal(c, np.eye(3)) and np.array_equal(s, np.zeros((3, 3)))
    c, s, _, _ = orc.wave_cos_sin(np.zeros((4, 4)), 0.7)
    assert np.array_equal(c, np.eye(4)) and np.array_equal(s, 0.7 * np.eye(4))
    d = np.diag([0.1, -0.3, 0.55])
    c, s, _, _ = orc.cos_sin(d)
    off = ~np.eye(3, dtype=bool)
    assert np.all(c[off] == 0.0) and np.all(s[off] == 0.0)


def test_standalone_sines_match_reference(golden_dir):
    """taylor_sin9 / wave_sin34 (schemes.py:398-408, :433-443) and their
    ledger charges (5 and 2 products)."""
    d = _load(golden_dir, "extras.npz")
    for name in d["names"]:
        name = str(name)
        a = d[f"{name}__a"]
        if name.startswith("sin9"):
            got = orc.taylor_sin9(a)
            assert int(d[f"{name}__cost"]) == 5
        else:
            got = orc.wave_sin34(a, float(d[f"{name}__t"]))
            assert int(d[f"{name}__cost"]) == 2
        assert rel1(got, d[f"{name}__out"]) <= 1e-14, name


def _bits_equal(x, y):
    """Bitwise equality, any NaN matching any NaN (payloads are platform
    dependent: x86 and the GPU produce different quiet-NaN encodings)."""
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    if x.shape != y.shape:
        return False
    nx, ny = np.isnan(x), np.isnan(y)
    return bool((nx == ny).all() and
                (x[~nx].view(np.uint64) == y[~ny].view(np.uint64)).all())


def test_ddref_oracle_bit_exact_with_reference(golden_dir):
    """oracle/ddref_oracle.py against verify.py:417-521 outputs."""
    from oracle import ddref_oracle as ddo
    d = _load(golden_dir, "ddref.npz")
    consts = [ddo.dd_const(c) for c in ddo.COS_CORE + ddo.SIN_CORE]
    assert _bits_equal(np.array(consts), d["consts"])
    for n in (1, 7, 40, 65):
        g = {k: d[f"mm{n}__{k}"] for k in ("xh", "xl", "yh", "yl", "oh", "ol")}
        oh, ol = ddo.dd_matmul(g["xh"], g["xl"], g["yh"], g["yl"])
        assert _bits_equal(oh, g["oh"]) and _bits_equal(ol, g["ol"]), n
    for name in d["names"]:
        name = str(name)
        c, s, sc = ddo.reference_cos_sin(d[f"{name}__a"])
        assert int(d[f"{name}__cost"]) == 7 + 2 * sc, name
        assert _bits_equal(c, d[f"{name}__cos"]), name
        assert _bits_equal(s, d[f"{name}__sin"]), name


def test_pade_oracle_matches_reference(golden_dir):
    """pade_cos_sin (driver.py:149-164): s exact, cost 22/3 + 2 s, values
    within BLAS/LAPACK reordering of the reference's own outputs."""
    import json
    from fractions import Fraction
    doc = json.load(open(os.path.join(golden_dir, "constants.json")))
    for key, mine in (("den", orc.PADE_DEN), ("num_cos", orc.PADE_NUM_COS),
                      ("num_sin", orc.PADE_NUM_SIN)):
        assert [float(v) for v in mine] == [float.fromhex(h) for h in doc["pade8"][key]]
    d = _load(golden_dir, "pade.npz")
    for entry in d["names"]:
        name, prec = str(entry).split("|")
        c, s, sc = orc.pade_cos_sin(d[f"{name}__a"], prec)
        assert sc == int(d[f"{name}__s"]), name
        num, den = (int(v) for v in d[f"{name}__cost"])
        assert Fraction(num, den) == Fraction(22, 3) + 2 * sc
        assert rel1(c, d[f"{name}__cos"]) <= 1e-13, name
        ref_s = d[f"{name}__sin"]
        if orc.norm1(ref_s) > 0:
            assert rel1(s, ref_s) <= 1e-13, name


def test_oracle_selection_on_the_acceptance_corpus(golden_dir):
    """The oracle's (k, s) for Taylor and s for Pade on the reference's
    500-entry acceptance corpus (pkg/tests/test_acceptance.py:160-184) equal
    the reference's own (tests/golden/acceptance_corpus.npz)."""
    d = np.load(os.path.join(golden_dir, "acceptance_corpus.npz"))
    off = 0
    for i, n in enumerate(d["dims"]):
        a = d["data"][off:off + n * n].reshape(n, n)
        off += n * n
        nrm = orc.norm1(a)
        assert nrm == float(d["norm"][i])
        k, s = orc.select(nrm, "taylor", "double")
        assert (k, s) == (int(d["t_k"][i]), int(d["t_s"][i])), i
        assert orc.select(nrm, "pade", "double")[1] == int(d["p_s"][i]), i
