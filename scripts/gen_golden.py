"""Generate golden vectors by running the REFERENCE itself (build container only).

Imports the read-only reference package from /root/reference/pkg/src and
records its outputs on seeded inputs into tests/golden/*.npz.  The oracle
(oracle/cossin_oracle.py) is pinned against these files by
tests/test_oracle_golden.py; the GPU parity tests then use the oracle.

Reference entry points exercised (paths under /root/reference):
  select_scheme  pkg/src/cossinm/driver.py:70-88
  cos_sin        pkg/src/cossinm/driver.py:108-123
  wave_cos_sin   pkg/src/cossinm/driver.py:126-146
  norm1          pkg/src/cossinm/matcore.py:100-104
  pade_cos_sin   pkg/src/cossinm/driver.py:149-164
  bench corpus   pkg/src/cossinm/gallery.py:186-220, cli.py:128-163
  acceptance     pkg/tests/test_acceptance.py:160-254 (criteria 3-5 corpus)

Usage: python scripts/gen_golden.py [acceptance]   (no argument: everything)
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, os.environ.get("COSSIN_REF_SRC", "/root/reference/pkg/src"))

import cossinm  # noqa: E402
from cossinm import Precision  # noqa: E402
from cossinm.theta_tables import PADE_TABLE, TAYLOR_TABLE, WAVE_TABLE  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden")


def selection_norms(table, rng) -> np.ndarray:
    """Random norms plus the boundary traps of driver.py:67 (log2/ceil)."""
    vals = list(10.0 ** rng.uniform(-6, 7, 3000))
    vals += [0.0, 5e-324, 1e-300, 1e300]
    for e in table.entries:
        th = e.theta_eff
        vals += [th, math.nextafter(th, 0), math.nextafter(th, math.inf)]
        for p in range(0, 45):
            base = math.ldexp(th, p)
            for j in range(0, 40):
                q = math.ldexp(1.0 + j * 2.0 ** -52, p)
                vals.append(q * th)
                vals.append(math.nextafter(base, 0))
            for j in (-3, -2, -1, 1, 2, 3):
                vals.append(base * (1.0 + j * 2.0 ** -52))
    return np.unique(np.array(vals, dtype=np.float64))


def gen_selection(rng):
    out = {}
    for fam, tabs in (("taylor", TAYLOR_TABLE), ("wave", WAVE_TABLE),
                      ("pade", PADE_TABLE)):
        for prec in (Precision.DOUBLE, Precision.SINGLE):
            tab = tabs[prec]
            norms = selection_norms(tab, rng)
            ks, ss = [], []
            for x in norms:
                scheme, s = cossinm.select_scheme(float(x), tab)
                ks.append(scheme.k_products)
                ss.append(s)
            key = f"{fam}_{prec.value}"
            out[f"{key}_norm"] = norms
            out[f"{key}_k"] = np.array(ks, dtype=np.int8)
            out[f"{key}_s"] = np.array(ss, dtype=np.int16)
    np.savez_compressed(os.path.join(OUT, "selection.npz"), **out)


def trig_cases(rng):
    cases = []
    g = np.random.default_rng(0).standard_normal((64, 64))
    cases.append(("cfg1", g * (2.0 / cossinm.norm1(g)), "double"))
    for n, target in ((1, 2.7), (2, 0.004), (3, 0.07), (4, 0.5), (5, 2.0),
                      (7, 9.0), (8, 50.0), (13, 1.3), (16, 0.9), (31, 3.3),
                      (32, 20.0), (33, 0.02), (48, 7.0), (63, 100.0),
                      (64, 0.3), (64, 31.0)):
        m = rng.standard_normal((n, n))
        cases.append((f"rand{n}_{target}", m * (target / cossinm.norm1(m)),
                      "double"))
    cases.append(("zero5", np.zeros((5, 5)), "double"))
    cases.append(("pi_diag", np.diag([math.pi, math.pi]), "double"))
    cases.append(("diag3", np.diag([0.1, -0.3, 0.55]), "double"))
    cases.append(("invol_1e4", np.array([[1.0, 1e4], [0.0, -1.0]]), "double"))
    nil = np.triu(rng.standard_normal((9, 9)), 1)
    cases.append(("nilpotent9", nil * (40.0 / cossinm.norm1(nil)), "double"))
    b = rng.standard_normal((8, 8))
    sym = b + b.T
    cases.append(("sym8_50", sym * (50.0 / cossinm.norm1(sym)), "double"))
    for n, target in ((6, 0.5), (17, 4.0), (64, 20.0), (40, 45.0)):
        m = rng.uniform(-1, 1, (n, n))
        cases.append((f"single{n}_{target}",
                      m * (target / cossinm.norm1(m)), "single"))
    return cases


def gen_trig(rng):
    out = {}
    names = []
    for name, a, prec in trig_cases(rng):
        rep = cossinm.cos_sin(a, Precision(prec))
        out[f"{name}__a"] = a
        out[f"{name}__cos"] = rep.result.cos_part
        out[f"{name}__sin"] = rep.result.sin_part
        out[f"{name}__ks"] = np.array([rep.scheme_used.k_products,
                                       rep.scaling_exponent], dtype=np.int32)
        names.append(f"{name}|{prec}")
    # float32 inputs as the reference sees them (its own mixed precision)
    for n, target in ((12, 3.0), (64, 25.0)):
        m = rng.uniform(-1, 1, (n, n))
        a32 = (m * (target / cossinm.norm1(m))).astype(np.float32)
        rep = cossinm.cos_sin(a32, Precision.SINGLE)
        name = f"f32in{n}_{target}"
        out[f"{name}__a"] = a32
        out[f"{name}__cos"] = rep.result.cos_part
        out[f"{name}__sin"] = rep.result.sin_part
        out[f"{name}__ks"] = np.array([rep.scheme_used.k_products,
                                       rep.scaling_exponent], dtype=np.int32)
        names.append(f"{name}|single")
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "trig.npz"), **out)


def gen_wave(rng):
    out = {}
    names = []
    cases = []
    for n, t in ((2, 2.0), (3, 1.3), (6, 0.05), (16, 0.7), (32, 0.01),
                 (64, 0.002)):
        b = rng.standard_normal((n, n))
        a = b @ b.T + 0.5 * np.eye(n)
        cases.append((f"spd{n}_{t}", a, t, "double"))
    cases.append(("diag4_t2", np.diag([4.0, 4.0]), 2.0, "double"))
    cases.append(("diag_small", np.diag([0.25, 0.01]), 1.0, "double"))
    cases.append(("zero4", np.zeros((4, 4)), 0.7, "double"))
    cases.append(("t0", rng.standard_normal((3, 3)), 0.0, "double"))
    cases.append(("neg", np.diag([-0.49]), 1.0, "double"))
    n = 48
    lap = (np.diag(2.0 * np.ones(n)) - np.diag(np.ones(n - 1), 1)
           - np.diag(np.ones(n - 1), -1)) * (n + 1) ** 2
    cases.append(("lap48", lap + np.diag(rng.uniform(0, 10, n)), 3e-3,
                  "double"))
    cases.append(("lap48_single", lap + np.diag(rng.uniform(0, 10, n)), 1e-2,
                  "single"))
    for name, a, t, prec in cases:
        rep = cossinm.wave_cos_sin(a, t, Precision(prec))
        out[f"{name}__a"] = a
        out[f"{name}__t"] = np.array(t)
        out[f"{name}__c"] = rep.result.c_part
        out[f"{name}__s"] = rep.result.s_part
        out[f"{name}__ks"] = np.array([rep.scheme_used.k_products,
                                       rep.scaling_exponent], dtype=np.int32)
        names.append(f"{name}|{prec}")
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "wave.npz"), **out)


def gen_norms(rng):
    """norm1 bits on shapes/dtypes whose column sums exercise the order."""
    out = {}
    for i, (n, dt) in enumerate(((3, np.float64), (64, np.float64),
                                 (257, np.float64), (64, np.float32),
                                 (300, np.float32))):
        a = (rng.standard_normal((n, n)) * 10.0 ** rng.uniform(-3, 3, (n, n)))
        a = a.astype(dt)
        out[f"a{i}"] = a
        out[f"n{i}"] = np.array(cossinm.norm1(a))
    np.savez_compressed(os.path.join(OUT, "norm1.npz"), **out)


def gen_extras(rng):
    """taylor_sin9 (schemes.py:398-408) and wave_sin34 (schemes.py:433-443)."""
    from cossinm import CostLedger, taylor_sin9, wave_sin34
    out = {}
    names = []
    for n, target in ((1, 0.3), (4, 0.05), (9, 0.4), (33, 0.2), (64, 0.1), (80, 0.15)):
        m = rng.standard_normal((n, n))
        a = m * (target / cossinm.norm1(m))
        led = CostLedger()
        out[f"sin9_{n}__a"] = a
        out[f"sin9_{n}__out"] = taylor_sin9(a, led)
        out[f"sin9_{n}__cost"] = np.array(int(led.total_cost))
        names.append(f"sin9_{n}")
        t = 0.7
        led = CostLedger()
        out[f"sin34_{n}__a"] = a
        out[f"sin34_{n}__t"] = np.array(t)
        out[f"sin34_{n}__out"] = wave_sin34(a, t, led)
        out[f"sin34_{n}__cost"] = np.array(int(led.total_cost))
        names.append(f"sin34_{n}")
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "extras.npz"), **out)


def gen_ddref(rng):
    """reference_cos_sin (verify.py:480-521), _dd_matmul (:449-459) and the
    _dd_const splits (:462-464) of the series coefficients."""
    from cossinm import verify as V
    out = {}
    names = []
    cases = [("one", np.array([[0.3]])), ("zero4", np.zeros((4, 4)))]
    for n, target in ((5, 2.0), (16, 30.0), (33, 1e-7), (40, 0.5),
                      (64, 4.0), (70, 11.0)):
        m = rng.standard_normal((n, n))
        cases.append((f"r{n}_{target}", m * (target / cossinm.norm1(m))))
    nanm = rng.standard_normal((3, 3))
    nanm[1, 2] = np.nan
    cases.append(("nan3", nanm))
    for name, a in cases:
        res = V.reference_cos_sin(a)
        out[f"{name}__a"] = a
        out[f"{name}__cos"] = res.cos_part
        out[f"{name}__sin"] = res.sin_part
        out[f"{name}__cost"] = np.array(int(res.cost.total_cost))
        names.append(name)
    out["names"] = np.array(names)
    for n in (1, 7, 40, 65):
        xh = rng.standard_normal((n, n))
        xl = xh * 1e-17 * rng.standard_normal((n, n))
        yh = rng.standard_normal((n, n)) * 10.0 ** rng.uniform(-5, 5, (n, n))
        yl = yh * 1e-17 * rng.standard_normal((n, n))
        oh, ol = V._dd_matmul(xh, xl, yh, yl)
        for k, v in (("xh", xh), ("xl", xl), ("yh", yh), ("yl", yl),
                     ("oh", oh), ("ol", ol)):
            out[f"mm{n}__{k}"] = v
    consts = [V._dd_const(c) for c in V._REF_COS_CORE + V._REF_SIN_CORE]
    out["consts"] = np.array(consts)
    np.savez_compressed(os.path.join(OUT, "ddref.npz"), **out)


def gen_pade(rng):
    """pade_cos_sin (driver.py:149-164) on seeded inputs, both tables."""
    out = {}
    names = []
    cases = []
    for n, target in ((1, 0.05), (3, 0.5), (8, 2.0), (16, 0.11), (33, 7.0),
                      (64, 2.0), (65, 30.0), (80, 0.9)):
        m = rng.standard_normal((n, n))
        cases.append((f"p{n}_{target}", m * (target / cossinm.norm1(m)), "double"))
    cases.append(("pzero4", np.zeros((4, 4)), "double"))
    for n, target in ((12, 3.0), (40, 20.0)):
        m = rng.uniform(-1, 1, (n, n))
        cases.append((f"psingle{n}_{target}", m * (target / cossinm.norm1(m)), "single"))
    for name, a, prec in cases:
        rep = cossinm.pade_cos_sin(a, Precision(prec))
        out[f"{name}__a"] = a
        out[f"{name}__cos"] = rep.result.cos_part
        out[f"{name}__sin"] = rep.result.sin_part
        out[f"{name}__s"] = np.array(rep.scaling_exponent)
        out[f"{name}__cost"] = np.array([rep.total_products.numerator,
                                         rep.total_products.denominator])
        names.append(f"{name}|{prec}")
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "pade.npz"), **out)


def gen_corpus():
    """The reference's own bench corpus (gallery.py:186-220) at a small spec,
    with its per-matrix (k, s, products) for cos_sin and pade_cos_sin and
    its errors against reference_cos_sin (cli.py:128-163)."""
    from cossinm.gallery import CorpusSpec, generate_corpus
    from cossinm.verify import reference_cos_sin, relative_error_2
    spec = CorpusSpec(dimension_cap=16, count_per_class=(24, 24, 12, 9), seed=0)
    mats, tags, dims = [], [], []
    rec = {k: [] for k in ("t_k", "t_s", "t_prod", "t_ec", "t_es", "p_s", "p_prod",
                           "p_ec", "p_es")}
    for m, tag in generate_corpus(spec):
        mats.append(m.ravel())
        tags.append(tag)
        dims.append(m.shape[0])
        with np.errstate(over="ignore", invalid="ignore"):
            ref = reference_cos_sin(m)
            t = cossinm.cos_sin(m)
            p = cossinm.pade_cos_sin(m)
        rec["t_k"].append(t.scheme_used.k_products)
        rec["t_s"].append(t.scaling_exponent)
        rec["t_prod"].append(float(t.total_products))
        rec["t_ec"].append(relative_error_2(t.result.cos_part, ref.cos_part))
        rec["t_es"].append(relative_error_2(t.result.sin_part, ref.sin_part))
        rec["p_s"].append(p.scaling_exponent)
        rec["p_prod"].append(float(p.total_products))
        rec["p_ec"].append(relative_error_2(p.result.cos_part, ref.cos_part))
        rec["p_es"].append(relative_error_2(p.result.sin_part, ref.sin_part))
    out = {"data": np.concatenate(mats), "dims": np.array(dims), "tags": np.array(tags)}
    out.update({k: np.array(v) for k, v in rec.items()})
    np.savez_compressed(os.path.join(OUT, "corpus.npz"), **out)


def gen_acceptance():
    """The corpus of the reference's acceptance criteria 3-5
    (pkg/tests/test_acceptance.py:160-184: 500 entries, classes
    162/220/109/9, norms in (1e-4, 1e4), seed 0) with the reference's own
    per-entry Taylor / Pade (k, s, products) and spectral-norm errors against
    reference_cos_sin, i.e. everything criteria 3-5 (:187-254) evaluate."""
    from cossinm.gallery import CorpusSpec, generate_corpus
    from cossinm.matcore import norm1
    from cossinm.verify import reference_cos_sin, relative_error_2
    spec = CorpusSpec(count_per_class=(162, 220, 109, 9), norm_range=(1e-4, 1e4), seed=0)
    mats, tags, dims = [], [], []
    rec = {k: [] for k in ("norm", "t_k", "t_s", "t_prod", "t_ec", "t_es", "p_s", "p_prod",
                           "p_ec", "p_es")}
    for m, tag in generate_corpus(spec):
        mats.append(m.ravel())
        tags.append(tag)
        dims.append(m.shape[0])
        with np.errstate(over="ignore", invalid="ignore"):
            ref = reference_cos_sin(m)
            t = cossinm.cos_sin(m)
            p = cossinm.pade_cos_sin(m)
        rec["norm"].append(norm1(m))
        rec["t_k"].append(t.scheme_used.k_products)
        rec["t_s"].append(t.scaling_exponent)
        rec["t_prod"].append(float(t.total_products))
        rec["t_ec"].append(relative_error_2(t.result.cos_part, ref.cos_part))
        rec["t_es"].append(relative_error_2(t.result.sin_part, ref.sin_part))
        rec["p_s"].append(p.scaling_exponent)
        rec["p_prod"].append(float(p.total_products))
        rec["p_ec"].append(relative_error_2(p.result.cos_part, ref.cos_part))
        rec["p_es"].append(relative_error_2(p.result.sin_part, ref.sin_part))
    out = {"data": np.concatenate(mats), "dims": np.array(dims), "tags": np.array(tags)}
    out.update({k: np.array(v) for k, v in rec.items()})
    np.savez_compressed(os.path.join(OUT, "acceptance_corpus.npz"), **out)


def main():
    os.makedirs(OUT, exist_ok=True)
    if sys.argv[1:] == ["acceptance"]:
        gen_acceptance()
        return
    rng = np.random.default_rng(20100465)
    gen_selection(rng)
    gen_trig(rng)
    gen_wave(rng)
    gen_norms(rng)
    gen_extras(np.random.default_rng(77))
    gen_ddref(np.random.default_rng(2010))
    gen_pade(np.random.default_rng(88))
    gen_corpus()
    gen_acceptance()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
