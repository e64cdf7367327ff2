"""CPU oracle for the cos/sin hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only tests/, the
``__graft_entry__.smoke()`` check and the ``cpu_baseline`` / ``--impl
reference`` legs of bench.py may import it.  The shipped path
(paper_2010_00465_b200) runs on the GPU through the C-ABI and fails loudly
when the CUDA library is missing.

It restates, in numpy, the reference algorithm of arXiv 2010.00465 as the
``cossinm`` package implements it (paths relative to /root/reference):

* 1-norm            pkg/src/cossinm/matcore.py:100-104
* linear comb.      pkg/src/cossinm/matcore.py:107-121  (sequential, no FMA)
* selection         pkg/src/cossinm/driver.py:64-88
* scaling/doubling  pkg/src/cossinm/driver.py:91-98, :108-146
* chains            pkg/src/cossinm/schemes.py:264-361
* trig / wave use   pkg/src/cossinm/schemes.py:376-395, :411-430
* coefficients      pkg/src/cossinm/schemes.py:51-52, :110-187
* theta tables      pkg/src/cossinm/theta_tables.py:79-144
* Pade-8 baseline   pkg/src/cossinm/schemes.py:188-200, :446-464,
                    driver.py:149-164, matcore.py:124-151

Pinning: tests/test_oracle_golden.py checks every function here against
tests/golden/*.npz and tests/golden/constants.json, which
scripts/gen_golden.py and scripts/gen_constants.py produced by importing
the reference itself in the build container.  GEMM output bits are those
of numpy's BLAS (the reference's own matmul, matcore.py:97), so on the same
machine the oracle reproduces the reference bit for bit.
"""
from __future__ import annotations

import math
from fractions import Fraction as Q

import numpy as np

# ---------------------------------------------------------------------------
# Constants (published values of the paper, restated; float() of each exact
# value is what the reference feeds its linear combinations, schemes.py:261).

_R36681 = math.sqrt(36681.0)


def _surd(p: Q, q: Q) -> float:
    # schemes.py:51-52: float(p) + float(q) * sqrt(36681.0)
    return float(p) + float(q) * _R36681


def _d(s: str) -> float:
    # exact decimal -> nearest float64 (Fraction is exact, float() rounds once)
    if "e" in s:
        m, e = s.split("e")
        return float(Q(m) * Q(10) ** int(e))
    return float(Q(s))


# degree-8 cos core x1..x8 (schemes.py:110-119)
X8 = {
    1: float(Q(7, 500)), 2: float(Q(-7, 60000)),
    3: _surd(Q(-1533, 2500), Q(7, 2500)),
    4: _surd(Q(-622905, 10594584), Q(-1955, 10594584)),
    5: float(Q(9775, 10594584)),
    6: _surd(Q(-5005, 508540032), Q(-5, 508540032)),
    7: float(Q(3125, 889945056)),
    8: _surd(Q(1549211, 63063000), Q(3246, 63063000)),
}
# degree-8 sine companion z0..z8 (schemes.py:125-135)
Z8 = {i: float(v) for i, v in enumerate([
    Q(8887, 4794), Q(-1897, 3196), Q(25259, 575280),
    Q(-965093875, 9674368704), Q(-4093, 4794), Q(25698275, 29023106112),
    Q(-3907675, 348277273344), Q(11865625, 3656911370112),
    Q(25, 308756448)])}
# degree-12 cos core: A12[j][i] multiplies y^i in c_j (schemes.py:149-166)
A12 = {
    1: [0.0, 0.0, _d("0.02264979811206039519"),
        _d("-0.00013110924142135755")],
    2: [_d("0.55751443809990408029"), _d("-0.61577924683458386455"),
        _d("0.00747198841446687051"), _d("-0.00003362444420476012")],
    3: [_d("0.75936877868464999248"), _d("-0.01560333979813817129"),
        _d("0.00010936989591908396"), _d("-1.03893360877457159499e-6")],
    4: [0.0, _d("-0.039649968743474473091"), _d("0.000155490073503821463"),
        _d("-1.126739663071170022488e-6")],
}
# degree-12 sine companion z0..z11 (schemes.py:174-187)
Z12 = [_d(s) for s in (
    "0.10090808375109885598", "-0.07668753546445299316",
    "0.00084924846993243257", "-0.00001220406904464391",
    "0.98499703159318860027", "-0.84925233648155398756", "1",
    "0.00095544138280925799", "4.56337109377154270633e-6",
    "2.73461259403000427141e-8", "0.00048550288474842477",
    "-4.15891109384923342531e-7")]

# theta_eff = min(theta_cos, theta_sin) per entry (theta_tables.py:45-47,
# :79-144); entries sorted by cost = k products.
_TH = {
    ("taylor", "double"): [(3, 0.006563322289762723, 0.01777015697577729),
                           (4, 0.11495105915204516, 0.08043801069944813),
                           (6, 0.9810763216215669, 1.118352319366378),
                           (7, 2.5674905328502904, 1.8554811337390547)],
    ("taylor", "single"): [(3, 0.18709270369684675, 0.3138563386485543),
                           (4, 0.8575551381567614, 0.7492030342174507),
                           (6, 2.9935285064988997, 3.215172177750302),
                           (7, 5.555547236845219, 4.381922344660116)],
    ("wave", "double"): [(3, 0.013213746049765359, 0.021345252850722786),
                         (4, 0.9625107503945455, 1.266344610496533),
                         (5, 6.592007661014267, 3.640429549980952)],
    ("wave", "single"): [(3, 0.7354008169503493, 1.1874758013210427),
                         (4, 8.961212972067917, 11.761988215232014),
                         (5, 30.86410513391181, 21.848395783984834)],
}
_TH[("pade", "double")] = [(5, 0.13959229566058115, 0.11212687277599737)]
_TH[("pade", "single")] = [(5, 1.021836815484684, 0.9951082066593949)]
THETA = {key: [(k, min(c, s)) for k, c, s in ents] for key, ents in _TH.items()}

# order-8 diagonal Pade of exp split into cos / sin parts, polynomials in
# y = A^2 (schemes.py:188-200)
PADE_DEN = [Q(1), Q(1, 28), Q(3, 3920), Q(1, 70560), Q(1, 2822400)]
PADE_NUM_COS = [Q(1), Q(-13, 28), Q(289, 11760), Q(-19, 70560), Q(1, 2822400)]
PADE_NUM_SIN = [Q(1), Q(-11, 84), Q(37, 11760), Q(-1, 70560)]


# ---------------------------------------------------------------------------
# Matrix core.

def norm1(a: np.ndarray) -> float:
    """max_j sum_i |a_ij| -- matcore.py:100-104 (numpy reduces axis 0 row by
    row, i.e. each column sum is a sequential accumulation in row order)."""
    if a.size == 0:
        return 0.0
    return float(np.abs(a).sum(axis=0).max())


def norm1_sequential(a: np.ndarray) -> float:
    """Explicit row-order restatement of norm1, used to pin the summation
    order the device kernel reproduces (same dtype as the input)."""
    if a.size == 0:
        return 0.0
    acc = np.zeros(a.shape[1], dtype=a.dtype)
    for row in np.abs(a):
        acc = acc + row
    return float(acc.max())


def lin(terms):
    """Sequential scalar-times-matrix sum -- matcore.py:107-121."""
    out = np.zeros(terms[0][1].shape, dtype=np.float64)
    for c, m in terms:
        out += float(c) * m
    return out


# ---------------------------------------------------------------------------
# Selection -- driver.py:64-88.

def select(norm: float, family: str = "taylor", precision: str = "double"):
    """(k, s) for one operand norm; raises like the reference."""
    if not (norm >= 0.0 and math.isfinite(norm)):
        raise ValueError(f"norm must be finite and nonnegative, got {norm}")
    table = THETA[(family, precision)]
    for k, th in table:
        if norm <= th:
            return k, 0
    best = None
    for k, th in table:
        s = 0 if norm <= th else max(0, math.ceil(math.log2(norm / th)))
        key = (k + 2 * s, s)
        if best is None or key < best[0]:
            best = (key, k, s)
    return best[1], best[2]


# ---------------------------------------------------------------------------
# Chains over dense matrices (schemes.py:264-361).  Each returns
# (cos_core, sin_core, products_used).

def _deg2(y, eye):
    y2 = y @ y
    c = lin([(1.0, eye), (-0.5, y), (float(Q(1, 24)), y2)])
    sc = lin([(1.0, eye), (float(Q(-1, 6)), y), (float(Q(1, 120)), y2)])
    return c, sc, 1


def _deg4(y, eye, exact_sine):
    y2 = y @ y
    q = y2 @ lin([(float(Q(-1, 720)), y), (float(Q(1, 40320)), y2)])
    c = lin([(1.0, eye), (-0.5, y), (float(Q(1, 24)), y2), (1.0, q)])
    base = [(1.0, eye), (float(Q(-1, 6)), y), (float(Q(1, 120)), y2)]
    if exact_sine:
        q9 = y2 @ lin([(float(Q(-1, 5040)), y), (float(Q(1, 362880)), y2)])
        return c, lin(base + [(1.0, q9)]), 3
    return c, lin(base + [(float(Q(720, 5040)), q)]), 2


def _deg8(y, eye):
    x, z = X8, Z8
    y2 = y @ y
    p8 = y2 @ lin([(x[1], y), (x[2], y2)])
    p16 = lin([(x[3], y2), (1.0, p8)]) @ lin(
        [(x[4], eye), (x[5], y), (x[6], y2), (x[7], p8)])
    c = lin([(1.0, eye), (-0.5, y), (x[8], y2), (1.0, p16)])
    inner = lin([(z[5], eye), (z[5], y), (z[6], y2), (z[7], p8), (z[8], c)])
    tail = inner @ p8
    sc = lin([(z[0], eye), (z[1], y), (z[2], y2), (z[3], p8), (z[4], c),
              (1.0, tail)])
    return c, sc, 4


def _deg12(y, eye):
    z = Z12
    y2 = y @ y
    y3 = y2 @ y
    cj = {j: lin([(A12[j][0], eye), (A12[j][1], y), (A12[j][2], y2),
                  (A12[j][3], y3)]) for j in (1, 2, 3, 4)}
    mid = lin([(1.0, cj[3]), (1.0, cj[4] @ cj[4])])
    c = lin([(1.0, cj[1]), (1.0, lin([(1.0, cj[2]), (1.0, mid)]) @ mid)])
    inner = lin([(z[6], eye), (z[7], y), (z[8], y2), (z[9], y3),
                 (z[10], mid), (z[11], c)])
    tail = inner @ c
    sc = lin([(z[0], eye), (z[1], y), (z[2], y2), (z[3], y3), (z[4], mid),
              (z[5], c), (1.0, tail)])
    return c, sc, 5


def taylor_core(a: np.ndarray, k: int):
    """cos and sin of an already-scaled a with the k-product scheme
    (schemes.py:376-395)."""
    eye = np.eye(a.shape[0])
    y = a @ a
    if k == 3:
        c, sc, _ = _deg2(y, eye)
    elif k == 4:
        c, sc, _ = _deg4(y, eye, exact_sine=False)
    elif k == 6:
        c, sc, _ = _deg8(y, eye)
    elif k == 7:
        c, sc, _ = _deg12(y, eye)
    else:
        raise ValueError(k)
    return c, a @ sc


def wave_core(a: np.ndarray, t: float, k: int):
    """c(t^2 a), s(t, a) with the k-product wave scheme (schemes.py:411-430)."""
    eye = np.eye(a.shape[0])
    y = float(t) * float(t) * a
    if k == 3:
        c, sc, _ = _deg4(y, eye, exact_sine=True)
    elif k == 4:
        c, sc, _ = _deg8(y, eye)
    elif k == 5:
        c, sc, _ = _deg12(y, eye)
    else:
        raise ValueError(k)
    return c, float(t) * sc


def taylor_sin9(a: np.ndarray):
    """Degree-9 sine alone (schemes.py:398-408): exact-sine degree-4 core."""
    eye = np.eye(a.shape[0])
    y = a @ a
    _, sc, _ = _deg4(y, eye, exact_sine=True)
    return a @ sc


def wave_sin34(a: np.ndarray, t: float):
    """Order-3 wave sine (schemes.py:433-443): inexact-sine degree-4 core."""
    eye = np.eye(a.shape[0])
    y = float(t) * float(t) * a
    _, sc, _ = _deg4(y, eye, exact_sine=False)
    return float(t) * sc


def double_angle(c, s, steps):
    """driver.py:91-98: S <- 2 S C (old C), then C <- 2 C C - I."""
    eye = np.eye(c.shape[0])
    for _ in range(steps):
        s = lin([(2.0, s @ c)])
        c = lin([(2.0, c @ c), (-1.0, eye)])
    return c, s


def _check(a):
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"matrix must be square, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ValueError("matrix entries must be finite")


def cos_sin(a: np.ndarray, precision: str = "double"):
    """driver.py:108-123 -> (cos, sin, k, s)."""
    _check(a)
    k, s = select(norm1(a), "taylor", precision)
    c, sn = taylor_core(a * 2.0 ** -s, k)
    c, sn = double_angle(c, sn, s)
    return c, sn, k, s


class SingularDenominator(RuntimeError):
    pass


def pade8_core(a: np.ndarray):
    """pade8_cos_sin (schemes.py:446-464) with lu_solve_pair
    (matcore.py:124-151): five products, one LU shared by two solves."""
    from scipy.linalg import lu_factor, lu_solve
    eye = np.eye(a.shape[0])
    y = a @ a
    y2 = y @ y
    y3 = y @ y2
    y4 = y @ y3
    powers = [eye, y, y2, y3, y4]
    den = lin([(float(c), p) for c, p in zip(PADE_DEN, powers)])
    num_c = lin([(float(c), p) for c, p in zip(PADE_NUM_COS, powers)])
    num_s = a @ lin([(float(c), p) for c, p in zip(PADE_NUM_SIN, powers)])
    lu, piv = lu_factor(den, check_finite=False)
    small = np.abs(np.diag(lu)).min()
    if small <= 1e3 * float(np.finfo(np.float64).eps) * norm1(den):
        raise SingularDenominator(f"pivot {small:.3e}")
    return (lu_solve((lu, piv), num_c, check_finite=False),
            lu_solve((lu, piv), num_s, check_finite=False))


def pade_cos_sin(a: np.ndarray, precision: str = "double"):
    """driver.py:149-164 -> (cos, sin, s); cost 22/3 + 2 s."""
    _check(a)
    _, s = select(norm1(a), "pade", precision)
    c, sn = pade8_core(a * 2.0 ** -s)
    c, sn = double_angle(c, sn, s)
    return c, sn, s


def wave_cos_sin(a: np.ndarray, t: float, precision: str = "double"):
    """driver.py:126-146 -> (c, s_part, k, s)."""
    _check(a)
    k, s = select(float(t) * float(t) * norm1(a), "wave", precision)
    c, sp = wave_core(a, float(t) / 2.0 ** s, k)
    c, sp = double_angle(c, sp, s)
    return c, sp, k, s
