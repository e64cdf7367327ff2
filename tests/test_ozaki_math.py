"""CPU checks of the Ozaki-II engine's integer arithmetic (csrc/ozaki.cuh,
oz_const in csrc/tiled.cu), restated with exact big-integer / Fraction
arithmetic: every fp64 operation the kernels perform is modelled as the exact
result rounded once to float64 (an fma rounds once, a multiply rounds once),
so these tests pin the bounds the kernels rely on -- not the kernels
themselves (those are the -m gpu tests)."""
import math
import random
from fractions import Fraction

import pytest

MODS = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]
LVB, LV = 42, 3
M52 = 6755399441055744.0  # 1.5 * 2^52


def rnd(x):
    """Round an exact rational to the nearest float64 (ties to even)."""
    return float(Fraction(x))


def fma(a, b, c):
    return rnd(Fraction(a) * Fraction(b) + Fraction(c))


def consts(nm, k):
    m = math.prod(MODS[:nm])
    log2m = sum(math.log2(x) for x in MODS[:nm])
    p = math.floor((log2m - 2.0 - math.log2(k)) / 2.0)
    mask = (1 << LVB) - 1
    w = []
    for t in range(nm):
        mt = m // MODS[t]
        inv = pow(mt % MODS[t], -1, MODS[t])
        wt = (mt * inv) % m
        w.append([float((wt >> (LVB * (LV - 1 - l))) & mask) for l in range(LV)])
    mdig = [float((m >> (LVB * (LV - 1 - l))) & mask) for l in range(LV)]
    return m, p, w, mdig, rnd(Fraction(1, m))


def test_moduli_pairwise_coprime_and_sizes():
    for i, a in enumerate(MODS):
        assert a <= 256
        for b in MODS[i + 1:]:
            assert math.gcd(a, b) == 1
    m16 = math.prod(MODS)
    assert m16 < 2 ** 126  # three 42-bit levels hold every W_t
    # P for 16 moduli: 57 / 56 / 55 at K = 256 / 1024 / 8192 (K7)
    assert [consts(16, k)[1] for k in (256, 1024, 8192)] == [57, 56, 55]
    assert consts(9, 256)[1] == 30


@pytest.mark.parametrize("nm,k", [(16, 1024), (16, 8192), (9, 256)])
def test_crt_reconstruction_is_exact(nm, k):
    """oz_crt_epi: level sums exact (< 2^53), q = round(S / M), levels
    minus q M_l, one final rounding: the product L'R' (|.| <= K 2^2P <= M/4)
    comes back correctly rounded (within 1 ulp)."""
    m, p, w, mdig, inv_m = consts(nm, k)
    assert k * 2 ** (2 * p) <= m // 4
    rng = random.Random(nm * 100003 + k)
    bound = k * 2 ** (2 * p)
    cases = [bound, -bound, 0, 1, -1] + [rng.randint(-bound, bound) for _ in range(300)]
    d1, d2 = 2.0 ** LVB, 2.0 ** (2 * LVB)
    for x in cases:
        r = []
        for mt in MODS[:nm]:
            v = x % mt
            r.append(v - mt if v > 127 else v)  # the GEMM epilogue's representative
        s = [0.0] * LV
        for t in range(nm):
            for l in range(LV):
                s[l] = fma(r[t], w[t][l], s[l])
                assert abs(s[l]) < 2.0 ** 53  # exact partial sums
        approx = fma(s[0], d2, fma(s[1], d1, s[2]))
        q = float(round(Fraction(rnd(Fraction(approx) * Fraction(inv_m)))))
        e = [fma(-q, mdig[l], s[l]) for l in range(LV)]
        assert Fraction(e[0]) == Fraction(s[0]) - Fraction(q) * Fraction(mdig[0])  # top level exact
        v = fma(e[0], d2, fma(e[1], d1, e[2]))
        assert abs(Fraction(v) - x) <= abs(Fraction(math.ulp(float(x)))) + 2 ** 45, x


def test_residue_tricks_are_exact():
    """oz_mod_group / oz_mod_small / oz_mod_acc on integer-valued doubles up
    to 2^57: the 1.5 2^52 quotient trick, the exact fma remainder, and the
    multiply-high by floor(2^32 / m) with one correction."""
    rng = random.Random(5)
    groups = [(0, 3), (3, 6), (6, 9), (9, 12), (12, 15), (15, 16)]
    vals = [0.0, 1.0, -1.0, 2.0 ** 57, -(2.0 ** 57)] + [
        float(rng.randint(-(2 ** 57), 2 ** 57) >> rng.randint(0, 56)) for _ in range(400)]
    for v in vals:
        vi = int(v)
        for lo, hi in groups:
            g = float(math.prod(MODS[lo:hi]))
            assert g < 2 ** 24
            q = rnd(Fraction(fma(v, rnd(1 / Fraction(g)), M52)) - Fraction(M52))
            rr = fma(-q, g, v)
            assert Fraction(rr) == Fraction(v) - Fraction(q) * Fraction(g)  # exact remainder
            assert abs(rr) < g
            x = int(rr) + int(g)  # __double2loint(r + M52) + G
            assert 0 <= x < 2 * int(g) < 2 ** 25
            for mt in MODS[lo:hi]:
                cdiv = (1 << 32) // mt
                r = x - ((x * cdiv) >> 32) * mt
                assert 0 <= r < 2 * mt
                if r >= mt:
                    r -= mt
                assert r == vi % mt  # the unsigned residue the GEMM consumes
    # GEMM epilogue: C_t in [0, K 255^2] with K <= 33025 stays below 2^31
    assert 33025 * 255 * 255 < 2 ** 31
    for x in [0, 1, 2 ** 31 - 1] + [rng.randint(0, 2 ** 31 - 1) for _ in range(300)]:
        for mt in MODS:
            r = x - ((x * ((1 << 32) // mt)) >> 32) * mt
            if r >= mt:
                r -= mt
            r = r - mt if r > 127 else r
            assert -128 <= r <= 127 and (r - x) % mt == 0
