"""GPU parity: the sm_100a path against the CPU oracle (pinned to the
reference's golden vectors) on the same seeded inputs.

Bars (BASELINE.json north_star): (k, s) bit-exact; relative 1-norm
difference <= 1e-12 for float64 and <= 1e-5 for float32; the Pythagorean
residual ||C^2 + S^2 - I||_1 is checked loosely (it is a float64 floor that
grows with ||cos||), never as the parity gate.
"""
import math
import os

import numpy as np
import pytest

import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc
from tests._util import cfg2_like, cfg3_like, laplacian_wave, pair_close, rel1

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5


def _golden(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def test_cfg1_matrix(cuda):
    """configs[0]: one 64x64 N(0,1) matrix rescaled to 1-norm 2."""
    g = np.random.default_rng(0).standard_normal((64, 64))
    a = g * (2.0 / orc.norm1(g))
    rep = csm.cos_sin(a)
    c, s, k, sc = orc.cos_sin(a)
    assert (rep.scheme_used.k_products, rep.scaling_exponent) == (k, sc) == (7, 1)
    assert rep.total_products == 9
    assert rel1(rep.result.cos_part, c) <= TOL64
    assert rel1(rep.result.sin_part, s) <= TOL64


def test_golden_trig_cases(cuda, golden_dir):
    g = _golden(golden_dir, "trig.npz")
    for entry in g["names"]:
        name, prec = str(entry).split("|")
        a = g[f"{name}__a"]
        rep = csm.cos_sin(a, csm.Precision(prec))
        k, s = (int(v) for v in g[f"{name}__ks"])
        assert (rep.scheme_used.k_products, rep.scaling_exponent) == (k, s), name
        assert rep.total_products == k + 2 * s
        tol = TOL64 if a.dtype == np.float64 else TOL32
        ref_c, ref_s = g[f"{name}__cos"], g[f"{name}__sin"]
        assert pair_close(rep.result.cos_part, ref_c, ref_s, tol)[0], name
        if orc.norm1(ref_s) > 0:
            assert pair_close(rep.result.sin_part, ref_s, ref_c, tol)[0], name
        else:
            assert np.array_equal(rep.result.sin_part, ref_s), name


def test_golden_wave_cases(cuda, golden_dir):
    g = _golden(golden_dir, "wave.npz")
    for entry in g["names"]:
        name, prec = str(entry).split("|")
        a, t = g[f"{name}__a"], float(g[f"{name}__t"])
        rep = csm.wave_cos_sin(a, t, csm.Precision(prec))
        k, s = (int(v) for v in g[f"{name}__ks"])
        assert (rep.scheme_used.k_products, rep.scaling_exponent) == (k, s), name
        ref_c, ref_s = g[f"{name}__c"], g[f"{name}__s"]
        assert pair_close(rep.result.c_part, ref_c, ref_s, TOL64)[0], name
        if orc.norm1(ref_s) > 0:
            assert pair_close(rep.result.s_part, ref_s, ref_c, TOL64)[0], name
        else:
            assert np.array_equal(rep.result.s_part, ref_s), name


def test_bitwise_identities(cuda):
    # pkg/tests/test_driver.py:89-94, test_schemes.py:69-110
    rep = csm.cos_sin(np.zeros((3, 3)))
    assert np.array_equal(rep.result.cos_part, np.eye(3))
    assert np.array_equal(rep.result.sin_part, np.zeros((3, 3)))
    assert rep.total_products == 3
    rep = csm.wave_cos_sin(np.zeros((4, 4)), 0.7)
    assert np.array_equal(rep.result.c_part, np.eye(4))
    assert np.array_equal(rep.result.s_part, 0.7 * np.eye(4))
    rng = np.random.default_rng(3)
    for k in (3, 4, 5):
        out = csm.wave_kernels(rng.standard_normal((3, 3)), 0.0,
                               csm.SchemeId(csm.SchemeFamily.WAVE_KERNEL, k),
                               csm.CostLedger())
        assert np.array_equal(out.c_part, np.eye(3))
        assert np.array_equal(out.s_part, np.zeros((3, 3)))
    d = np.diag([0.1, -0.3, 0.55])
    off = ~np.eye(3, dtype=bool)
    for k in (3, 4, 6, 7):
        out = csm.taylor_cos_sin(d, csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, k),
                                 csm.CostLedger())
        assert np.all(out.cos_part[off] == 0.0) and np.all(out.sin_part[off] == 0.0)
        if k >= 6:
            for i, x in enumerate(np.diag(d)):
                assert out.cos_part[i, i] == pytest.approx(math.cos(x), abs=1e-15)
                assert out.sin_part[i, i] == pytest.approx(math.sin(x), abs=1e-15)


def test_scheme_cores_match_oracle(cuda, rng):
    """taylor_cos_sin / wave_kernels per k, fixed scheme, no scaling."""
    for n in (5, 64, 100):
        a = rng.standard_normal((n, n))
        a *= 0.8 / orc.norm1(a)
        for k in (3, 4, 6, 7):
            led = csm.CostLedger()
            out = csm.taylor_cos_sin(a, csm.SchemeId(csm.SchemeFamily.COS_SIN_TAYLOR, k), led)
            c, s = orc.taylor_core(a, k)
            assert led.total_cost == k
            assert rel1(out.cos_part, c) <= TOL64, (n, k)
            assert rel1(out.sin_part, s) <= TOL64, (n, k)
        for k in (3, 4, 5):
            led = csm.CostLedger()
            out = csm.wave_kernels(a, 0.9, csm.SchemeId(csm.SchemeFamily.WAVE_KERNEL, k), led)
            c, s = orc.wave_core(a, 0.9, k)
            assert led.total_cost == k
            assert rel1(out.c_part, c) <= TOL64, (n, k)
            assert rel1(out.s_part, s) <= TOL64, (n, k)


def test_standalone_sines_golden(cuda, golden_dir):
    """taylor_sin9 / wave_sin34 (schemes.py:398-408, :433-443) against the
    reference's own outputs, ledger charges 5 and 2."""
    g = _golden(golden_dir, "extras.npz")
    for name in g["names"]:
        name = str(name)
        a = g[f"{name}__a"]
        led = csm.CostLedger()
        if name.startswith("sin9"):
            got = csm.taylor_sin9(a, led)
        else:
            got = csm.wave_sin34(a, float(g[f"{name}__t"]), led)
        assert led.total_cost == int(g[f"{name}__cost"]), name
        assert got.shape == a.shape and got.dtype == np.float64
        assert rel1(got, g[f"{name}__out"]) <= TOL64, name


@pytest.mark.parametrize("n", [64, 130, 256])
def test_standalone_sines_match_oracle(cuda, rng, n):
    a = rng.standard_normal((n, n))
    a *= 0.3 / orc.norm1(a)
    assert rel1(csm.taylor_sin9(a, csm.CostLedger()), orc.taylor_sin9(a)) <= TOL64
    got = csm.wave_sin34(a, 1.7, csm.CostLedger())
    assert rel1(got, orc.wave_sin34(a, 1.7)) <= TOL64
    a32 = a.astype(np.float32)
    got = csm.taylor_sin9(a32, csm.CostLedger())
    assert got.dtype == np.float64
    assert rel1(got, orc.taylor_sin9(a32.astype(np.float64))) <= TOL64


def test_batched_cfg2_distribution(cuda):
    """configs[1] distribution (64x64, norms 1e-3..1e2), 512 matrices."""
    rng = np.random.default_rng(11)
    a = cfg2_like(rng, 512)
    rep = csm.cos_sin_batched(a)
    worst = 0.0
    for i in range(a.shape[0]):
        c, s, k, sc = orc.cos_sin(a[i])
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc), i
        worst = max(worst, rel1(rep.cos_part[i], c), rel1(rep.sin_part[i], s))
    assert worst <= TOL64, worst


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 16, 17, 33, 63])
def test_batched_small_orders(cuda, n):
    rng = np.random.default_rng(100 + n)
    a = cfg2_like(rng, 24, n=n, lo=-3, hi=1.5)
    rep = csm.cos_sin_batched(a)
    for i in range(a.shape[0]):
        c, s, k, sc = orc.cos_sin(a[i])
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc)
        assert rel1(rep.cos_part[i], c) <= TOL64
        assert rel1(rep.sin_part[i], s) <= TOL64


@pytest.mark.parametrize("n", [65, 96, 128, 200, 256])
def test_batched_tiled_orders(cuda, n):
    rng = np.random.default_rng(200 + n)
    a = cfg2_like(rng, 12, n=n, lo=-3, hi=1.7)
    rep = csm.cos_sin_batched(a)
    for i in range(a.shape[0]):
        c, s, k, sc = orc.cos_sin(a[i])
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc)
        assert rel1(rep.cos_part[i], c) <= TOL64, (n, i)
        assert rel1(rep.sin_part[i], s) <= TOL64, (n, i)


@pytest.mark.parametrize("n", [66, 99, 127])
def test_cluster_kernel_orders(cuda, n):
    """64 < n <= 128 runs on the 4-CTA cluster kernel (K1c): partial last
    bands, odd n (unaligned bands take the synchronous staging path)."""
    rng = np.random.default_rng(250 + n)
    a = cfg2_like(rng, 10, n=n, lo=-3, hi=2.0)
    rep = csm.cos_sin_batched(a)
    for i in range(a.shape[0]):
        c, s, k, sc = orc.cos_sin(a[i])
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc)
        assert rel1(rep.cos_part[i], c) <= TOL64, (n, i)
        assert rel1(rep.sin_part[i], s) <= TOL64, (n, i)


def test_cluster_kernel_many_turns(cuda):
    """More matrices than clusters: every cluster walks several turns of the
    snake schedule, with s = 0 matrices (direct stores) mixed in."""
    rng = np.random.default_rng(260)
    a = cfg2_like(rng, 300, n=128, lo=-4, hi=2.0)
    rep = csm.cos_sin_batched(a)
    for i in list(range(0, 300, 23)) + [299]:
        c, s, k, sc = orc.cos_sin(a[i])
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc)
        assert rel1(rep.cos_part[i], c) <= TOL64, i
        assert rel1(rep.sin_part[i], s) <= TOL64, i
    assert (rep.s == 0).any() and (rep.s > 3).any()


def test_cluster_kernel_with_side_chain(cuda):
    """A batch large enough that the tail runs on the concurrent side tiled
    chain (the SMs K1c's 4-SM clusters leave idle): both parts correct,
    float32 storage too."""
    rng = np.random.default_rng(270)
    a = cfg2_like(rng, 1100, n=100, lo=-3, hi=2.0)
    rep = csm.cos_sin_batched(a)
    for i in list(range(0, 1100, 97)) + list(range(1020, 1100, 9)) + [1099]:
        c, s, k, sc = orc.cos_sin(a[i])
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc), i
        assert rel1(rep.cos_part[i], c) <= TOL64, i
        assert rel1(rep.sin_part[i], s) <= TOL64, i
    a32 = cfg3_like(rng, 1030, n=128)
    rep = csm.cos_sin_batched(a32, csm.Precision.SINGLE)
    for i in (0, 500, 1000, 1029):
        c, s, k, sc = orc.cos_sin(a32[i], "single")
        assert rel1(rep.cos_part[i], c) <= TOL32, i
        assert rel1(rep.sin_part[i], s) <= TOL32, i
    aw, tw = laplacian_wave(rng, 1040, 112)
    rep = csm.wave_cos_sin_batched(aw, tw)
    for i in (0, 520, 1000, 1039):
        c, s, k, sc = orc.wave_cos_sin(aw[i], tw[i])
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc), i
        assert pair_close(rep.cos_part[i], c, s, TOL64)[0], i
        assert pair_close(rep.sin_part[i], s, c, TOL64)[0], i


@pytest.mark.parametrize("n", [64, 99, 128, 256])
def test_batched_float32(cuda, n):
    """configs[2] variant: float32 storage, float64 compute, SINGLE table."""
    rng = np.random.default_rng(300 + n)
    a32 = cfg3_like(rng, 16, n=n)
    rep = csm.cos_sin_batched(a32, csm.Precision.SINGLE)
    assert rep.cos_part.dtype == np.float32
    for i in range(a32.shape[0]):
        c, s, k, sc = orc.cos_sin(a32[i], "single")           # reference as-is
        c64, s64, _, _ = orc.cos_sin(a32[i].astype(np.float64), "single")
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc)
        assert rel1(rep.cos_part[i], c) <= TOL32
        assert rel1(rep.sin_part[i], s) <= TOL32
        assert rel1(rep.cos_part[i], c64) <= TOL32
        assert rel1(rep.sin_part[i], s64) <= TOL32


@pytest.mark.parametrize("n", [48, 100, 130])
def test_batched_wave_laplacian(cuda, n):
    """configs[3] family (SPD Laplacian + potential), smaller n."""
    rng = np.random.default_rng(400 + n)
    a, t = laplacian_wave(rng, 8, n)
    rep = csm.wave_cos_sin_batched(a, t)
    for i in range(a.shape[0]):
        c, s, k, sc = orc.wave_cos_sin(a[i], t[i])
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc)
        assert rel1(rep.cos_part[i], c) <= TOL64, (n, i, sc)
        assert rel1(rep.sin_part[i], s) <= TOL64, (n, i, sc)


def test_device_tensors_in_and_out(cuda):
    import torch
    rng = np.random.default_rng(5)
    a = cfg2_like(rng, 8)
    ad = torch.from_numpy(a).to(cuda)
    rep = csm.cos_sin_batched(ad)
    assert rep.cos_part.is_cuda and rep.k.is_cuda
    ref = csm.cos_sin_batched(a)
    assert np.array_equal(rep.cos_part.cpu().numpy(), ref.cos_part)
    assert np.array_equal(rep.sin_part.cpu().numpy(), ref.sin_part)


def test_input_errors(cuda):
    with pytest.raises(csm.MatrixInputError):
        csm.cos_sin(np.zeros((2, 3)))
    with pytest.raises(csm.MatrixInputError):
        csm.cos_sin(np.array([[math.inf, 0.0], [0.0, 0.0]]))
    with pytest.raises(csm.MatrixInputError):
        csm.wave_cos_sin(np.array([[math.nan]]), 1.0)
    with pytest.raises(ValueError):  # column sum overflows to inf
        csm.cos_sin(np.full((2, 2), 1e308))
    with pytest.raises(OverflowError):  # norm / theta overflows
        csm.cos_sin(np.diag([1.7e308, 0.0]))
    a = np.stack([np.eye(3), np.eye(3)])
    a[1, 0, 0] = math.nan
    rep = csm.cos_sin_batched(a, raise_on_error=False)
    assert list(rep.status) == [0, 1]
    assert np.all(np.isnan(rep.cos_part[1]))


@pytest.mark.parametrize("n,count", [(100, 40), (128, 1200), (300, 12)])
def test_bad_statuses_on_every_path(cuda, n, count):
    """Non-finite entries, infinite norms and norm/theta overflow inside a
    batch on K1c, K1c + side chain and the tiled chain: those matrices get
    their status and NaN outputs, their neighbours stay exact."""
    rng = np.random.default_rng(600 + n)
    a = cfg2_like(rng, count, n=n, lo=-2, hi=1.0)
    bad = {1: 1, count - 2: 1, count // 2: 2, count - 1: 3}
    a[1, 3, 5] = math.nan
    a[count - 2, 0, 0] = math.inf
    a[count // 2, :, 0] = 1e308  # column sum overflows: non-finite norm
    a[count - 1] = 0.0
    a[count - 1, 0, 0] = 1.7e308  # finite norm, norm / theta overflows
    rep = csm.cos_sin_batched(a, raise_on_error=False)
    st = np.asarray(rep.status)
    for i, code in bad.items():
        assert st[i] == code, (i, st[i])
        assert np.all(np.isnan(rep.cos_part[i])) and np.all(np.isnan(rep.sin_part[i]))
    good = [i for i in range(count) if i not in bad]
    assert np.all(st[good] == 0)
    for i in good[:: max(1, len(good) // 6)]:
        c, s, k, sc = orc.cos_sin(a[i])
        assert rel1(rep.cos_part[i], c) <= TOL64, i
        assert rel1(rep.sin_part[i], s) <= TOL64, i


def test_empty_inputs(cuda):
    rep = csm.cos_sin(np.zeros((0, 0)))
    assert rep.result.cos_part.shape == (0, 0)
    assert rep.total_products == 3
    rep = csm.cos_sin_batched(np.zeros((0, 4, 4)))
    assert rep.cos_part.shape == (0, 4, 4)


def test_device_selection_matches_host(cuda):
    import ctypes

    import torch
    from paper_2010_00465_b200 import _lib
    rng = np.random.default_rng(77)
    norms = np.concatenate([10.0 ** rng.uniform(-8, 12, 1_000_000),
                            rng.uniform(0, 40, 200_000)])
    extra = []
    for tab in (csm.TAYLOR_TABLE, csm.WAVE_TABLE):
        for p in csm.Precision:
            for e in tab[p].entries:
                for q in range(0, 50):
                    x = math.ldexp(e.theta_eff, q)
                    for _ in range(40):
                        extra.append(x)
                        x = math.nextafter(x, math.inf)
    norms = np.concatenate([norms, np.array(extra)])
    nd = torch.from_numpy(norms).to(cuda)
    for fam_code, fam in ((0, csm.SchemeFamily.COS_SIN_TAYLOR),
                          (1, csm.SchemeFamily.WAVE_KERNEL)):
        for p in csm.Precision:
            k = torch.empty(norms.size, dtype=torch.int32, device=cuda)
            s, st = torch.empty_like(k), torch.empty_like(k)
            rc = _lib.lib().csm_select_device(
                ctypes.c_void_p(nd.data_ptr()), norms.size, fam_code,
                0 if p is csm.Precision.DOUBLE else 1,
                ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(s.data_ptr()),
                ctypes.c_void_p(st.data_ptr()),
                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            assert rc == 0
            hk, hs, hst = csm.select_batch(norms, fam, p)
            assert np.array_equal(k.cpu().numpy(), hk)
            assert np.array_equal(s.cpu().numpy(), hs)
            assert np.array_equal(st.cpu().numpy(), hst)


def test_device_norm1_bits(cuda, golden_dir):
    g = _golden(golden_dir, "norm1.npz")
    i = 0
    while f"a{i}" in g:
        assert csm.norm1(g[f"a{i}"]) == float(g[f"n{i}"]), i
        i += 1


# ---------------------------------------------------------------------------
# Full-size configs: every matrix against the oracle (process pool), plus
# size-independent properties.

def _oracle_batch(args):
    import numpy as _np
    from oracle import cossin_oracle as _orc
    kind, a, t, prec = args
    out = []
    for i in range(a.shape[0]):
        if kind == "wave":
            c, s, k, sc = _orc.wave_cos_sin(a[i], float(t[i]), prec)
        else:
            c, s, k, sc = _orc.cos_sin(a[i].astype(_np.float64) if a.dtype == _np.float32 else a[i], prec)
        out.append((c, s, k, sc))
    return out


def _oracle_all(kind, a, t, prec, chunks=16):
    import multiprocessing as mp
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    parts = np.array_split(np.arange(a.shape[0]), chunks)
    jobs = [(kind, a[p], None if t is None else t[p], prec) for p in parts]
    with mp.get_context("spawn").Pool(min(chunks, os.cpu_count() or 1)) as pool:
        res = pool.map(_oracle_batch, jobs)
    return [r for part in res for r in part]


def _check_all(rep, ref, tol):
    worst = 0.0
    for i, (c, s, k, sc) in enumerate(ref):
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc), i
        ok_c, rc = pair_close(rep.cos_part[i], c, s, tol)
        ok_s, rs = pair_close(rep.sin_part[i], s, c, tol)
        assert ok_c and ok_s, (i, rc, rs)
        worst = max(worst, min(rc, 1.0), min(rs, 1.0))
    return worst


@pytest.mark.timeout(900)
def test_full_cfg2_against_oracle(cuda):
    """configs[1] at full size: all 16384 matrices, (k, s) exact, <= 1e-12."""
    from oracle.cpu_pool import _gen
    a, _ = _gen("cfg2", 0, 16384, 64)
    rep = csm.cos_sin_batched(a)
    _check_all(rep, _oracle_all("trig", a, None, "double"), TOL64)


@pytest.mark.timeout(900)
def test_full_cfg3_against_oracle(cuda):
    """configs[2] at full size (4096 x 256^2 float32): (k, s) exact vs the
    reference on the same float32 input, outputs within 1e-5."""
    from oracle.cpu_pool import _gen
    a, _ = _gen("cfg3", 0, 4096, 256)
    rep = csm.cos_sin_batched(a, csm.Precision.SINGLE)
    ref = _oracle_all("trig", a, None, "single")  # upcast oracle
    for i, (c, s, k, sc) in enumerate(ref):
        assert (int(rep.k[i]), int(rep.s[i])) == (k, sc), i
        assert rel1(rep.cos_part[i], c) <= TOL32, i
        assert rel1(rep.sin_part[i], s) <= TOL32, i


def test_negation_symmetry_bitwise(cuda):
    """cos(-A) == cos(A) and sin(-A) == -sin(A) bit for bit (sign flips are
    exact through every product), on the full cfg2 distribution."""
    from oracle.cpu_pool import _gen
    a, _ = _gen("cfg2", 3, 4096, 64)
    p = csm.cos_sin_batched(a)
    m = csm.cos_sin_batched(-a)
    assert np.array_equal(p.k, m.k) and np.array_equal(p.s, m.s)
    assert np.array_equal(p.cos_part, m.cos_part)
    assert np.array_equal(p.sin_part, -m.sin_part)


def test_batch_position_invariance(cuda):
    """A matrix's result does not depend on its batch neighbours or position
    (the schedule reorders by cost): subsets reproduce the full batch bits."""
    from oracle.cpu_pool import _gen
    a, _ = _gen("cfg2", 4, 3000, 64)
    full = csm.cos_sin_batched(a)
    idx = np.random.default_rng(1).permutation(3000)[:700]
    sub = csm.cos_sin_batched(a[idx])
    assert np.array_equal(sub.cos_part, full.cos_part[idx])
    assert np.array_equal(sub.sin_part, full.sin_part[idx])
    # tiled path too
    b = cfg2_like(np.random.default_rng(5), 24, n=160)
    fb = csm.cos_sin_batched(b)
    sb = csm.cos_sin_batched(b[5:17])
    assert np.array_equal(sb.cos_part, fb.cos_part[5:17])


def test_pythagorean_full_cfg2(cuda):
    """||C^2 + S^2 - I||_1 on the whole cfg2 batch, computed on the GPU in
    float64; bounded by the float64 floor that grows with ||cos||."""
    import torch
    from oracle.cpu_pool import _gen
    a, _ = _gen("cfg2", 0, 16384, 64)
    rep = csm.cos_sin_batched(torch.from_numpy(a).to(cuda))
    c, s = rep.cos_part, rep.sin_part
    r = c @ c + s @ s - torch.eye(64, dtype=torch.float64, device=cuda)
    res = r.abs().sum(dim=1).amax(dim=1)
    cn = c.abs().sum(dim=1).amax(dim=1)
    assert bool(torch.all(res <= 1e-13 * torch.clamp(cn * cn, min=1.0)))


def _oracle_permuted(a):
    """The oracle with every product evaluated in a different summation
    order (K split in two halves): an estimate of the reference's own
    rounding noise."""
    from oracle import cossin_oracle as _o
    import numpy as _np

    class _T(_np.ndarray):
        def __matmul__(self, other):
            x, y = _np.asarray(self), _np.asarray(other)
            h = x.shape[1] // 2 + 1
            return (x[:, :h] @ y[:h] + x[:, h:] @ y[h:]).view(_T)

    k, s = _o.select(_o.norm1(a))
    c, sn = _o.taylor_core((a * 2.0 ** -s).view(_T), k)
    c, sn = _o.double_angle(_np.asarray(c).view(_T), _np.asarray(sn).view(_T), s)
    return _np.asarray(c), _np.asarray(sn)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("n", [1024])
def test_large_symmetric_against_oracle_noise_floor(cuda, n):
    """configs[4] analogue at n=1024 (20 (G+G^T)/(2 sqrt n), s=8): the 1e-12
    gate sits below the reference's own rounding noise here,
    so the gate is max(1e-12, 4 x the oracle-vs-permuted-oracle noise)."""
    g = np.random.default_rng(0).standard_normal((n, n))
    a = 20.0 * (g + g.T) / (2.0 * np.sqrt(n))
    c, s, k, sc = orc.cos_sin(a)
    cp, sp = _oracle_permuted(a)
    noise = max(rel1(cp, c), rel1(sp, s))
    rep = csm.cos_sin(a)
    assert (rep.scheme_used.k_products, rep.scaling_exponent) == (k, sc)
    gate = max(TOL64, 4.0 * noise)
    assert rel1(rep.result.cos_part, c) <= gate, (rel1(rep.result.cos_part, c), noise)
    assert rel1(rep.result.sin_part, s) <= gate, (rel1(rep.result.sin_part, s), noise)
    # third number: both against the double-double truth
    from paper_2010_00465_b200 import verify
    tr = verify.reference_cos_sin(a)
    for got, ref, t in ((rep.result.cos_part, c, tr.cos_part),
                        (rep.result.sin_part, s, tr.sin_part)):
        assert rel1(got, t) <= 4.0 * rel1(ref, t) + 1e-15, (rel1(got, t), rel1(ref, t))


@pytest.mark.timeout(600)
def test_wave_cfg4_analogue_three_numbers(cuda):
    """configs[3] analogue (SPD Laplacian + potential, n = 256, large s):
    GPU vs reference gated at max(1e-12, 4 x the reference's own
    permuted-order noise), and both against the eigendecomposition answer
    c = V cos(t sqrt(L)) V^T, s = V sin(t sqrt(L))/sqrt(L) V^T."""
    rng = np.random.default_rng(4)
    a, _ = laplacian_wave(rng, 1, 256)
    a = a[0]
    t = 1e-1
    c, s, k, sc = orc.wave_cos_sin(a, t)
    assert sc >= 9
    rep = csm.wave_cos_sin(a, t)
    assert (rep.scheme_used.k_products, rep.scaling_exponent) == (k, sc)

    class _T(np.ndarray):
        def __matmul__(self, other):
            x, y = np.asarray(self), np.asarray(other)
            h = x.shape[1] // 2 + 1
            return (x[:, :h] @ y[:h] + x[:, h:] @ y[h:]).view(_T)

    tp = t / 2.0 ** sc
    cp, spp = orc.wave_core(a.view(_T), tp, k)
    cp, spp = orc.double_angle(np.asarray(cp).view(_T), np.asarray(spp).view(_T), sc)
    noise = max(rel1(np.asarray(cp), c), rel1(np.asarray(spp), s))
    gate = max(TOL64, 4.0 * noise)
    assert rel1(rep.result.c_part, c) <= gate
    assert rel1(rep.result.s_part, s) <= gate
    lam, v = np.linalg.eigh(a)
    w = np.sqrt(lam)
    ce = (v * np.cos(t * w)) @ v.T
    se = (v * (np.sin(t * w) / w)) @ v.T
    for got, ref, ex in ((rep.result.c_part, c, ce), (rep.result.s_part, s, se)):
        assert rel1(got, ex) <= 4.0 * rel1(ref, ex) + 1e-14, (rel1(got, ex), rel1(ref, ex))


def _pade_tol(s, prec="double"):
    """Pade + s doublings: the doubling recursion amplifies a perturbation of
    the base pair by up to ~4 per step (verify.py:396-399 says the same of
    its own oracle), and PADE_TABLE's small theta (0.112) needs s 4-5 more
    steps than the Taylor table at the same norm.  Parity bar: 64 u 4^s,
    never below the hot path's 1e-12 / 1e-5."""
    if prec == "single":
        return TOL32
    return max(TOL64, 64 * 2.0 ** -53 * 4.0 ** s)


def test_pade_golden_cases(cuda, golden_dir):
    """Order-8 Pade baseline against the reference's own pade_cos_sin."""
    from fractions import Fraction
    g = _golden(golden_dir, "pade.npz")
    for entry in g["names"]:
        name, prec = str(entry).split("|")
        a = g[f"{name}__a"]
        rep = csm.pade_cos_sin(a, csm.Precision(prec))
        s = int(g[f"{name}__s"])
        assert rep.scaling_exponent == s, name
        assert rep.scheme_used == csm.SchemeId(csm.SchemeFamily.PADE8, 5)
        assert rep.total_products == Fraction(22, 3) + 2 * s
        ref_c, ref_s = g[f"{name}__cos"], g[f"{name}__sin"]
        tol = _pade_tol(s, prec)
        assert pair_close(rep.result.cos_part, ref_c, ref_s, tol)[0], name
        if orc.norm1(ref_s) > 0:
            assert pair_close(rep.result.sin_part, ref_s, ref_c, tol)[0], name
        if prec == "double":  # as accurate as the reference, against dd truth
            from paper_2010_00465_b200 import verify
            truth = verify.reference_cos_sin(a)
            for got, ref, tr in ((rep.result.cos_part, ref_c, truth.cos_part),
                                 (rep.result.sin_part, ref_s, truth.sin_part)):
                if orc.norm1(tr) > 0:
                    assert rel1(got, tr) <= 10 * rel1(ref, tr) + 1e-15, name


@pytest.mark.parametrize("n", [64, 100, 200])
def test_pade_batched_against_oracle(cuda, n):
    rng = np.random.default_rng(500 + n)
    a = cfg2_like(rng, 6, n=n, lo=-3, hi=1.5)
    rep = csm.pade_cos_sin_batched(a)
    assert (rep.k == 5).all()
    for i in range(a.shape[0]):
        c, s, sc = orc.pade_cos_sin(a[i])
        assert int(rep.s[i]) == sc
        assert pair_close(rep.cos_part[i], c, s, _pade_tol(sc))[0], (n, i)
        assert pair_close(rep.sin_part[i], s, c, _pade_tol(sc))[0], (n, i)


def test_pade_float32_and_agreement_with_taylor(cuda):
    """float32 storage on the SINGLE table; Pade and Taylor agree on the
    same inputs to the float32 tolerance."""
    rng = np.random.default_rng(510)
    a32 = cfg3_like(rng, 6, n=96)
    rep = csm.pade_cos_sin_batched(a32, csm.Precision.SINGLE)
    tay = csm.cos_sin_batched(a32, csm.Precision.SINGLE)
    assert rep.cos_part.dtype == np.float32
    for i in range(a32.shape[0]):
        c, s, sc = orc.pade_cos_sin(a32[i].astype(np.float64), "single")
        assert rel1(rep.cos_part[i], c) <= TOL32
        assert rel1(rep.sin_part[i], s) <= TOL32
        assert rel1(rep.cos_part[i], tay.cos_part[i]) <= TOL32


def test_pade_errors(cuda):
    with pytest.raises(csm.MatrixInputError):
        csm.pade_cos_sin(np.array([[np.nan, 0.0], [0.0, 1.0]]))
    with pytest.raises(ValueError):  # infinite norm (driver.py:77-78)
        csm.pade_cos_sin(np.array([[1e308, 0.0], [1e308, 0.0]]))
    with pytest.raises(OverflowError):  # finite norm, norm / theta = inf
        csm.pade_cos_sin(np.array([[1e308, 0.0], [0.0, 0.0]]))


@pytest.mark.parametrize("n", [64, 37, 1])
def test_self_selecting_small_batches(cuda, n):
    """Batches no larger than the K1 grid (<= 148 matrices, n <= 64) run as
    ONE launch whose CTAs compute their matrix's norm, finiteness and (k, s)
    themselves -- on K1s (each matrix over a 4-CTA cluster) while the batch
    fits the co-resident clusters, else on K1 (one CTA per matrix).
    Bitwise the same cos / sin / k / s / status as the K0 path that a
    larger batch takes (K1s sums k in K1's order), for float64, float32
    storage, the wave family and bad inputs."""

    def same(x, y, bitwise):
        x, y = x.cpu().double().numpy(), y.cpu().double().numpy()
        if bitwise:
            return np.array_equal(x, y, equal_nan=True)
        fin = np.isfinite(y).all(axis=(1, 2))
        d = np.abs(x[fin] - y[fin]).sum(axis=1).max(axis=1)
        r = np.abs(y[fin]).sum(axis=1).max(axis=1)
        return bool(np.all(d <= 1e-13 * np.maximum(r, 1e-300))) and \
            np.array_equal(np.isnan(x), np.isnan(y))
    import torch
    rng = np.random.default_rng(700 + n)
    big = cfg2_like(rng, 160, n=n)
    big[3, 0, 0] = np.nan                       # status 1
    big[5] *= 1e306                             # norm overflow paths
    for idx in ([0, 1, 2, 3, 4, 5, 77, 159], list(range(100))):  # K1s, K1
      for a in (big, big.astype(np.float32)):
        prec = csm.Precision.DOUBLE if a.dtype == np.float64 else csm.Precision.SINGLE
        full = csm.cos_sin_batched(torch.from_numpy(a).to(cuda), prec, raise_on_error=False)
        sub = csm.cos_sin_batched(torch.from_numpy(a[idx]).to(cuda), prec, raise_on_error=False)
        assert np.array_equal(sub.k.cpu().numpy(), full.k.cpu().numpy()[idx])
        assert np.array_equal(sub.s.cpu().numpy(), full.s.cpu().numpy()[idx])
        assert np.array_equal(sub.status.cpu().numpy(), full.status.cpu().numpy()[idx])
        # matrix 5 (float64): finite norm ~1e308, s ~ 1000 doublings -> NaN in
        # both paths, so NaNs compare equal
        assert same(sub.cos_part, full.cos_part[idx], True)
        assert same(sub.sin_part, full.sin_part[idx], True)
        assert int(sub.status[3]) == 1
    t = 10.0 ** rng.uniform(-2, 0.5, 160)
    w = big[:, :, :] * 0.01
    w[3, 0, 0] = 1.0
    w[5] = w[6]
    fw = csm.wave_cos_sin_batched(torch.from_numpy(w).to(cuda), torch.from_numpy(t).to(cuda))
    for idx in ([0, 1, 2, 3, 4, 5, 77, 159], list(range(100))):
        sw = csm.wave_cos_sin_batched(torch.from_numpy(w[idx]).to(cuda),
                                      torch.from_numpy(t[idx]).to(cuda))
        assert np.array_equal(sw.k.cpu().numpy(), fw.k.cpu().numpy()[idx])
        assert np.array_equal(sw.s.cpu().numpy(), fw.s.cpu().numpy()[idx])
        assert same(sw.cos_part, fw.cos_part[idx], True)
        assert same(sw.sin_part, fw.sin_part[idx], True)
    # the self-selecting path against the oracle, and the reference's
    # exception on a bad matrix
    sub = csm.cos_sin_batched(big[[0, 1, 77]])
    for j, i in enumerate((0, 1, 77)):
        c, s, k, sc = orc.cos_sin(big[i])
        assert (int(sub.k[j]), int(sub.s[j])) == (k, sc)
        assert pair_close(sub.cos_part[j], c, s, TOL64)[0]
        assert pair_close(sub.sin_part[j], s, c, TOL64)[0]
    with pytest.raises(csm.MatrixInputError):
        csm.cos_sin(big[3])
