"""The C-ABI library loads and exports exactly what include/cossin_b200.h
declares (CPU-only: no compute calls)."""
import ctypes
import os
import re

import pytest

import paper_2010_00465_b200 as csm
from paper_2010_00465_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "cossin_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(csm_[a-z0-9_]+)\s*\(", text))


def test_header_lists_the_bound_symbols():
    assert header_functions() == set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in header_functions():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_version_and_workspace_size():
    lib = _lib.lib()
    assert b"sm_100a" in lib.csm_version()
    small = lib.csm_workspace_size(0, 16, 64)
    big = lib.csm_workspace_size(0, 16, 256)
    assert 0 < small < big
    # tiled path: 9 float64 slots of 256^2 per matrix at least
    assert big >= 16 * 9 * 256 * 256 * 8


def test_argument_errors_without_device():
    lib = _lib.lib()
    rc = lib.csm_cos_sin(7, 0, None, None, None, 1, 4, None, None, None,
                         None, 0, None)
    assert rc == _lib.ERR_ARG
    assert "dtype" in _lib.last_error()
    rc = lib.csm_taylor_core(0, 5, None, None, None, 1, 4, None, None,
                             1 << 20, None)
    assert rc == _lib.ERR_ARG
    rc = lib.csm_cos_sin(0, 0, None, None, None, 4, 8, None, None, None,
                         None, 0, None)
    assert rc == _lib.ERR_WORKSPACE


def test_elf_is_sm100a():
    """The .so carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_ddref_series_constants_match_reference(golden_dir):
    """The library's _dd_const splits (computed with an exact fma residual)
    equal the reference's Fraction-based ones bit for bit."""
    import ctypes
    import os
    import numpy as np
    d = np.load(os.path.join(golden_dir, "ddref.npz"))["consts"]  # (14, 2)
    out = (ctypes.c_double * 28)()
    assert _lib.lib().csm_ddref_series_consts(out) == 0
    got = np.array(out[:])
    want = np.concatenate([d[:7, 0], d[:7, 1], d[7:, 0], d[7:, 1]])
    assert (got.view(np.uint64) == want.view(np.uint64)).all()


def test_engine_switch_without_device():
    """csm_set_engine is host-only: a bad engine is CSM_ERR_ARG, and the
    Ozaki engine enlarges the tiled workspace (n = 256) but not n = 64 or
    the DMMA-only orders (NP % 256 != 0)."""
    lib = _lib.lib()
    assert lib.csm_get_engine() == 0  # DMMA: the default engine
    assert lib.csm_workspace_size(0, 1, 4096) < 9 * 4096 * 4096 * 8 + 16 * 3 * 4096 * 4096
    assert lib.csm_set_thread_engine(2) == 0  # auto: Ozaki scratch from padded order 768 up
    try:
        assert lib.csm_workspace_size(0, 1, 4096) > 9 * 4096 * 4096 * 8 + 16 * 3 * 4096 * 4096
    finally:
        assert lib.csm_set_thread_engine(-1) == 0
    assert lib.csm_set_engine(5) == _lib.ERR_ARG
    assert lib.csm_set_engine(0) == 0
    assert "engine" in _lib.last_error()
    dm256, dm320, dm64 = (lib.csm_workspace_size(0, 8, n) for n in (256, 320, 64))
    assert lib.csm_slab_engine_bytes(512, 1024) == 0
    assert lib.csm_set_engine(1) == 0
    try:
        assert lib.csm_get_engine() == 1
        assert lib.csm_workspace_size(0, 8, 256) > dm256
        assert lib.csm_workspace_size(0, 8, 320) == dm320
        assert lib.csm_workspace_size(0, 8, 64) == dm64
        # residue planes of L (M x NP), R (NP x NP) and the product, 16 moduli
        assert lib.csm_slab_engine_bytes(512, 1024) >= 16 * (2 * 512 * 1024 + 1024 * 1024)
    finally:
        assert lib.csm_set_engine(0) == 0


def test_slab_op_pair_argument_errors_without_device():
    """csm_slab_op_pair runs a doubling step: dbl_step < 0 and bad shapes are
    CSM_ERR_ARG before any device work."""
    lib = _lib.lib()
    op = ctypes.create_string_buffer(int(lib.csm_op_bytes()))
    dummy = ctypes.c_void_p(16)
    rc = lib.csm_slab_op_pair(op, op, dummy, 64, 128, 0, dummy, dummy, 0, 0.0, -1,
                              dummy, dummy, 0, dummy, 1 << 40, None)
    assert rc == _lib.ERR_ARG and "doubling" in _lib.last_error()
    rc = lib.csm_slab_op_pair(op, op, dummy, 60, 128, 0, dummy, dummy, 0, 0.0, 0,
                              dummy, dummy, 0, dummy, 1 << 40, None)
    assert rc == _lib.ERR_ARG
    rc = lib.csm_slab_op_pair(None, op, dummy, 64, 128, 0, dummy, dummy, 0, 0.0, 0,
                              dummy, dummy, 0, dummy, 1 << 40, None)
    assert rc == _lib.ERR_ARG


def test_slab_scratch_size_is_checked_without_device():
    """The slab calls take the scratch size and refuse a buffer smaller than
    csm_slab_scratch_bytes() + csm_slab_engine_bytes(M, NP) of the call's
    engine (CSM_ERR_WORKSPACE) before touching the device."""
    lib = _lib.lib()
    op = ctypes.create_string_buffer(int(lib.csm_op_bytes()))
    dummy = ctypes.c_void_p(16)
    base = int(lib.csm_slab_scratch_bytes())
    assert lib.csm_set_thread_engine(1) == 0  # Ozaki: engine bytes at 512 x 1024
    try:
        need = base + int(lib.csm_slab_engine_bytes(512, 1024))
        assert need > base
        rc = lib.csm_slab_op(op, dummy, 512, 1024, 0, dummy, dummy, 0, 0.0, -1,
                             dummy, dummy, 0, dummy, need - 1, None)
        assert rc == _lib.ERR_WORKSPACE and "scratch" in _lib.last_error()
        rc = lib.csm_slab_op_pair(op, op, dummy, 512, 1024, 0, dummy, dummy, 0, 0.0, 0,
                                  dummy, dummy, 0, dummy, base, None)
        assert rc == _lib.ERR_WORKSPACE
    finally:
        assert lib.csm_set_thread_engine(-1) == 0


def test_thread_engine_override_is_per_thread():
    """csm_set_thread_engine overrides the process default for the calling
    thread only; engine_scope nests and restores."""
    import threading
    lib = _lib.lib()
    assert lib.csm_set_thread_engine(7) == _lib.ERR_ARG
    seen = {}
    with csm.engine_scope("dmma"):
        assert csm.get_engine() == "dmma"
        with csm.engine_scope("ozaki"):
            assert csm.get_engine() == "ozaki"
            th = threading.Thread(target=lambda: seen.setdefault("other", csm.get_engine()))
            th.start()
            th.join()
        assert csm.get_engine() == "dmma"
    assert csm.get_engine() == "dmma"
    assert seen["other"] == "dmma"  # another thread sees the process default


def test_dist_workspace_sizes_and_argument_errors():
    """csm_dist_workspace_size (host arithmetic, no device): slab + partial
    products + staging, plus the gather pool only when ranks gather; and
    argument errors are reported before any device work."""
    import ctypes

    from paper_2010_00465_b200 import _lib
    L = _lib.lib()
    n, w = 8192, 8
    M = n // w
    base = L.csm_dist_workspace_size(n, w, 0)
    assert base > (9 + 2) * M * n * 8
    one = L.csm_dist_workspace_size(n, 1, 0)
    assert (9 + 2) * n * n * 8 < one < (9 + 2) * n * n * 8 + (1 << 20)  # no pool at W = 1
    forced = L.csm_dist_workspace_size(n, 1, 1)
    pool = forced - one
    assert pool % (n * n * 8) == 0 and 1 <= pool // (n * n * 8) <= 5
    assert L.csm_dist_workspace_size(100, 3, 0) == 0
    k = ctypes.c_int32()
    for n_bad in (0, 100):
        rc = L.csm_dist_cos_sin_virtual(0, ctypes.c_void_p(1), ctypes.c_void_p(1),
                                        ctypes.c_void_p(1), n_bad, 2, ctypes.byref(k),
                                        ctypes.byref(k), ctypes.byref(k), ctypes.c_void_p(1),
                                        1 << 40, None)
        assert rc == _lib.ERR_ARG
    g, p = ctypes.c_int32(), ctypes.c_int32()
    assert L.csm_dist_last_stats(ctypes.byref(g), ctypes.byref(p)) == 0


def test_profile_modes_without_device():
    """csm_profile_enable: 0 off, 1 pipeline intervals, 2 int8 GEMM launches,
    3 the fused K0 launch; anything else is an argument error.  No events
    exist without a launch, so collect returns zero intervals."""
    import ctypes
    lib = _lib.lib()
    for mode in (1, 2, 3, 0):
        assert lib.csm_profile_enable(mode) == 0
    assert lib.csm_profile_enable(4) == _lib.ERR_ARG
    assert lib.csm_profile_enable(-1) == _lib.ERR_ARG
    tot, cnt = ctypes.c_double(-1.0), ctypes.c_int64(-1)
    assert lib.csm_profile_collect(ctypes.byref(tot), ctypes.byref(cnt)) == 0
    assert tot.value == 0.0 and cnt.value == 0
