"""ctypes binding of libcossin_b200.so (the C-ABI in include/cossin_b200.h).

There is deliberately no fallback: if the library is missing, importing
this module's ``lib()`` raises; if no sm_100 device is present, every
compute entry point returns CSM_ERR_NO_DEVICE and the Python layer raises
RuntimeError.
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import build as _build

# dtype codes
F64, F32, F32_IN_F64_OUT = 0, 1, 2
PREC_DOUBLE, PREC_SINGLE = 0, 1
FAMILY_TAYLOR, FAMILY_WAVE, FAMILY_PADE = 0, 1, 2
# per-matrix status
OK, NONFINITE_INPUT, NONFINITE_NORM, SELECT_OVERFLOW, SINGULAR = 0, 1, 2, 3, 4
# return codes
SUCCESS, ERR_ARG, ERR_CUDA, ERR_WORKSPACE, ERR_NO_DEVICE = 0, -1, -2, -3, -4

_vp, _i32, _i64, _sz, _dp = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                             ctypes.c_size_t, ctypes.c_double)

# symbol -> (restype, argtypes); exactly the functions include/cossin_b200.h
# declares (tests/test_abi.py checks both directions).
SIGNATURES = {
    "csm_version": (ctypes.c_char_p, []),
    "csm_last_error": (ctypes.c_char_p, []),
    "csm_workspace_size": (_sz, [_i32, _i64, _i32]),
    "csm_norm1": (_i32, [_i32, _vp, _i64, _i32, _vp, _vp, _vp]),
    "csm_select_host": (_i32, [_vp, _i64, _i32, _i32, _vp, _vp, _vp]),
    "csm_select_device": (_i32, [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp]),
    "csm_select_table": (_i32, [_vp, _i64, _vp, _vp, _vp, _i32, _vp, _vp,
                                _vp]),
    "csm_cos_sin": (_i32, [_i32, _i32, _vp, _vp, _vp, _i64, _i32, _vp, _vp,
                           _vp, _vp, _sz, _vp]),
    "csm_wave": (_i32, [_i32, _i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp,
                        _vp, _vp, _sz, _vp]),
    "csm_taylor_core": (_i32, [_i32, _i32, _vp, _vp, _vp, _i64, _i32, _vp,
                               _vp, _sz, _vp]),
    "csm_wave_core": (_i32, [_i32, _i32, _vp, _vp, _vp, _vp, _i64, _i32,
                             _vp, _vp, _sz, _vp]),
    "csm_theta_table": (_i32, [_i32, _i32, _vp, _vp, _vp, _i32]),
    "csm_sine_workspace_size": (_sz, [_i32, _i64, _i32]),
    "csm_taylor_sin9": (_i32, [_i32, _vp, _vp, _i64, _i32, _vp, _vp, _sz, _vp]),
    "csm_wave_sin34": (_i32, [_i32, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _sz, _vp]),
    "csm_pade_workspace_size": (_sz, [_i32, _i64, _i32]),
    "csm_pade_cos_sin": (_i32, [_i32, _i32, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "csm_pade_core": (_i32, [_i32, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _sz, _vp]),
    "csm_residual_workspace_size": (_sz, [_i64, _i32]),
    "csm_pythagorean_residual": (_i32, [_i32, _vp, _vp, _i64, _i32, _vp, _vp, _sz, _vp]),
    "csm_ddref_workspace_size": (_sz, [_i64, _i32]),
    "csm_ddref_cos_sin": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _sz, _vp]),
    "csm_dd_matmul": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp]),
    "csm_ddref_series_consts": (_i32, [_vp]),
    "csm_fp64_peak": (_i32, [_i32, _vp, _vp]),
    "csm_last_launch_count": (_i64, []),
    "csm_op_bytes": (_sz, []),
    "csm_slab_scratch_bytes": (_sz, []),
    "csm_slab_engine_bytes": (_sz, [_i32, _i32]),
    "csm_chain_program": (_i32, [_i32, _i32, _i32, _vp, _i32, _vp, _i32, _vp, _vp]),
    "csm_doubling_program": (_i32, [_i32, _i32, _i32, _i32, _vp]),
    "csm_slab_op": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp, _vp, _i32, _dp, _i32, _vp, _vp,
                           _i32, _vp, _sz, _vp]),
    "csm_slab_op_peer": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _dp, _i32,
                                _vp, _vp, _i32, _vp, _sz, _vp]),
    "csm_slab_op_pair": (_i32, [_vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _i32, _dp, _i32,
                                _vp, _vp, _i32, _vp, _sz, _vp]),
    "csm_dist_workspace_size": (_sz, [_i32, _i32, _i32]),
    "csm_dist_cos_sin": (_i32, [_i32, _vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _sz,
                                _vp]),
    "csm_dist_cos_sin_virtual": (_i32, [_i32, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _sz,
                                        _vp]),
    "csm_dist_last_stats": (_i32, [_vp, _vp]),
    "csm_nccl_get_unique_id": (_i32, [_vp]),
    "csm_nccl_comm_init_rank": (_i32, [_vp, _i32, _vp, _i32]),
    "csm_nccl_comm_destroy": (_i32, [_vp]),
    "csm_graph_safe": (_i32, [_i32, _i64, _i32]),
    "csm_set_engine": (_i32, [_i32]),
    "csm_get_engine": (_i32, []),
    "csm_set_thread_engine": (_i32, [_i32]),
    "csm_profile_enable": (_i32, [_i32]),
    "csm_profile_collect": (_i32, [_vp, _vp]),
}

_LOCK = threading.Lock()
_LIB: ctypes.CDLL | None = None


def lib_path() -> str:
    """The in-tree library, or $CSM_LIB_PATH (e.g. an instrumented build)."""
    return os.environ.get("CSM_LIB_PATH") or _build.LIB


def lib() -> ctypes.CDLL:
    """Load (once) and return the library; raise if it was never built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    with _LOCK:
        if _LIB is None:
            path = lib_path()
            if not os.path.exists(path):
                raise ImportError(
                    f"{path} is missing: build the sm_100a library first "
                    "(python paper_2010_00465_b200/build.py); there is no "
                    "CPU fallback")
            handle = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _LIB = handle
    return _LIB


def last_error() -> str:
    msg = lib().csm_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> int:
    """Raise for a negative return code; pass counts through."""
    if rc < 0:
        raise RuntimeError(f"{what} failed (code {rc}): {last_error()}")
    return rc
