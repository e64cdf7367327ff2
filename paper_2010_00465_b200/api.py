"""Drop-in entry points of the cos/sin hot path, backed by sm_100a kernels.

Single-matrix functions keep the reference's names, signatures, return
types and exceptions (paths under /root/reference/pkg/src/cossinm):

* cos_sin(a, precision) ............... driver.py:108-123
* wave_cos_sin(a, t, precision) ....... driver.py:126-146
* select_scheme(norm, table) .......... driver.py:70-88   (C++ host twin)
* taylor_cos_sin(a, scheme, ledger) ... schemes.py:376-395
* wave_kernels(a, t, scheme, ledger) .. schemes.py:411-430
* norm1(a) ............................ matcore.py:100-104 (device kernel)
* matrix_from_rows(rows) .............. matcore.py:69-83  (host validation)

Batched functions (cos_sin_batched / wave_cos_sin_batched) are the B200
path proper: one C-ABI call per batch; inputs may be numpy arrays, torch
CPU tensors (pinned for speed) or torch CUDA tensors.  Every numeric
result comes from the CUDA library; there is no CPU fallback.
"""
from __future__ import annotations

import contextlib
import ctypes
import threading
from dataclasses import dataclass
from fractions import Fraction
from typing import Any, Sequence

import numpy as np

from . import _lib
from .records import (
    TAYLOR_TABLE,
    WAVE_TABLE,
    ComputationReport,
    CosSinResult,
    CostLedger,
    MatrixInputError,
    Precision,
    SchemeFamily,
    SingularMatrixError,
    SchemeId,
    ThetaTable,
    WaveResult,
    _PREC_CODE,
)

_TORCH = None


def _torch():
    global _TORCH
    if _TORCH is None:
        import torch
        _TORCH = torch
    return _TORCH


def _device():
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError(
            "no CUDA device: the cos/sin path runs only on the sm_100a "
            "kernels (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream_handle(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _vp(x: int) -> ctypes.c_void_p:
    return ctypes.c_void_p(x)


# ---------------------------------------------------------------------------
# Operand normalisation.

@dataclass
class _Batch:
    dev: Any           # torch CUDA tensor (B, n, n), float64 or float32
    code: int          # C-ABI dtype code
    host: str | None   # None (device in/out), "numpy" or "torch"
    out_dtype: Any     # torch dtype of the results


def _as_batch(a, batched: bool, f32_out: bool) -> _Batch:
    torch = _torch()
    if isinstance(a, torch.Tensor):
        t, host = a, (None if a.is_cuda else "torch")
    else:
        arr = np.asarray(a)
        if np.iscomplexobj(arr):
            raise TypeError("complex matrices are not supported on this path")
        if arr.dtype != np.float32 and arr.dtype != np.float64:
            arr = arr.astype(np.float64)
        t, host = torch.from_numpy(np.ascontiguousarray(arr)), "numpy"
    want = 3 if batched else 2
    if t.dim() != want or t.shape[-1] != t.shape[-2]:
        kind = "batch of square matrices (B, n, n)" if batched else "square"
        raise MatrixInputError(
            f"matrix must be {kind}, got shape {tuple(t.shape)}")
    if t.is_complex():
        raise TypeError("complex matrices are not supported on this path")
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    if t.dtype == torch.float32:
        code = _lib.F32 if f32_out else _lib.F32_IN_F64_OUT
    else:
        code = _lib.F64
    out_dtype = torch.float32 if code == _lib.F32 else torch.float64
    dev = _device()
    if not batched:
        t = t.unsqueeze(0)
    if t.is_cuda:
        t = t.contiguous()
    else:
        t = t.contiguous().to(dev, non_blocking=t.is_pinned())
    return _Batch(t, code, host, out_dtype)


def _status_error(status: int, norm: float) -> Exception:
    if status == _lib.NONFINITE_INPUT:
        return MatrixInputError("matrix entries must be finite")
    if status == _lib.SINGULAR:
        return SingularMatrixError(
            "denominator singular to working precision (pivot <= 1e3 eps "
            "||den||_1)")
    if status == _lib.NONFINITE_NORM:
        return ValueError(f"norm must be finite and nonnegative, got {norm}")
    return OverflowError("cannot convert float infinity to integer")


# ---------------------------------------------------------------------------
# Batched pipeline.

@dataclass
class BatchReport:
    """Results of a batched call: cos/sin (or c/s) parts plus per-matrix
    (k, s); total_products[b] = k[b] + 2 s[b] (the ledger of driver.py:122).
    """

    cos_part: Any
    sin_part: Any
    k: Any
    s: Any
    status: Any
    family: SchemeFamily

    @property
    def total_products(self):
        """k + 2 s per matrix; 22/3 + 2 s (as float) for the Pade family."""
        if self.family is SchemeFamily.PADE8:
            return self.k + 2 * self.s + 7.0 / 3.0
        return self.k + 2 * self.s

    def report(self, i: int) -> ComputationReport:
        """The reference's per-matrix ComputationReport for entry i."""
        k, s = int(self.k[i]), int(self.s[i])
        ledger = CostLedger()
        ledger.charge_product(k + 2 * s)
        if self.family is SchemeFamily.PADE8:
            ledger.charge_lu(solves=2)
        if self.family is SchemeFamily.WAVE_KERNEL:
            res = WaveResult(self.cos_part[i], self.sin_part[i], ledger)
        else:
            res = CosSinResult(self.cos_part[i], self.sin_part[i], ledger)
        return ComputationReport(res, SchemeId(self.family, k), s,
                                 ledger.total_cost)


def _launch(fn_name: str, batch: _Batch, precision: Precision, t_dev,
            stream=None):
    """Run csm_cos_sin / csm_wave on a device batch; returns device tensors
    (cos, sin, k, s, status, norms_view)."""
    torch = _torch()
    L = _lib.lib()
    a = batch.dev
    B, n = int(a.shape[0]), int(a.shape[-1])
    dev = a.device
    cos = torch.empty((B, n, n), dtype=batch.out_dtype, device=dev)
    sin = torch.empty_like(cos)
    k = torch.empty(B, dtype=torch.int32, device=dev)
    s = torch.empty_like(k)
    status = torch.empty_like(k)
    ws_bytes = int(L.csm_workspace_size(batch.code, B, n))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    h = _stream_handle(stream)
    common = [batch.code, _PREC_CODE[precision], _vp(a.data_ptr())]
    outs = [_vp(cos.data_ptr()), _vp(sin.data_ptr()), B, n,
            _vp(k.data_ptr()), _vp(s.data_ptr()), _vp(status.data_ptr()),
            _vp(ws.data_ptr()), ws_bytes, _vp(h)]
    if fn_name == "csm_wave":
        rc = L.csm_wave(*common, _vp(t_dev.data_ptr()), *outs)
    else:
        rc = L.csm_cos_sin(*common, *outs)
    _lib.check(rc, fn_name)
    return cos, sin, k, s, status, ws


def _finish(batch: _Batch, family: SchemeFamily, precision, cos, sin, k, s,
            status, ws, t_host, raise_on_error: bool) -> BatchReport:
    torch = _torch()
    if raise_on_error:
        st = status.cpu().numpy()
        bad = np.nonzero(st)[0]
        if bad.size:
            i = int(bad[0])
            norm = float(ws[: 8 * st.size].view(torch.float64)[i].item())
            if family is SchemeFamily.WAVE_KERNEL and t_host is not None:
                norm = float(t_host[i]) * float(t_host[i]) * norm
            raise _status_error(int(st[i]), norm)
    if batch.host is None:
        return BatchReport(cos, sin, k, s, status, family)
    ks = k.cpu().numpy()
    ss = s.cpu().numpy()
    st = status.cpu().numpy()
    c_h, s_h = cos.cpu(), sin.cpu()
    if batch.host == "numpy":
        c_h, s_h = c_h.numpy(), s_h.numpy()
    return BatchReport(c_h, s_h, ks, ss, st, family)


def cos_sin_batched(a, precision: Precision = Precision.DOUBLE, *,
                    raise_on_error: bool = True, stream=None) -> BatchReport:
    """cos(A_b) and sin(A_b) for a batch (B, n, n): the reference's cos_sin
    (driver.py:108-123) applied to every matrix, in one device call.

    float32 input computes in float64 and returns float32.  Results live
    where the input lives (numpy / torch CPU / torch CUDA)."""
    batch = _as_batch(a, batched=True, f32_out=True)
    cos, sin, k, s, st, ws = _launch("csm_cos_sin", batch, precision, None,
                                     stream)
    return _finish(batch, SchemeFamily.COS_SIN_TAYLOR, precision, cos, sin,
                   k, s, st, ws, None, raise_on_error)


def pade_cos_sin_batched(a, precision: Precision = Precision.DOUBLE, *,
                         raise_on_error: bool = True,
                         stream=None) -> BatchReport:
    """The order-8 Pade baseline (driver.py:149-164) for a batch (B, n, n):
    PADE_TABLE selection, five products, one batched LU with partial
    pivoting shared by two solves, s doublings -- all on the device."""
    batch = _as_batch(a, batched=True, f32_out=True)
    return _pade(batch, precision, raise_on_error, stream)


def _pade(batch: _Batch, precision, raise_on_error, stream=None) -> BatchReport:
    torch = _torch()
    L = _lib.lib()
    x = batch.dev
    B, n = int(x.shape[0]), int(x.shape[-1])
    dev = x.device
    cos = torch.empty((B, n, n), dtype=batch.out_dtype, device=dev)
    sin = torch.empty_like(cos)
    k = torch.empty(B, dtype=torch.int32, device=dev)
    s = torch.empty_like(k)
    status = torch.empty_like(k)
    ws_bytes = int(L.csm_pade_workspace_size(batch.code, B, n))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    _lib.check(L.csm_pade_cos_sin(batch.code, _PREC_CODE[precision],
                                  _vp(x.data_ptr()), _vp(cos.data_ptr()),
                                  _vp(sin.data_ptr()), B, n, _vp(k.data_ptr()),
                                  _vp(s.data_ptr()), _vp(status.data_ptr()),
                                  _vp(ws.data_ptr()), ws_bytes,
                                  _vp(_stream_handle(stream))),
               "csm_pade_cos_sin")
    return _finish(batch, SchemeFamily.PADE8, precision, cos, sin, k, s,
                   status, ws, None, raise_on_error)


def pade_cos_sin(a, precision: Precision = Precision.DOUBLE
                 ) -> ComputationReport:
    """Drop-in for driver.pade_cos_sin (driver.py:149-164); total_products
    is the reference's 22/3 + 2 s."""
    batch = _as_batch(a, batched=False, f32_out=False)
    if int(batch.dev.shape[-1]) == 0:
        # lu_solve_pair on a 0 x 0 denominator: min pivot 0 <= threshold 0
        # (matcore.py:141-147), so the reference raises
        raise SingularMatrixError(
            "denominator singular to working precision (pivot 0.000e+00 <= 0.000e+00)")
    return _single(_pade(batch, precision, True))


def pade8_cos_sin(a, ledger: CostLedger) -> CosSinResult:
    """The order-8 Pade base pair at a, no scaling (schemes.py:446-464):
    five products, one LU with partial pivoting shared by two solves, all on
    the device (csm_pade_core).  Charges 5 products and one LU with two
    solves (7 + 1/3 product-equivalents), raising SingularMatrixError like
    lu_solve_pair (matcore.py:124-151) after the products are charged."""
    torch = _torch()
    L = _lib.lib()
    batch = _as_batch(a, batched=False, f32_out=False)
    x = batch.dev
    n = int(x.shape[-1])
    dev = x.device
    c = torch.empty((1, n, n), dtype=batch.out_dtype, device=dev)
    s = torch.empty_like(c)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    ws_bytes = int(L.csm_pade_workspace_size(batch.code, 1, n))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    if n > 0:
        _lib.check(L.csm_pade_core(batch.code, _vp(x.data_ptr()), _vp(c.data_ptr()),
                                   _vp(s.data_ptr()), 1, n, _vp(status.data_ptr()),
                                   _vp(ws.data_ptr()), ws_bytes, _vp(_stream_handle())),
                   "csm_pade_core")
    ledger.charge_product(5)
    if n == 0 or int(status.item()) == _lib.SINGULAR:
        raise _status_error(_lib.SINGULAR, 0.0)
    ledger.charge_lu(solves=2)
    if batch.host == "numpy":
        c, s = c[0].cpu().numpy(), s[0].cpu().numpy()
    elif batch.host == "torch":
        c, s = c[0].cpu(), s[0].cpu()
    else:
        c, s = c[0], s[0]
    return CosSinResult(cos_part=c, sin_part=s, cost=ledger)


def _t_vector(t, B: int, dev):
    torch = _torch()
    if isinstance(t, torch.Tensor):
        tv = t.to(device=dev, dtype=torch.float64).reshape(-1)
    else:
        tv = torch.as_tensor(np.asarray(t, dtype=np.float64).reshape(-1),
                             device=dev)
    if tv.numel() == 1 and B != 1:
        tv = tv.expand(B).contiguous()
    if tv.numel() != B:
        raise ValueError(f"need one t per matrix ({B}), got {tv.numel()}")
    return tv.contiguous()


def wave_cos_sin_batched(a, t, precision: Precision = Precision.DOUBLE, *,
                         raise_on_error: bool = True,
                         stream=None) -> BatchReport:
    """c(t_b^2 A_b), s(t_b, A_b) for a batch; t is a scalar or one value per
    matrix (driver.py:126-146 applied to every matrix)."""
    batch = _as_batch(a, batched=True, f32_out=True)
    B = int(batch.dev.shape[0])
    tv = _t_vector(t, B, batch.dev.device)
    c, s_, k, s, st, ws = _launch("csm_wave", batch, precision, tv, stream)
    return _finish(batch, SchemeFamily.WAVE_KERNEL, precision, c, s_, k, s,
                   st, ws, tv.cpu().numpy(), raise_on_error)


# ---------------------------------------------------------------------------
# Reference-compatible single-matrix API.

def _single(batch_report: BatchReport) -> ComputationReport:
    rep = batch_report.report(0)
    return rep


def cos_sin(a, precision: Precision = Precision.DOUBLE) -> ComputationReport:
    """Simultaneous cos(a) and sin(a) (driver.py:108-123)."""
    batch = _as_batch(a, batched=False, f32_out=False)
    cos, sin, k, s, st, ws = _launch("csm_cos_sin", batch, precision, None)
    rep = _finish(batch, SchemeFamily.COS_SIN_TAYLOR, precision, cos, sin, k,
                  s, st, ws, None, True)
    return _single(rep)


def wave_cos_sin(a, t: float, precision: Precision = Precision.DOUBLE
                 ) -> ComputationReport:
    """Wave kernels c(t^2 a), s(t, a) at any t^2 norm (driver.py:126-146)."""
    batch = _as_batch(a, batched=False, f32_out=False)
    tv = _t_vector(float(t), 1, batch.dev.device)
    c, s_, k, s, st, ws = _launch("csm_wave", batch, precision, tv)
    rep = _finish(batch, SchemeFamily.WAVE_KERNEL, precision, c, s_, k, s,
                  st, ws, [float(t)], True)
    return _single(rep)


def _core(a, family: SchemeFamily, k: int, t, ledger: CostLedger):
    torch = _torch()
    L = _lib.lib()
    batch = _as_batch(a, batched=False, f32_out=False)
    x = batch.dev
    n = int(x.shape[-1])
    dev = x.device
    c = torch.empty((1, n, n), dtype=batch.out_dtype, device=dev)
    s = torch.empty_like(c)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    ws_bytes = int(L.csm_workspace_size(batch.code, 1, n))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    h = _vp(_stream_handle())
    if family is SchemeFamily.WAVE_KERNEL:
        tv = _t_vector(float(t), 1, dev)
        rc = L.csm_wave_core(batch.code, k, _vp(x.data_ptr()),
                             _vp(tv.data_ptr()), _vp(c.data_ptr()),
                             _vp(s.data_ptr()), 1, n, _vp(status.data_ptr()),
                             _vp(ws.data_ptr()), ws_bytes, h)
    else:
        rc = L.csm_taylor_core(batch.code, k, _vp(x.data_ptr()),
                               _vp(c.data_ptr()), _vp(s.data_ptr()), 1, n,
                               _vp(status.data_ptr()), _vp(ws.data_ptr()),
                               ws_bytes, h)
    _lib.check(rc, "scheme core")
    ledger.charge_product(k)
    if batch.host == "numpy":
        return c[0].cpu().numpy(), s[0].cpu().numpy()
    if batch.host == "torch":
        return c[0].cpu(), s[0].cpu()
    return c[0], s[0]


def taylor_cos_sin(a, scheme: SchemeId, ledger: CostLedger) -> CosSinResult:
    """One trigonometric pair scheme at a, no scaling (schemes.py:376-395);
    charges exactly scheme.k_products to the ledger."""
    if scheme.family is not SchemeFamily.COS_SIN_TAYLOR:
        raise ValueError(f"not a trigonometric scheme: {scheme}")
    c, s = _core(a, scheme.family, scheme.k_products, None, ledger)
    return CosSinResult(cos_part=c, sin_part=s, cost=ledger)


def wave_kernels(a, t: float, scheme: SchemeId,
                 ledger: CostLedger) -> WaveResult:
    """One wave-kernel pair scheme c(t^2 a), s(t, a) (schemes.py:411-430)."""
    if scheme.family is not SchemeFamily.WAVE_KERNEL:
        raise ValueError(f"not a wave-kernel scheme: {scheme}")
    c, s = _core(a, scheme.family, scheme.k_products, t, ledger)
    return WaveResult(c_part=c, s_part=s, cost=ledger)


def _sine(a, t, ledger: CostLedger, charge: int):
    torch = _torch()
    L = _lib.lib()
    batch = _as_batch(a, batched=False, f32_out=False)
    x = batch.dev
    n = int(x.shape[-1])
    dev = x.device
    out = torch.empty((1, n, n), dtype=batch.out_dtype, device=dev)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    ws_bytes = int(L.csm_sine_workspace_size(batch.code, 1, n))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    h = _vp(_stream_handle())
    if t is None:
        rc = L.csm_taylor_sin9(batch.code, _vp(x.data_ptr()),
                               _vp(out.data_ptr()), 1, n,
                               _vp(status.data_ptr()), _vp(ws.data_ptr()),
                               ws_bytes, h)
    else:
        tv = _t_vector(float(t), 1, dev)
        rc = L.csm_wave_sin34(batch.code, _vp(x.data_ptr()),
                              _vp(tv.data_ptr()), _vp(out.data_ptr()), 1, n,
                              _vp(status.data_ptr()), _vp(ws.data_ptr()),
                              ws_bytes, h)
    _lib.check(rc, "standalone sine")
    ledger.charge_product(charge)
    if batch.host == "numpy":
        return out[0].cpu().numpy()
    if batch.host == "torch":
        return out[0].cpu()
    return out[0]


def taylor_sin9(a, ledger: CostLedger):
    """Degree-9 sine alone (schemes.py:398-408): the exact-sine degree-4
    core times a, no scaling; charges 5 products like the reference."""
    return _sine(a, None, ledger, 5)


def wave_sin34(a, t: float, ledger: CostLedger):
    """Order-3 wave sine t * core(t^2 a) (schemes.py:433-443), no scaling;
    charges 2 products like the reference."""
    return _sine(a, t, ledger, 2)


def select_scheme(norm: float, table: ThetaTable) -> tuple[SchemeId, int]:
    """(scheme, s) for an operand norm (driver.py:70-88), computed by the
    C++ host twin of the device selection (bit-exact log2/ceil rule)."""
    L = _lib.lib()
    x = np.array([float(norm)], dtype=np.float64)
    th = np.array([e.theta_eff for e in table.entries], dtype=np.float64)
    num = np.array([Fraction(e.cost).numerator for e in table.entries],
                   dtype=np.int64)
    den = np.array([Fraction(e.cost).denominator for e in table.entries],
                   dtype=np.int64)
    idx = np.zeros(1, dtype=np.int32)
    s = np.zeros(1, dtype=np.int32)
    st = np.zeros(1, dtype=np.int32)
    p = lambda arr: arr.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.check(L.csm_select_table(p(x), 1, p(th), p(num), p(den), len(th),
                                  p(idx), p(s), p(st)), "csm_select_table")
    if st[0] != _lib.OK:
        raise _status_error(int(st[0]), float(norm))
    return table.entries[int(idx[0])].scheme, int(s[0])


def select_batch(norms, family: SchemeFamily = SchemeFamily.COS_SIN_TAYLOR,
                 precision: Precision = Precision.DOUBLE):
    """Vectorised host-twin selection over built-in tables: (k, s, status)."""
    L = _lib.lib()
    x = np.ascontiguousarray(np.asarray(norms, dtype=np.float64).reshape(-1))
    k = np.zeros(x.size, dtype=np.int32)
    s = np.zeros(x.size, dtype=np.int32)
    st = np.zeros(x.size, dtype=np.int32)
    fam = {SchemeFamily.COS_SIN_TAYLOR: _lib.FAMILY_TAYLOR,
           SchemeFamily.WAVE_KERNEL: _lib.FAMILY_WAVE,
           SchemeFamily.PADE8: _lib.FAMILY_PADE}[family]
    p = lambda arr: arr.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.check(L.csm_select_host(p(x), x.size, fam, _PREC_CODE[precision],
                                 p(k), p(s), p(st)), "csm_select_host")
    return k, s, st


def norm1(a) -> float:
    """Induced 1-norm, column sums in row order (matcore.py:100-104),
    computed on the device."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        if a.numel() == 0:
            return 0.0
    elif np.asarray(a).size == 0:
        return 0.0
    batch = _as_batch(a, batched=False, f32_out=True)
    x = batch.dev
    n = int(x.shape[-1])
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    st = torch.empty(1, dtype=torch.int32, device=x.device)
    code = _lib.F32 if x.dtype == torch.float32 else _lib.F64
    _lib.check(_lib.lib().csm_norm1(code, _vp(x.data_ptr()), 1, n,
                                    _vp(out.data_ptr()), _vp(st.data_ptr()),
                                    _vp(_stream_handle())), "csm_norm1")
    return float(out.item())


def pythagorean_residual(cos_part, sin_part, *, stream=None):
    """||C C + S S - I||_1 per matrix, on the device (csm_pythagorean_residual):
    the reference's accuracy witness for a computed pair (pkg/README.md:
    172-176, tests/test_driver.py:149-157).  Accepts one (n, n) pair or a
    batch (B, n, n); float64 or float32.  Returns a float for one pair,
    else a float64 array (numpy for host inputs, a CUDA tensor for device
    inputs)."""
    torch = _torch()
    single = (cos_part.ndim if hasattr(cos_part, "ndim") else np.asarray(cos_part).ndim) == 2
    cb = _as_batch(cos_part, batched=not single, f32_out=True)
    sb = _as_batch(sin_part, batched=not single, f32_out=True)
    c, s = cb.dev, sb.dev
    if c.shape != s.shape or c.dtype != s.dtype:
        raise ValueError("cos and sin parts must have the same shape and dtype")
    L = _lib.lib()
    B, n = int(c.shape[0]), int(c.shape[-1])
    out = torch.empty(B, dtype=torch.float64, device=c.device)
    ws_bytes = int(L.csm_residual_workspace_size(B, n))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=c.device)
    code = _lib.F32 if c.dtype == torch.float32 else _lib.F64
    _lib.check(L.csm_pythagorean_residual(code, _vp(c.data_ptr()), _vp(s.data_ptr()), B, n,
                                          _vp(out.data_ptr()), _vp(ws.data_ptr()), ws_bytes,
                                          _vp(_stream_handle(stream))),
               "csm_pythagorean_residual")
    if single:
        return float(out[0].item())
    return out if cb.host is None else out.cpu().numpy()


def matrix_from_rows(rows: Sequence[Sequence[float]]) -> np.ndarray:
    """Validated matrix from nested sequences (matcore.py:69-83)."""
    try:
        a = np.array(rows, dtype=np.float64)
    except ValueError as exc:
        raise MatrixInputError(f"ragged or non-numeric rows: {exc}") from None
    if a.ndim != 2 or a.shape[0] == 0 or a.shape[1] == 0:
        raise MatrixInputError(f"expected a 2-D matrix, got shape {a.shape}")
    if not np.isfinite(a).all():
        raise MatrixInputError("matrix entries must be finite")
    return a


def identity(n: int) -> np.ndarray:
    return np.eye(n, dtype=np.float64)


def read_matrix(path: str) -> np.ndarray:
    """Matrix text file: a "rows cols" header line, then one whitespace-
    separated line per row; blank lines are ignored (matcore.py:154-195).
    Every malformation raises MatrixInputError naming the file and line."""
    with open(path, "r", encoding="ascii") as fh:
        body = [ln.strip() for ln in fh]
    body = [ln for ln in body if ln]
    if not body:
        raise MatrixInputError(f"{path}: empty file (line 1: missing header)")
    head = body[0].split()
    if len(head) != 2:
        raise MatrixInputError(
            f"{path}: line 1: header must be 'rows cols', got {body[0]!r}")
    try:
        nr, nc = (int(v) for v in head)
    except ValueError:
        raise MatrixInputError(
            f"{path}: line 1: non-integer dimensions {body[0]!r}") from None
    if nr <= 0 or nc <= 0:
        raise MatrixInputError(f"{path}: line 1: dimensions must be positive")
    if len(body) != nr + 1:
        raise MatrixInputError(
            f"{path}: expected {nr} data lines, found {len(body) - 1}")
    rows = []
    for lineno, ln in enumerate(body[1:], start=2):
        fields = ln.split()
        if len(fields) != nc:
            raise MatrixInputError(f"{path}: line {lineno}: expected {nc} "
                                   f"entries, found {len(fields)}")
        try:
            rows.append([float(v) for v in fields])
        except ValueError:
            raise MatrixInputError(
                f"{path}: line {lineno}: non-numeric entry") from None
    try:
        return matrix_from_rows(rows)
    except MatrixInputError as exc:
        raise MatrixInputError(f"{path}: {exc}") from None


def write_matrix(path: str, a) -> None:
    """Write `a` in the format read_matrix accepts, each entry as repr()
    of its float64 value so the round trip is exact (matcore.py:198-204)."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    a = np.asarray(a, dtype=np.float64)
    nr, nc = a.shape
    with open(path, "w", encoding="ascii") as fh:
        fh.write(f"{nr} {nc}\n")
        for row in a:
            fh.write(" ".join(repr(float(v)) for v in row) + "\n")


_ENGINES = {"dmma": 0, "ozaki": 1, "auto": 2, "ozaki-unguarded": 3}


def set_engine(name: str) -> None:
    """Select the product engine of the tiled chain (n > 128) and the
    block-row chain, process-wide (csm_set_engine): "dmma" (FP64 DMMA, the
    default: componentwise error like the reference's fp64 GEMM), "ozaki"
    (Ozaki-II: exact int8 tensor-core GEMMs per modulus + CRT, for padded
    orders that are multiples of 256, every product guarded by a norm-wise
    a-priori error bound with a DMMA rerun), "auto" (Ozaki from padded
    order 768 up, DMMA below) or "ozaki-unguarded" (experiments only).
    Size workspaces (BatchPlan) after changing it."""
    if name not in _ENGINES:
        raise ValueError(f"engine must be one of {sorted(_ENGINES)}")
    _lib.check(_lib.lib().csm_set_engine(_ENGINES[name]), "csm_set_engine")


def get_engine() -> str:
    """The engine calls on this thread run with (a thread override from
    engine_scope, else the process default)."""
    code = int(_lib.lib().csm_get_engine())
    return {v: k for k, v in _ENGINES.items()}[code]


_TLS = threading.local()


@contextlib.contextmanager
def engine_scope(name: str):
    """Run the calls of this thread inside the block on `name`
    (csm_set_thread_engine), leaving the process default and other threads
    untouched; scopes nest.  Workspaces sized inside the block match the
    calls made in it."""
    if name not in _ENGINES:
        raise ValueError(f"engine must be one of {sorted(_ENGINES)}")
    L = _lib.lib()
    stack = getattr(_TLS, "engines", None)
    if stack is None:
        stack = _TLS.engines = []
    stack.append(_ENGINES[name])
    _lib.check(L.csm_set_thread_engine(_ENGINES[name]), "csm_set_thread_engine")
    try:
        yield
    finally:
        stack.pop()
        _lib.check(L.csm_set_thread_engine(stack[-1] if stack else -1),
                   "csm_set_thread_engine")


__all__ = [
    "BatchReport", "cos_sin", "engine_scope", "get_engine", "set_engine", "cos_sin_batched", "identity",
    "pade_cos_sin", "pade_cos_sin_batched",
    "matrix_from_rows", "norm1", "pythagorean_residual", "read_matrix", "select_batch",
    "select_scheme", "taylor_cos_sin", "taylor_sin9", "wave_cos_sin",
    "wave_cos_sin_batched", "wave_kernels", "wave_sin34", "write_matrix",
]
