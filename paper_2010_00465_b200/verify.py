"""Double-double reference values on the GPU.

The reference measures every scheme's accuracy against reference_cos_sin
(pkg/src/cossinm/verify.py:480-521): heavy scaling to ||A||_1 <= 2^-20, a
degree-12 Taylor pair and s doubling steps in compensated double-double
arithmetic.  In numpy each product is n passes of O(n^2) vector work, which
puts the 8192^2 configuration out of reach; here the same arithmetic runs
in csm_ddref_cos_sin (csrc/ddref.cu), element by element in the
reference's exact operation order, so the values are bit-identical to the
reference's (NaN payloads aside) and seconds instead of hours.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .api import _as_batch, _stream_handle, _torch, _vp
from .records import CosSinResult, CostLedger, MatrixInputError


def _to_host(x, host):
    if host == "numpy":
        return x.cpu().numpy()
    if host == "torch":
        return x.cpu()
    return x


def reference_cos_sin_batched(a, *, stream=None):
    """cos/sin reference values for a batch (B, n, n) of float64 matrices.
    Returns (cos, sin, s) with s the per-matrix doubling count (numpy int32).
    Raises OverflowError like the reference when norm / 2^-20 overflows."""
    torch = _torch()
    batch = _as_batch(a, batched=True, f32_out=True)
    x = batch.dev
    if x.dtype != torch.float64:
        raise TypeError("reference_cos_sin is float64-only on this path")
    B, n = int(x.shape[0]), int(x.shape[-1])
    L = _lib.lib()
    cos = torch.empty_like(x)
    sin = torch.empty_like(x)
    s = np.zeros(B, dtype=np.int32)
    st = np.zeros(B, dtype=np.int32)
    ws_bytes = int(L.csm_ddref_workspace_size(B, n))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=x.device)
    p = lambda arr: arr.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.check(L.csm_ddref_cos_sin(_vp(x.data_ptr()), _vp(cos.data_ptr()),
                                   _vp(sin.data_ptr()), B, n, p(s), p(st),
                                   _vp(ws.data_ptr()), ws_bytes,
                                   _vp(_stream_handle(stream))),
               "csm_ddref_cos_sin")
    if (st == _lib.SELECT_OVERFLOW).any():
        raise OverflowError("cannot convert float infinity to integer")
    return _to_host(cos, batch.host), _to_host(sin, batch.host), s


def reference_cos_sin(a) -> CosSinResult:
    """Drop-in for verify.reference_cos_sin (verify.py:480-521); the ledger
    charges 7 + 2 s products like the reference's."""
    shape = tuple(np.shape(a))
    if len(shape) != 2 or shape[0] != shape[1]:
        raise MatrixInputError(f"matrix must be square, got shape {shape}")
    torch = _torch()
    if isinstance(a, torch.Tensor):
        a = a.to(torch.float64)
    else:
        a = np.asarray(a, dtype=np.float64)
    c, s, sc = reference_cos_sin_batched(a[None])
    ledger = CostLedger()
    ledger.charge_product(7 + 2 * int(sc[0]))
    return CosSinResult(cos_part=c[0], sin_part=s[0], cost=ledger)


def dd_matmul(xh, xl, yh, yl=None):
    """The compensated product of verify.py:449-459 on the GPU: (hi, lo)
    of X Y for square (n, n) or batched (B, n, n) float64 operands; a low
    part of None is the zero matrix."""
    torch = _torch()
    single = np.ndim(xh) == 2
    parts = []
    host = None
    for v in (xh, xl, yh, yl):
        if v is None:
            parts.append(None)
            continue
        b = _as_batch(v[None] if single else v, batched=True, f32_out=True)
        if b.dev.dtype != torch.float64:
            raise TypeError("dd_matmul is float64-only")
        host = b.host
        parts.append(b.dev)
    x_h, x_l, y_h, y_l = parts
    B, n = int(x_h.shape[0]), int(x_h.shape[-1])
    oh = torch.empty_like(x_h)
    ol = torch.empty_like(x_h)
    ptr = lambda t: _vp(t.data_ptr() if t is not None else 0)  # noqa: E731
    _lib.check(_lib.lib().csm_dd_matmul(ptr(x_h), ptr(x_l), ptr(y_h), ptr(y_l),
                                        ptr(oh), ptr(ol), B, n,
                                        _vp(_stream_handle())), "csm_dd_matmul")
    if single:
        oh, ol = oh[0], ol[0]
    return _to_host(oh, host), _to_host(ol, host)


__all__ = ["dd_matmul", "reference_cos_sin", "reference_cos_sin_batched"]
