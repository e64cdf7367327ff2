"""Planned batched pipeline: buffers allocated once, stream-ordered runs.

``BatchPlan`` is the serving/benchmark form of cos_sin_batched /
wave_cos_sin_batched: it owns the device outputs, the (k, s, status) arrays
and the C-ABI workspace, so a run is one C call with no allocation and no
host synchronisation (n <= 64, and n <= 128 below the side-chain batch).
Such plans can also be captured once into a CUDA graph (``capture`` /
``replay``): the norm, selection, schedule and fused kernels then launch
as one graph, which is what small batches (launch-latency bound) want.  ``run_host`` streams a batch from pinned
host memory through the device and back in chunks on three CUDA streams
(H2D, compute, D2H), so the two PCIe directions and the kernels overlap.
"""
from __future__ import annotations

import ctypes

from . import _lib
from .records import _PREC_CODE, Precision


def _vp(x: int) -> ctypes.c_void_p:
    return ctypes.c_void_p(x)


class BatchPlan:
    """Pre-allocated pipeline for `batch` matrices of order n.

    dtype: torch.float64 or torch.float32 (float32 computes in float64 and
    stores float32).  wave=True plans the wave pair c(t^2 A), s(t, A)."""

    def __init__(self, batch: int, n: int, dtype=None, *,
                 precision: Precision = Precision.DOUBLE, wave: bool = False,
                 device=None, chunk: int | None = None):
        import torch
        self.torch = torch
        self.batch, self.n = int(batch), int(n)
        self.dtype = dtype or torch.float64
        self.code = _lib.F64 if self.dtype == torch.float64 else _lib.F32
        self.precision = precision
        self.wave = wave
        self.device = torch.device(device or "cuda")
        dev = self.device
        shape = (self.batch, self.n, self.n)
        self.cos = torch.empty(shape, dtype=self.dtype, device=dev)
        self.sin = torch.empty_like(self.cos)
        self.k = torch.empty(self.batch, dtype=torch.int32, device=dev)
        self.s = torch.empty_like(self.k)
        self.status = torch.empty_like(self.k)
        self.chunk = int(chunk or self.batch) or 1
        L = _lib.lib()
        self.ws_bytes = int(L.csm_workspace_size(self.code, self.chunk, self.n))
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8,
                              device=dev)
        self._a_dev = None
        self._t_dev = None
        self._streams = None
        self.launches = 0

    # -- one C-ABI call on a contiguous slice [lo, hi) -----------------------
    def _call(self, a_ptr: int, lo: int, hi: int, stream_handle: int,
              t_ptr: int | None) -> None:
        L = _lib.lib()
        esz = self.cos.element_size()
        nn = self.n * self.n
        cnt = hi - lo
        out = [_vp(self.cos.data_ptr() + lo * nn * esz),
               _vp(self.sin.data_ptr() + lo * nn * esz), cnt, self.n,
               _vp(self.k.data_ptr() + 4 * lo), _vp(self.s.data_ptr() + 4 * lo),
               _vp(self.status.data_ptr() + 4 * lo), _vp(self.ws.data_ptr()),
               self.ws_bytes, _vp(stream_handle)]
        if self.wave:
            rc = L.csm_wave(self.code, _PREC_CODE[self.precision], _vp(a_ptr),
                            _vp(t_ptr), *out)
        else:
            rc = L.csm_cos_sin(self.code, _PREC_CODE[self.precision],
                               _vp(a_ptr), *out)
        _lib.check(rc, "csm_wave" if self.wave else "csm_cos_sin")
        self.launches += int(L.csm_last_launch_count())

    def run(self, a, t=None, stream=None):
        """Device-resident run on the whole batch (a: CUDA tensor, C-order).
        Returns (cos, sin, k, s, status) device tensors; no host sync."""
        torch = self.torch
        if a.shape != (self.batch, self.n, self.n) or a.dtype != self.dtype:
            raise ValueError("input does not match the plan")
        a = a.contiguous()
        st = stream or torch.cuda.current_stream()
        h = int(st.cuda_stream)
        tp = None
        if self.wave:
            tp = t.contiguous().data_ptr()
        esz = a.element_size()
        nn = self.n * self.n
        tsz = 8
        for lo in range(0, self.batch, self.chunk):
            hi = min(self.batch, lo + self.chunk)
            self._call(a.data_ptr() + lo * nn * esz, lo, hi, h,
                       None if tp is None else tp + lo * tsz)
        return self.cos, self.sin, self.k, self.s, self.status

    @property
    def graph_safe(self) -> bool:
        return bool(_lib.lib().csm_graph_safe(self.code, self.chunk, self.n))

    def capture(self, a, t=None):
        """Capture run(a, t) into a CUDA graph; `a` (and t) become the
        graph's static inputs -- copy new data into them, then replay()."""
        torch = self.torch
        if not self.graph_safe:
            raise RuntimeError("this plan synchronises the host (tiled chain); "
                               "it cannot be captured in a CUDA graph")
        self._g_a = a.contiguous()
        self._g_t = None if t is None else t.contiguous()
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up outside the capture
            self.run(self._g_a, self._g_t)
        torch.cuda.current_stream().wait_stream(side)
        self._graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._graph):
            self.run(self._g_a, self._g_t)
        return self._g_a

    def replay(self):
        """Replay the captured run on the current stream; returns the same
        (cos, sin, k, s, status) tensors as run()."""
        self._graph.replay()
        return self.cos, self.sin, self.k, self.s, self.status

    def capture_host(self, a_host, cos_host, sin_host, t_host=None):
        """Capture host -> device -> host in ONE CUDA graph: the H2D copy of
        the pinned input, the (graph-safe) run and the D2H copies of cos and
        sin into the pinned outputs.  For repeated small calls (latency
        bound, configs[0]): refill a_host, replay_host(), synchronize, read."""
        torch = self.torch
        if not self.graph_safe:
            raise RuntimeError("this plan synchronises the host (tiled chain); "
                               "it cannot be captured in a CUDA graph")
        for x in (a_host, cos_host, sin_host) + ((t_host,) if self.wave else ()):
            if not x.is_pinned():
                raise ValueError("capture_host needs pinned host tensors")
        if self._a_dev is None:
            self._a_dev = torch.empty((self.batch, self.n, self.n), dtype=self.dtype,
                                      device=self.device)
            if self.wave:
                self._t_dev = torch.empty(self.batch, dtype=torch.float64,
                                          device=self.device)

        def body():
            self._a_dev.copy_(a_host, non_blocking=True)
            if self.wave:
                self._t_dev.copy_(t_host, non_blocking=True)
            self.run(self._a_dev, self._t_dev)
            cos_host.copy_(self.cos, non_blocking=True)
            sin_host.copy_(self.sin, non_blocking=True)

        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up outside the capture
            body()
        torch.cuda.current_stream().wait_stream(side)
        self._host_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._host_graph):
            body()

    def replay_host(self):
        """Replay the captured host round trip on the current stream."""
        self._host_graph.replay()

    def run_host(self, a_host, cos_host, sin_host, t_host=None,
                 chunks: int = 8) -> None:
        """Host->device->host run: pinned CPU tensors in and out, chunked
        over H2D / compute / D2H streams.  Ends with the current stream
        waiting on the last D2H copy (call synchronize to read results).
        The host input buffer is read asynchronously: do not overwrite it
        until the current stream has passed this call."""
        torch = self.torch
        if self._a_dev is None:
            self._a_dev = torch.empty((self.batch, self.n, self.n),
                                      dtype=self.dtype, device=self.device)
            if self.wave:
                self._t_dev = torch.empty(self.batch, dtype=torch.float64,
                                          device=self.device)
            self._streams = [torch.cuda.Stream(device=self.device)
                             for _ in range(3)]
        if self.chunk < (self.batch + chunks - 1) // chunks:
            chunks = (self.batch + self.chunk - 1) // self.chunk
        s_h2d, s_cmp, s_d2h = self._streams
        cur = torch.cuda.current_stream()
        step = (self.batch + chunks - 1) // chunks
        # Back-to-back calls pipeline across the call boundary: the next
        # call's H2D of chunk j only waits for THIS call's compute of chunk j
        # (the one reader of that input slice), so it overlaps this call's
        # remaining D2H -- the two PCIe directions stay busy together.
        prev = self._cmp_done if getattr(self, "_pipe_step", None) == step else None
        s_cmp.wait_stream(cur)  # outputs are rewritten: after the caller's work
        if prev is None:
            s_h2d.wait_stream(cur)
        self._pipe_step = step
        self._cmp_done = []
        nn = self.n * self.n
        esz = self._a_dev.element_size()
        for j, lo in enumerate(range(0, self.batch, step)):
            hi = min(self.batch, lo + step)
            if prev is not None:
                s_h2d.wait_event(prev[j])
            with torch.cuda.stream(s_h2d):
                self._a_dev[lo:hi].copy_(a_host[lo:hi], non_blocking=True)
                if self.wave:
                    self._t_dev[lo:hi].copy_(t_host[lo:hi], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_h2d)
            s_cmp.wait_event(ev_in)
            for clo in range(lo, hi, self.chunk):
                chi = min(hi, clo + self.chunk)
                self._call(self._a_dev.data_ptr() + clo * nn * esz, clo, chi,
                           int(s_cmp.cuda_stream),
                           None if not self.wave
                           else self._t_dev.data_ptr() + 8 * clo)
            ev_out = torch.cuda.Event()
            ev_out.record(s_cmp)
            self._cmp_done.append(ev_out)
            s_d2h.wait_event(ev_out)
            with torch.cuda.stream(s_d2h):
                cos_host[lo:hi].copy_(self.cos[lo:hi], non_blocking=True)
                sin_host[lo:hi].copy_(self.sin[lo:hi], non_blocking=True)
        cur.wait_stream(s_d2h)
        cur.wait_stream(s_cmp)
