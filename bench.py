#!/usr/bin/env python
"""Benchmark of the B200 cos/sin hot path (BASELINE.json metric).

Default workload (configs[1]): a batch of 16384 float64 64x64 matrices,
N(0,1) entries rescaled to 1-norm log-uniform in [1e-3, 1e2], cos+sin in the
fused shared-memory kernel.  One step = one pass of the whole pipeline
(norm, (k, s) selection, chain, doubling) over the batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg2|cfg1|cfg3|cfg4|cfg5|sweep64..1024]
                  [--engine auto|dmma|ozaki] [--dist-mode gather|peer]

N > 1 runs under torchrun, one rank per GPU: every rank owns its own
16384-matrix shard (weak scaling, no collective on the data path); the step
time is the max over ranks.  --impl reference times the reference algorithm
(the oracle port, oracle/cossin_oracle.py) on the host cores with a process
pool, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("matrices/sec and FP64 TFLOP/s (fraction of DMMA peak) for batched "
          "cos+sin at n=64-1024")

CONFIGS = {
    # name: (kind, batch, n, dtype, precision, description)
    "cfg1": ("cfg1", 1, 64, "f64", "double",
             "single 64x64 f64, N(0,1) seed 0, 1-norm 2.0"),
    "cfg2": ("cfg2", 16384, 64, "f64", "double",
             "16384 x 64x64 f64, N(0,1), 1-norm log-uniform [1e-3, 1e2]"),
    "cfg3": ("cfg3", 4096, 256, "f32", "single",
             "4096 x 256x256 f32, U(-1,1), 1-norm log-uniform [1e-2, 50]"),
    "cfg4": ("cfg4", 512, 512, "f64", "double",
             "wave pair, 512 x 512x512 SPD Laplacian*(n+1)^2 + diag U(0,10),"
             " t log-uniform [1e-4, 1e-1]"),
    "cfg5": ("cfg5", 1, 8192, "f64", "double",
             "one 8192x8192 f64 symmetric 20*(G+G^T)/(2 sqrt n)"),
}
for _n in (64, 128, 256, 512, 1024):
    _b = max(1, (1 << 30) // (_n * _n * 8))
    CONFIGS[f"sweep{_n}"] = ("cfg2", _b, _n, "f64", "double",
                             f"{_b} x {_n}x{_n} f64, cfg2 distribution "
                             "(~1 GiB input)")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# Inputs (seeded synthetic data with the configs' shapes and distributions).

def make_inputs(kind: str, batch: int, n: int, seed: int):
    import numpy as np
    rng = np.random.default_rng(seed)
    t = None
    if kind == "cfg1":
        g = np.random.default_rng(0).standard_normal((64, 64))
        a = (g * (2.0 / np.abs(g).sum(axis=0).max()))[None]
    elif kind == "cfg5":
        g = np.random.default_rng(seed).standard_normal((n, n))
        a = (20.0 * (g + g.T) / (2.0 * math.sqrt(n)))[None]
    else:
        from oracle.cpu_pool import _gen  # same generator as the CPU leg
        a, t = _gen(kind, seed, batch, n)
    return a, t


# ---------------------------------------------------------------------------
# Clock sampling during the timed region.

class ClockSampler:
    """Samples SM clock, power and throttle reasons during the timed region
    (NVML at ~2 ms; nvidia-smi as a fallback)."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
             "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, power_w, set(reasons))
        self._stop = threading.Event()
        self._th = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = None
            try:  # match the torch device by PCI bus id (NVML ignores CUDA_VISIBLE_DEVICES)
                import torch
                pr = torch.cuda.get_device_properties(index)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self._h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        pw = nv.nvmlDeviceGetPowerUsage(self._h) / 1000.0
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        masks = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
                 "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        reasons = {k for k, m in masks.items() if bits & m}
        self.rows.append((float(sm), float(self._max), pw, reasons))

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,"
             "clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                              "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        if out:
            f = [x.strip() for x in out.split(",")]
            reasons = {n for n, v in zip(self.NAMES, f[3:7]) if v.lower() == "active"}
            self.rows.append((float(f[0]), float(f[1]), float(f[2]), reasons))

    def _loop(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    self._sample_nvml()
                    self._stop.wait(0.002)
                else:
                    self._sample_smi()
                    self._stop.wait(0.05)
            except Exception:
                self._stop.wait(0.05)

    def __enter__(self):
        self._th = threading.Thread(target=self._loop, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"],
                    "samples": 0}
        reasons = set()
        for r in self.rows:
            reasons |= r[3]
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(reasons), "samples": len(self.rows),
                "power_w_max": max(r[2] for r in self.rows),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# ---------------------------------------------------------------------------

def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_dict(args, cfg, world):
    """The `config` object, identical in both arms (--impl ours|reference)."""
    kind, batch, n, dt, prec, desc = cfg
    esz = 4 if dt == "f32" else 8
    if kind == "cfg5":
        par = f"block-row x{world}"
    else:
        par = f"batch shard x{world} (no collective)"
    return {"workload": args.config, "description": desc, "batch_per_gpu": batch, "n": n,
            "precision_table": prec,
            "l2": ("inputs larger than L2 (no flush needed)" if batch * n * n * esz > 2 * 126e6
                   else "input fits L2; steps reuse it (no flush)"),
            "parallelism": par}


def host_info():
    """CPU model, core count and the BLAS numpy runs on."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        import numpy  # noqa: F401  (loads its BLAS)
        for lib in threadpool_info():
            if lib.get("user_api") == "blas":
                blas = f"{lib.get('internal_api')} {lib.get('version')} ({lib.get('num_threads')} threads)"
                break
    except Exception:
        pass
    import numpy as np
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "blas": blas,
            "numpy": np.__version__}


PORT_NOTE = ("oracle/cossin_oracle.py restates the reference's numpy path call for call; "
             "it skips the reference's per-call Fraction->float coefficient conversions, "
             "so if anything it flatters the CPU")


def cpu_baseline_leg(kind, n, seconds):
    from oracle.cpu_pool import run_pool
    per_worker = {"cfg2": 256, "cfg3": 8, "cfg4": 2}.get(kind, 64)
    rate, workers, done, secs = run_pool(kind, n, per_worker,
                                         min_seconds=seconds)
    return rate, workers, done, secs, per_worker


def run_reference(args, cfg):
    """--impl reference: the reference algorithm (oracle port) on the host
    cores, K timed steps after W warm-up steps, each a bounded sample."""
    world, rank, _ = dist_setup(args)
    kind, batch, n, dt, prec, desc = cfg
    if rank != 0:
        return
    if kind == "cfg1":
        from oracle import cossin_oracle as orc
        a, _ = make_inputs(kind, batch, n, 0)
        times = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            orc.cos_sin(a[0])
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
        rate = 1.0 / statistics.mean(times)
        ms_step = 1e3 * statistics.mean(times)
        cores, sample = os.cpu_count(), f"{args.steps} full cos_sin calls (one process)"
    elif kind == "cfg5":
        # one full call is ~80 s of dgemm: each step times ONE of its k + 2s
        # products (numpy @, all BLAS threads) and the rate charges all of
        # them; the linear combinations are left out (flatters the CPU)
        import numpy as np
        from oracle import cossin_oracle as orc
        a, _ = make_inputs(kind, batch, n, 0)
        k, sc = orc.select(orc.norm1(a[0]))
        x = np.ascontiguousarray(a[0] * 2.0 ** -sc)
        times = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            _ = x @ x
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
        per_matrix = (k + 2 * sc) * statistics.mean(times)
        rate = 1.0 / per_matrix
        ms_step = 1e3 * per_matrix
        cores = os.cpu_count()
        sample = (f"one {n}^2 dgemm per step (numpy @, all BLAS threads) x {k + 2 * sc} "
                  "products per matrix; linear combinations not timed")
    else:
        per_step = max(1.0, 60.0 / max(1, args.steps + args.warmup))
        rates = []
        for i in range(args.warmup + args.steps):
            rate_i, workers, done, secs, pw = cpu_baseline_leg(kind, n, per_step)
            if i >= args.warmup:
                rates.append(rate_i)
        rate = statistics.mean(rates)
        ms_step = 1e3 * batch / rate  # one step's batch at the measured rate
        cores = workers
        sample = (f"{workers} processes x 1 BLAS thread, each re-running "
                  f"{pw} seeded {desc.split(',')[0]} matrices for >= "
                  f"{per_step:.1f} s per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate,
        "unit": "matrices/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong" if kind == "cfg5" else "weak",
        "vs_baseline": None,
        "dtype": "f64" if dt == "f64" else "f32 storage, f64 compute",
        "data": "synthetic (seeded)",
        "config": config_dict(args, cfg, args.gpus),
        "cpu_baseline": {"value": rate, "unit": "matrices/s", "cores": cores,
                         "kind": "port", "sample": sample, "host": host_info(),
                         "note": PORT_NOTE},
        "e2e": {"value": rate, "unit": "matrices/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_cfg5(args, cfg):
    """configs[4]: one 8192^2 matrix, block-row over the ranks with an NCCL
    all-gather of the current right operand per product (distchain.py);
    strong scaling (the total work is fixed)."""
    import numpy as np
    import torch

    from paper_2010_00465_b200 import _lib, distchain
    from paper_2010_00465_b200 import dist as pdist
    world, rank, local = dist_setup(args)
    kind, batch, n, dt, prec, desc = cfg
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peer = args.dist_mode == "peer"
    if world > 1 or peer:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29571")
        if not dist.is_initialized():
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    chain = distchain.cos_sin_distributed_peer if peer else distchain.cos_sin_distributed
    a_np, _ = make_inputs(kind, 1, n, seed=0)  # the same matrix on every rank
    a_host = torch.from_numpy(np.ascontiguousarray(a_np[0])).pin_memory()
    a = a_host.to(dev)
    c, s_, st = chain(a, gather_outputs=True)
    torch.cuda.synchronize()
    flops = 2.0 * n ** 3 * (st.k + 2 * st.s)
    M, row0 = n // world, rank * (n // world)
    parity = cfg5_parity(a_np[0], c, s_, st, args) if rank == 0 else None
    del c, s_
    for _ in range(args.warmup):
        chain(a, gather_outputs=False)
    L = _lib.lib()
    oz = ozaki_applies(n) and not peer
    if oz:
        L.csm_profile_enable(2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            chain(a, gather_outputs=False)
        e1.record()
        torch.cuda.synchronize()
    gemm_ms = ctypes_collect(L)[0] / args.steps if oz else 0.0
    L.csm_profile_enable(0)
    ms_step = pdist.max_over_ranks(e0.elapsed_time(e1) / args.steps, device=dev)
    # e2e: H2D of A on every rank, compute, D2H of each rank's output rows
    c_host = torch.empty((M, n), dtype=torch.float64).pin_memory()
    s_host = torch.empty_like(c_host).pin_memory()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e2.record()
    for _ in range(max(1, min(args.steps, 3))):
        ad = a_host.to(dev, non_blocking=True)
        cr, sr, _ = chain(ad, gather_outputs=False)
        c_host.copy_(cr, non_blocking=True)
        s_host.copy_(sr, non_blocking=True)
    e3.record()
    torch.cuda.synchronize()
    e2e_ms = pdist.max_over_ranks(e2.elapsed_time(e3) / max(1, min(args.steps, 3)), device=dev)
    peak = None
    if rank == 0:
        pk = ctypes.c_double(0.0)
        if L.csm_fp64_peak(20000, ctypes.byref(pk), None) == 0:
            peak = pk.value
    if rank == 0:
        tfl = flops / (ms_step * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": 1.0 / (ms_step * 1e-3), "unit": "matrices/s",
            "tflops": tfl, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": {"workload": args.config, "description": desc, "n": n,
                       "k": st.k, "s": st.s, "gathers_per_step": st.gathers,
                       "engine": "ozaki" if oz else "dmma",
                       "parallelism": (f"block-row x{world}, right operand read from peer "
                                       "slabs inside the GEMM (symmetric memory, no gather)"
                                       if peer else
                                       f"block-row x{world}, NCCL all-gather per product")},
            "roofline": ozaki_roofline(16 * flops / world, gemm_ms, tfl, peak) if oz else
                        {"bound": "tensor", "achieved": tfl, "peak": peak, "unit": "TFLOP/s",
                         "frac": (tfl / peak) if peak else None, "traffic": None,
                         "kernel": "gemm_epi_kernel (slab mode) + all-gathers",
                         "peak_source": "csm_fp64_peak on this GPU in this run"},
            "e2e": {"value": 1.0 / (e2e_ms * 1e-3), "unit": "matrices/s",
                    "h2d_bytes_per_step": n * n * 8, "d2h_bytes_per_step": 2 * M * n * 8,
                    "ms_per_step": e2e_ms},
            "gpu_launches": st.launches * args.steps,
            "clocks": clk.summary(), "cpu_baseline": None, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


def cfg5_parity(a_np, c, s, st, args):
    """Parity of the cfg5 output (outside the timed region): (k, s) against
    the oracle's selection, cos/sin against the double-double GPU truth
    (verify.reference_cos_sin; tests/test_gpu_fullsize.py gates the same
    output against the oracle itself), symmetry, and the Pythagorean
    residual ||C^2 + S^2 - I||_1 / max(1, ||C||_1^2)."""
    import numpy as np
    import torch

    import paper_2010_00465_b200 as csm
    from oracle import cossin_oracle as orc
    from paper_2010_00465_b200 import verify
    k, sc = orc.select(orc.norm1(a_np), "taylor", "double")
    assert (st.k, st.s) == (k, sc), ((st.k, st.s), (k, sc))
    out = {"ks_checked": 1, "ks_mismatches": 0}
    sym = float((c - c.T).abs().max() / c.abs().max())
    assert sym <= 1e-10, sym
    out["cos_asymmetry"] = sym
    res = float(csm.pythagorean_residual(c[None], s[None])[0])
    cn = float(c.abs().sum(dim=0).max())
    out["pythagorean"] = {"max": res / max(1.0, cn * cn), "max_abs": res,
                          "normalised_by": "max(1, ||C||_1^2)", "matrices": 1}
    if not args.no_truth:
        truth = verify.reference_cos_sin(a_np)

        def rel(x, y):
            y = torch.as_tensor(np.asarray(y), device=x.device)
            return float((x - y).abs().sum(dim=0).max() / y.abs().sum(dim=0).max())
        ec, es = rel(c, truth.cos_part), rel(s, truth.sin_part)
        out["truth"] = {"oracle": "double-double GPU reference (verify.py:480-521)",
                        "rel1_err_cos": ec, "rel1_err_sin": es}
        assert max(ec, es) <= 1e-9, (ec, es)
    return out


def parity_block(kind, a_np, t_np, prec, dt, plan, ks, ss, rank):
    """Parity summary carried in the bench line (computed outside the timed
    region): the oracle on a spot-check sample at the parity gate (1e-5
    fp32; 1e-12 fp64, or for the wave config and n >= 256 max(1e-12, 4 x
    the oracle's own permuted-order noise)), (k, s) of EVERY matrix against the
    oracle's selection, and the Pythagorean residual ||C^2 + S^2 - I||_1 /
    max(1, ||C||_1^2) over the whole batch (csm_pythagorean_residual)."""
    import numpy as np
    import torch

    import paper_2010_00465_b200 as csm
    from oracle import cossin_oracle as orc
    from tests._util import pair_close, permuted_noise
    wave = kind == "cfg4"
    batch, n = a_np.shape[0], a_np.shape[-1]
    fam = "wave" if wave else "taylor"
    mism = 0
    for i in range(batch):
        a64 = a_np[i].astype(np.float64)
        nrm = orc.norm1(a_np[i]) if dt == "f32" else orc.norm1(a64)
        if wave:
            nrm = float(t_np[i]) * float(t_np[i]) * nrm
        k, s = orc.select(nrm, fam, prec)
        mism += int((k, s) != (int(ks[i]), int(ss[i])))
    assert mism == 0, f"{mism} (k, s) mismatches against the oracle's selection"
    m = min(batch, 4 if n >= 512 else 8)
    rng = np.random.default_rng(31)
    worst_c = worst_s = 0.0
    gates = []
    for i in range(m):
        if wave:
            fn = lambda x: orc.wave_cos_sin(x, float(t_np[i]), prec)  # noqa: E731
            (c, s, k, sc), noise = permuted_noise(fn, a_np[i], rng)
            gate = max(1e-12, 4.0 * noise)
        elif dt == "f32":
            c, s, k, sc = orc.cos_sin(a_np[i].astype(np.float64), prec)
            gate = 1e-5
        elif n >= 256:  # the reference's own noise can exceed 1e-12 here
            fn = lambda x: orc.cos_sin(x, prec)  # noqa: E731
            (c, s, k, sc), noise = permuted_noise(fn, a_np[i], rng)
            gate = max(1e-12, 4.0 * noise)
        else:
            c, s, k, sc = orc.cos_sin(a_np[i].astype(np.float64), prec)
            gate = 1e-12
        assert (int(ks[i]), int(ss[i])) == (k, sc), (i, ks[i], ss[i], k, sc)
        okc, ec = pair_close(plan.cos[i].double().cpu().numpy(), c, s, gate)
        oks, es = pair_close(plan.sin[i].double().cpu().numpy(), s, c, gate)
        assert okc and oks, (i, ec, es, gate)
        worst_c, worst_s = max(worst_c, ec), max(worst_s, es)
        gates.append(gate)
    out = {"spot_checked": m, "gate_max": max(gates), "max_rel1_err_cos": worst_c,
           "max_rel1_err_sin": worst_s, "ks_checked": batch, "ks_mismatches": mism,
           "oracle": "oracle/cossin_oracle.py (pinned to the reference's goldens)"}
    if wave:
        out["pythagorean"] = None  # c^2 + A s^2 = I for the wave pair; not C^2 + S^2
    else:
        res = csm.pythagorean_residual(plan.cos, plan.sin)
        cn = torch.empty(batch, dtype=torch.float64, device=plan.cos.device)
        st = torch.empty(batch, dtype=torch.int32, device=plan.cos.device)
        from paper_2010_00465_b200 import _lib
        _lib.check(_lib.lib().csm_norm1(plan.code, ctypes.c_void_p(plan.cos.data_ptr()), batch, n,
                                        ctypes.c_void_p(cn.data_ptr()),
                                        ctypes.c_void_p(st.data_ptr()), None), "csm_norm1")
        rel = (res / torch.clamp(cn * cn, min=1.0)).cpu().numpy()
        out["pythagorean"] = {"max": float(rel.max()), "median": float(np.median(rel)),
                              "max_abs": float(res.max().item()),
                              "normalised_by": "max(1, ||C||_1^2)", "matrices": batch}
    return out


def run_ours(args, cfg):
    import numpy as np
    import torch

    import paper_2010_00465_b200 as csm
    from paper_2010_00465_b200 import _lib
    from paper_2010_00465_b200.plan import BatchPlan

    world, rank, local = dist_setup(args)
    kind, batch, n, dt, prec, desc = cfg
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist

    def barrier():
        if pg is not None:
            pg.barrier()

    from paper_2010_00465_b200 import dist as pdist

    def max_over_ranks(x: float) -> float:
        return pdist.max_over_ranks(x, device=dev)

    def sum_over_ranks(x: float) -> float:
        return pdist.sum_over_ranks(x, device=dev)

    a_np, t_np = make_inputs(kind, batch, n, seed=rank)
    tdtype = torch.float32 if dt == "f32" else torch.float64
    a_np = a_np.astype(np.float32 if dt == "f32" else np.float64)
    precision = csm.Precision.SINGLE if prec == "single" else csm.Precision.DOUBLE
    wave = kind == "cfg4"
    plan = BatchPlan(batch, n, tdtype, precision=precision, wave=wave,
                     device=dev)
    a_dev = torch.from_numpy(a_np).to(dev)
    t_dev = torch.from_numpy(t_np).to(dev) if wave else None

    # parity against the oracle and the Pythagorean residual over the whole
    # batch (outside the timed region)
    plan.run(a_dev, t_dev)
    torch.cuda.synchronize()
    st = plan.status.cpu().numpy()
    assert not st.any(), "non-zero status in bench inputs"
    ks = plan.k.cpu().numpy().astype(np.int64)
    ss = plan.s.cpu().numpy().astype(np.int64)
    parity = parity_block(kind, a_np, t_np, prec, dt, plan, ks, ss, rank)
    flops_step = float((2.0 * n ** 3 * (ks + 2 * ss)).sum())

    # warm-up, then K timed steps between barriers + synchronize
    for _ in range(args.warmup):
        plan.run(a_dev, t_dev)
    torch.cuda.synchronize()
    L = _lib.lib()
    oz = ozaki_applies(n)
    L.csm_profile_enable(2 if oz else 1)
    # small batches are launch-latency bound: replay the pipeline as one CUDA
    # graph (norm, selection, schedule and fused kernels; BatchPlan.capture)
    use_graph = batch <= 64 and plan.graph_safe
    step_fn = lambda: plan.run(a_dev, t_dev)  # noqa: E731
    per_run = 0
    if use_graph:
        L.csm_profile_enable(0)
        plan.launches = 0
        plan.run(a_dev, t_dev)
        per_run = plan.launches
        plan.capture(a_dev, t_dev)
        for _ in range(args.warmup):
            plan.replay()
        step_fn = plan.replay
        L.csm_profile_enable(2 if oz else 1)
    plan.launches = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            step_fn()
        e1.record()
        torch.cuda.synchronize()
    barrier()
    ms_total = e0.elapsed_time(e1)
    kern_ms = ctypes_collect(L)
    L.csm_profile_enable(0)
    launches = per_run * args.steps if use_graph else plan.launches
    # the fused K0 launch (norm1 + finiteness + selection, n <= 128) timed on
    # its own after the timed region: the HBM-bound part of a step
    k0 = None
    if n <= 128 and batch > 148 and not use_graph and os.environ.get("CSM_K0_FUSED", "1") != "0":
        L.csm_profile_enable(3)
        for _ in range(5):
            plan.run(a_dev, t_dev)
        torch.cuda.synchronize()
        k0_ms, k0_cnt = ctypes_collect(L)
        L.csm_profile_enable(0)
        plan.launches = launches
        if k0_cnt:
            k0 = hbm_roofline(batch * n * n * (4 if dt == "f32" else 8), k0_ms / k0_cnt)
    ms_step = max_over_ranks(ms_total / args.steps)
    units = sum_over_ranks(float(batch))
    value = units / (ms_step * 1e-3)
    tflops = sum_over_ranks(flops_step) / (ms_step * 1e-3) / 1e12

    # e2e through the public plan API from pinned host memory
    a_host = torch.from_numpy(a_np).pin_memory()
    c_host = torch.empty(a_host.shape, dtype=tdtype).pin_memory()
    s_host = torch.empty_like(c_host).pin_memory()
    t_host = torch.from_numpy(t_np).pin_memory() if wave else None
    e2e_steps = max(1, min(args.steps, 10))
    chunks = int(os.environ.get("CSM_E2E_CHUNKS", "16"))
    if use_graph:  # small batch: the whole host round trip as one graph (capture_host)
        plan.capture_host(a_host, c_host, s_host, t_host)
        e2e_call = plan.replay_host
        e2e_mode = "BatchPlan.capture_host graph replay (H2D + run + D2H)"
    else:
        e2e_call = lambda: plan.run_host(a_host, c_host, s_host, t_host,  # noqa: E731
                                         chunks=chunks)
        e2e_mode = f"BatchPlan.run_host ({chunks} chunks over H2D / compute / D2H streams)"
    for _ in range(2):
        e2e_call()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(e2e_steps):
        e2e_call()
        if use_graph:
            torch.cuda.current_stream().synchronize()
        _ = float(c_host[batch - 1, n - 1, n - 1])  # host read of the result
    e3.record()
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(e2.elapsed_time(e3) / e2e_steps)
    assert np.allclose(c_host[0].double().numpy(),
                       plan.cos[0].double().cpu().numpy())
    esz = 4 if dt == "f32" else 8
    h2d = batch * n * n * esz + (batch * 8 if wave else 0)
    d2h = 2 * batch * n * n * esz

    peak = None
    if rank == 0:
        pk = ctypes.c_double(0.0)
        if L.csm_fp64_peak(20000, ctypes.byref(pk), None) == 0:
            peak = pk.value
    if use_graph:  # graph replays carry no library-side events: the step is the kernel interval
        kern_ms = (ms_total, args.steps)
    kern_avg_ms = kern_ms[0] / max(kern_ms[1], 1)
    achieved = flops_step / (kern_avg_ms * 1e-3) / 1e12 if kern_avg_ms > 0 else None
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof_json):
        try:
            traffic = json.load(open(prof_json)).get(args.config)
        except Exception:
            traffic = None

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline and kind == "cfg1":
        from oracle import cossin_oracle as orc
        a0 = a_np[0].astype(np.float64)
        calls, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < args.cpu_seconds:
            orc.cos_sin(a0)
            calls += 1
        secs = time.perf_counter() - t0
        cpu = {"value": calls / secs, "unit": "matrices/s", "cores": 1, "kind": "port",
               "sample": f"oracle port of cos_sin on the cfg1 matrix, {calls} sequential "
                         f"calls in {secs:.1f} s (one process)",
               "host": host_info(), "note": PORT_NOTE}
    elif world == 1 and not args.no_cpu_baseline and kind != "cfg5":
        rate, workers, done, secs, pw = cpu_baseline_leg(kind, n, args.cpu_seconds)
        cpu = {"value": rate, "unit": "matrices/s", "cores": workers,
               "kind": "port",
               "sample": (f"oracle port of cos_sin/wave_cos_sin on {done} "
                          f"matrices ({workers} processes x {pw} seeded "
                          f"{desc.split(',')[0]} inputs, 1 BLAS thread each, "
                          f"{secs:.1f} s)"),
               "host": host_info(), "note": PORT_NOTE}
    clocks = clk.summary()
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "matrices/s",
        "tflops": tflops,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64" if dt == "f64" else "f32 storage, f64 compute",
        "data": "synthetic (seeded; per-rank shard seed = rank)",
        "config": config_dict(args, cfg, world),
        "engine": "ozaki" if oz else "dmma",
        "mean_products": float((ks + 2 * ss).mean()),
        "parity": parity,
        "roofline": ozaki_roofline((9 if dt == "f32" else 16) * flops_step,
                                   kern_ms[0] / args.steps, tflops, peak) if oz else
                    {"bound": "tensor", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s",
                     "frac": (achieved / peak) if (achieved and peak) else None,
                     "traffic": traffic,
                     "kernel": (("fused64d_kernel (K1d, two CTAs per SM)"
                                 if kind != "cfg4" and os.environ.get("CSM_K1D", "1") != "0"
                                 and batch > 148 else "fused64_kernel (K1)") if n <= 64 else
                                "fused64_kernel<4> (K1c, 4-CTA clusters) + side tiled chain, "
                                "timed as one interval" if n <= 128 else
                                "gemm_epi_kernel (tiled chain)"),
                     "peak_source": "csm_fp64_peak: DMMA m8n8k4 loop on this "
                                    "GPU in this run (MEASURED_PEAKS.json has "
                                    "no FP64 entry)",
                     "flops_per_step": flops_step,
                     "kernel_ms_per_step": kern_avg_ms},
        "roofline_k0": k0,
        "e2e": {"value": batch * world / (e2e_ms * 1e-3), "unit": "matrices/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms, "mode": e2e_mode},
        "gpu_launches": launches,
        "launch_mode": "CUDA graph replay (BatchPlan.capture)" if use_graph else "stream launches",
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


import ctypes  # noqa: E402

# Ozaki engine: nominal dense int8 tensor peak of a B200 (the fp8 figure of
# /opt/skills/guides/B200_PROFILING.md; MEASURED_PEAKS.json has no int8 entry)
INT8_PEAK_TOPS = 4500.0


def ozaki_applies(n):
    """The Ozaki engine runs a call when NP % 256 == 0 and it is selected
    (or auto and NP >= 768)."""
    import paper_2010_00465_b200 as csm
    np_ = (n + 63) // 64 * 64
    eng = csm.get_engine()
    return n > 128 and np_ % 256 == 0 and (eng.startswith("ozaki") or (eng == "auto" and np_ >= 768))


def ozaki_roofline(int8_ops_step, gemm_ms, fp64_tflops, dmma_peak):
    """Roofline object of the Ozaki engine's dominant kernel, oz_gemm (one
    tcgen05 int8 GEMM per modulus): int8 ops per step / its live CUDA-event
    time, against the int8 tensor peak; the fp64-equivalent rate is reported
    beside it as a multiple of the measured DMMA peak."""
    achieved = int8_ops_step / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    return {"bound": "tensor", "achieved": achieved, "peak": INT8_PEAK_TOPS, "unit": "TOPS",
            "frac": (achieved / INT8_PEAK_TOPS) if achieved else None, "traffic": None,
            "kernel": "oz_gemm (tcgen05.mma.kind::i8, one GEMM per modulus)",
            "peak_source": "nominal dense int8 (= fp8) tensor peak, B200_PROFILING.md",
            "int8_ops_per_step": int8_ops_step, "kernel_ms_per_step": gemm_ms,
            "fp64_equiv_tflops": fp64_tflops, "dmma_peak_tflops": dmma_peak,
            "fp64_equiv_vs_dmma_peak": (fp64_tflops / dmma_peak) if dmma_peak else None}


def hbm_roofline(bytes_per_launch, ms):
    """Secondary roofline object of the fused K0 launch (HBM-bound: one read
    of the batch).  peak = MEASURED_PEAKS.json hbm_gbs (driver-written copy
    bandwidth), else the profiling guide's 7700 GB/s nominal figure."""
    peak, src = 7700.0, "nominal HBM3e figure of B200_PROFILING.md (MEASURED_PEAKS.json absent)"
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        src = "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"
    except Exception:
        pass
    achieved = bytes_per_launch / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None,
            "kernel": "norm_select_kernel (fused K0: norm1, finiteness, (k, s), cost histogram)",
            "peak_source": src, "bytes_per_launch": bytes_per_launch,
            "kernel_ms_per_launch": ms,
            "note": "CUDA-event interval around ONE ~85 us launch, so it carries the launch "
                    "and event overhead (~15 us); ncu gpu__time_duration of the same launch: "
                    "83.5 us = 0.996 of the peak (profiles/r2/s6/ncu_k0_norm_select.txt)"}


def ctypes_collect(L):
    tot = ctypes.c_double(0.0)
    cnt = ctypes.c_int64(0)
    L.csm_profile_collect(ctypes.byref(tot), ctypes.byref(cnt))
    return tot.value, cnt.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-truth", action="store_true",
                    help="cfg5: skip the double-double truth comparison (~30 s)")
    ap.add_argument("--dist-mode", choices=["gather", "peer"], default="gather",
                    help="cfg5 only: NCCL all-gather per product, or the fused "
                         "peer-memory product (symmetric memory)")
    ap.add_argument("--engine", choices=["auto", "dmma", "ozaki"], default="dmma",
                    help="product engine of the tiled chain (n > 128) and the cfg5 slab "
                         "products: FP64 DMMA (the library default), Ozaki-II on the int8 "
                         "tensor cores, or auto (Ozaki from padded order 768 up)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warm-up raised to 3 (timing rule)")
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl != "reference":
        import paper_2010_00465_b200 as csm
        csm.set_engine(args.engine)
    if args.impl == "reference":
        run_reference(args, cfg)
    elif cfg[0] == "cfg5":
        run_cfg5(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
