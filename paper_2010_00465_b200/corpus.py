"""GPU backend for corpus runs.

The reference's ``bench`` command (cli.py:128-163) walks a test-matrix
corpus one matrix at a time: reference values (verify.reference_cos_sin),
then ``cos_sin`` and ``pade_cos_sin`` per matrix, each timed with
perf_counter, and writes one ``RunRecord`` (cli.py:51-60) per matrix and
method to a CSV.  Here the same records come from batched device calls:
matrices are grouped by order n, every group runs in one call per method
(Taylor on K1 / K1c / the tiled chain, Pade on the tiled chain + batched
LU, the double-double reference values on csrc/ddref.cu), and each
record's ``wall_time`` is its group's device time divided by the group
size.  The spectral-norm relative errors (cli.py:147-150,
verify.py:524-534) are the reference's own metric, evaluated on the host
with numpy exactly as verify.py does (scoring, not the cos/sin path).

The corpus itself is the caller's (any list of square float64 matrices
with class tags); tests/golden/corpus.npz holds the reference's own
gallery corpus (gallery.py:186-220) with its per-matrix (k, s, products)
and errors, against which tests/test_gpu_corpus.py checks this backend.
"""
from __future__ import annotations

import csv
import math
from dataclasses import dataclass, fields  # noqa: F401  (fields re-exported for tests)
from typing import Iterable, Sequence

import numpy as np

from .api import _torch, cos_sin_batched, norm1, pade_cos_sin_batched
from . import verify


@dataclass
class RunRecord:
    """One CSV row (cli.py:51-60)."""

    matrix_id: str
    class_tag: str
    norm: float
    method: str
    rel_err_cos: float
    rel_err_sin: float
    products: float
    scaling_s: int
    wall_time: float


def _rel_err_2(approx, ref) -> "np.ndarray":
    """relative_error_2 (verify.py:524-534) for a batch: the reference's own
    metric, evaluated as it is -- numpy's spectral norm on the host (LAPACK
    SVD) -- on the device results copied back.  It scores a corpus run; it
    is not part of the cos/sin path, which stays on the device."""
    a = approx.double().cpu().numpy() if hasattr(approx, "cpu") else np.asarray(approx)
    r = ref.double().cpu().numpy() if hasattr(ref, "cpu") else np.asarray(ref)
    out = np.empty(a.shape[0])
    for i in range(a.shape[0]):
        if not (np.all(np.isfinite(a[i])) and np.all(np.isfinite(r[i]))):
            out[i] = math.inf
            continue
        den = float(np.linalg.norm(r[i], 2))
        num = float(np.linalg.norm(a[i] - r[i], 2))
        out[i] = (0.0 if num == 0.0 else math.inf) if den == 0.0 else num / den
    return out


def _timed(fn):
    torch = _torch()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) * 1e-3


def run_corpus(matrices: Sequence, tags: Sequence[str],
               methods: Iterable[str] = ("taylor", "pade")) -> list[RunRecord]:
    """RunRecords for every (matrix, method), grouped by n on the device."""
    torch = _torch()
    methods = list(methods)
    mats = [np.asarray(m, dtype=np.float64) for m in matrices]
    if len(mats) != len(tags):
        raise ValueError("need one class tag per matrix")
    groups: dict[int, list[int]] = {}
    for i, m in enumerate(mats):
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ValueError(f"matrix {i} is not square: {m.shape}")
        groups.setdefault(m.shape[0], []).append(i)
    recs: dict[tuple[int, str], RunRecord] = {}
    for n, idx in sorted(groups.items()):
        a = torch.from_numpy(np.stack([mats[i] for i in idx])).cuda()
        ref_c, ref_s, _ = verify.reference_cos_sin_batched(a)
        for method in methods:
            run = cos_sin_batched if method == "taylor" else pade_cos_sin_batched
            rep, secs = _timed(lambda: run(a, raise_on_error=False))
            ec = _rel_err_2(rep.cos_part, ref_c)
            es = _rel_err_2(rep.sin_part, ref_s)
            k = rep.k.cpu().numpy()
            s = rep.s.cpu().numpy()
            per = secs / len(idx)
            for j, i in enumerate(idx):
                prod = float(k[j] + 2 * s[j]) + (7.0 / 3.0 if method == "pade" else 0.0)
                recs[(i, method)] = RunRecord(
                    matrix_id=f"{i:05d}", class_tag=str(tags[i]), norm=norm1(mats[i]),
                    method=method, rel_err_cos=float(ec[j]), rel_err_sin=float(es[j]),
                    products=prod, scaling_s=int(s[j]), wall_time=per)
    return [recs[(i, m)] for i in range(len(mats)) for m in methods]


def write_csv(records: Sequence[RunRecord], path: str) -> None:
    """The reference's CSV layout (cli.py:157-162)."""
    names = [f.name for f in fields(RunRecord)]
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(names)
        for r in records:
            w.writerow([getattr(r, n) for n in names])


def summary(records: Sequence[RunRecord]) -> str:
    """Taylor-vs-Pade error tally (cli.py:166-187)."""
    by_id: dict[str, dict[str, RunRecord]] = {}
    for r in records:
        by_id.setdefault(r.matrix_id, {})[r.method] = r
    parts = []
    for func in ("cos", "sin"):
        tb = pb = eq = 0
        for pair in by_id.values():
            te = getattr(pair["taylor"], f"rel_err_{func}")
            pe = getattr(pair["pade"], f"rel_err_{func}")
            if te < pe:
                tb += 1
            elif pe < te:
                pb += 1
            else:
                eq += 1
        parts.append(f"{func}: taylor_better={tb} pade_better={pb} equal={eq}")
    return "; ".join(parts)


__all__ = ["RunRecord", "run_corpus", "summary", "write_csv"]
