"""Worker of tests/test_gpu_k0_fused.py: runs seeded batches through the
drop-in batched entry points and saves (k, s, status, outputs).  The parent
runs it twice -- CSM_K0_FUSED=1 (one norm/select/histogram launch) and =0
(norm1_kernel + select_kernel + histogram launches) -- and compares bits."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def cases():
    out = {}
    rng = np.random.default_rng(11)
    for n, count, dtype in ((64, 700, np.float64), (63, 300, np.float64), (5, 200, np.float64),
                            (37, 200, np.float32), (64, 300, np.float32), (100, 120, np.float64),
                            (128, 140, np.float64), (66, 64, np.float32), (2, 50, np.float64),
                            (1, 40, np.float64)):
        g = rng.standard_normal((count, n, n))
        norm = np.abs(g).sum(axis=1).max(axis=1)
        tgt = 10.0 ** rng.uniform(-3, 2.5, count)
        a = (g * (tgt / norm)[:, None, None]).astype(dtype)
        out[f"trig_{n}_{np.dtype(dtype).name}"] = (a, None)
    # rejected inputs and extreme norms (statuses 1, 2 / 3 through the selection)
    a = out["trig_64_float64"][0][:256].copy()
    a[3, 5, 7] = np.nan
    a[100, 63, 63] = np.inf
    a[255, 0, 0] = -np.inf
    a[17] *= 1e300
    a[18] *= 1e-300
    a[19] = 0.0
    out["status_64"] = (a, None)
    # wave family (norm scaled by t * t before the selection)
    n = 64
    lap = (np.diag(2.0 * np.ones(n)) - np.diag(np.ones(n - 1), 1)
           - np.diag(np.ones(n - 1), -1)) * float((n + 1) ** 2)
    count = 300
    a = lap[None] + np.stack([np.diag(rng.uniform(0, 10, n)) for _ in range(count)])
    out["wave_64"] = (a, 10.0 ** rng.uniform(-4, -1, count))
    n = 96
    lap = (np.diag(2.0 * np.ones(n)) - np.diag(np.ones(n - 1), 1)
           - np.diag(np.ones(n - 1), -1)) * float((n + 1) ** 2)
    a = lap[None] + np.stack([np.diag(rng.uniform(0, 10, n)) for _ in range(80)])
    out["wave_96"] = (a, 10.0 ** rng.uniform(-4, -1, 80))
    return out


def main(path):
    import torch

    import paper_2010_00465_b200 as csm

    res = {}
    for name, (a, t) in cases().items():
        x = torch.from_numpy(a).cuda()
        if t is None:
            rep = csm.cos_sin_batched(x, raise_on_error=False)
            # the same data 8 bytes (4 for float32) off a 16-byte boundary:
            # the scalar-load variant of the kernel
            if a.shape[-1] <= 64:
                flat = torch.empty(x.numel() + 1, dtype=x.dtype, device=x.device)
                flat[1:].copy_(x.reshape(-1))
                rep_u = csm.cos_sin_batched(flat[1:].view(x.shape), raise_on_error=False)
                res[f"{name}/k_unaligned"] = rep_u.k.cpu().numpy()
                res[f"{name}/s_unaligned"] = rep_u.s.cpu().numpy()
                res[f"{name}/st_unaligned"] = rep_u.status.cpu().numpy()
        else:
            rep = csm.wave_cos_sin_batched(x, torch.from_numpy(t).cuda(), raise_on_error=False)
        res[f"{name}/k"] = rep.k.cpu().numpy()
        res[f"{name}/s"] = rep.s.cpu().numpy()
        res[f"{name}/st"] = rep.status.cpu().numpy()
        res[f"{name}/c"] = rep.cos_part.cpu().numpy()
        res[f"{name}/sn"] = rep.sin_part.cpu().numpy()
    np.savez(path, **res)


if __name__ == "__main__":
    main(sys.argv[1])
