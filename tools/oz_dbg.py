"""Scratch: Ozaki vs DMMA vs the oracle vs the double-double truth on
cfg2-like n = 256 matrices at growing norms (where does Ozaki's row/column
max scaling lose to fp64 accuracy?)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2010_00465_b200 as csm
from paper_2010_00465_b200 import verify
from oracle import cossin_oracle as orc
from tests._util import cfg2_like, rel1

rng = np.random.default_rng(815)
for norm in (1e1, 1e2, 1e3, 3e3, 1e4):
    a = cfg2_like(rng, 2, n=256, lo=0, hi=0)
    a *= (norm / np.abs(a).sum(axis=1).max(axis=1))[:, None, None]
    tc, ts, _ = verify.reference_cos_sin_batched(a)
    row = []
    for eng in ("dmma", "ozaki"):
        csm.set_engine(eng)
        rep = csm.cos_sin_batched(a)
        e_or = max(rel1(rep.cos_part[i], orc.cos_sin(a[i])[0]) for i in range(2))
        e_tr = max(rel1(rep.cos_part[i], tc[i]) for i in range(2))
        row.append(f"{eng}: vs oracle {e_or:.1e} vs truth {e_tr:.1e}")
    e_ot = max(rel1(orc.cos_sin(a[i])[0], tc[i]) for i in range(2))
    print(f"norm {norm:.0e} s={int(rep.s[0])}: " + " | ".join(row) + f" | oracle vs truth {e_ot:.1e}", flush=True)
csm.set_engine("auto")
