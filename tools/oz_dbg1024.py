import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2010_00465_b200 as csm
from paper_2010_00465_b200 import verify
from oracle import cossin_oracle as orc
from tests._util import cfg2_like, rel1
rng = np.random.default_rng(820)
a = cfg2_like(rng, 3, n=1024, lo=-1.0, hi=2.0)
tc, ts, _ = verify.reference_cos_sin_batched(a)
for eng in ("dmma", "ozaki"):
    csm.set_engine(eng)
    rep = csm.cos_sin_batched(a)
    for i in range(3):
        c, s, k, sc = orc.cos_sin(a[i])
        print(eng, i, "norm", round(orc.norm1(a[i]), 2), "k,s", k, sc,
              "vs oracle %.2e %.2e" % (rel1(rep.cos_part[i], c), rel1(rep.sin_part[i], s)),
              "vs truth %.2e %.2e" % (rel1(rep.cos_part[i], tc[i]), rel1(rep.sin_part[i], ts[i])),
              "oracle vs truth %.2e %.2e" % (rel1(c, tc[i]), rel1(s, ts[i])), flush=True)
