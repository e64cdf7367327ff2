"""One block-row chain call (cfg5 shape) under the selected engine, for ncu
launch lists: python tools/oz_prof_slab.py N [engine]."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2010_00465_b200 as csm
from paper_2010_00465_b200 import distchain

n = int(sys.argv[1])
csm.set_engine(sys.argv[2] if len(sys.argv) > 2 else "ozaki")
g = np.random.default_rng(0).standard_normal((n, n))
a = torch.from_numpy(20.0 * (g + g.T) / (2.0 * np.sqrt(n))).cuda()
c, s, st = distchain.cos_sin_distributed(a, gather_outputs=False)
torch.cuda.synchronize()
print("k", st.k, "s", st.s, "products", st.products)
