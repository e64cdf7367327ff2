"""One Ozaki-engine cos_sin_batched call (for ncu launch lists):
python tools/oz_prof.py N B [engine]."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2010_00465_b200 as csm
from tests._util import cfg2_like

n = int(sys.argv[1]); B = int(sys.argv[2])
csm.set_engine(sys.argv[3] if len(sys.argv) > 3 else "ozaki")
a = torch.from_numpy(cfg2_like(np.random.default_rng(0), B, n=n)).cuda()
rep = csm.cos_sin_batched(a)
torch.cuda.synchronize()
print("k", rep.k.tolist(), "s", rep.s.tolist())
