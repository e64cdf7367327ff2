import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2010_00465_b200 as csm
from paper_2010_00465_b200 import verify
from oracle import cossin_oracle as orc
d = np.load("tests/golden/corpus.npz")
mats, off = [], 0
for n in d["dims"]:
    mats.append(d["data"][off:off + n * n].reshape(n, n)); off += n * n
for i in (23, 29, 30):
    a = mats[i]
    np.set_printoptions(precision=3, linewidth=150)
    rep = csm.pade_cos_sin(a)
    c, s, sc = orc.pade_cos_sin(a)
    tr = verify.reference_cos_sin(a)
    e = lambda x, y: np.linalg.norm(x - y, 2) / np.linalg.norm(y, 2)
    print(i, a.shape, "norm %.3e" % orc.norm1(a), "s", sc, "ours-vs-truth cos %.3e sin %.3e" % (e(rep.result.cos_part, tr.cos_part), e(rep.result.sin_part, tr.sin_part)),
          "oracle-vs-truth cos %.3e sin %.3e" % (e(c, tr.cos_part), e(s, tr.sin_part)), "ref golden %.3e %.3e" % (d["p_ec"][i], d["p_es"][i]))
    if i == 23:
        print(a)
