import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2010_00465_b200 import corpus
d = np.load("tests/golden/corpus.npz")
mats, off = [], 0
for n in d["dims"]:
    mats.append(d["data"][off:off + n * n].reshape(n, n)); off += n * n
recs = corpus.run_corpus(mats, [str(t) for t in d["tags"]])
for meth, key in (("taylor", "t"), ("pade", "p")):
    rat = []
    for i in range(len(mats)):
        r = recs[2 * i + (meth == "pade")]
        for mine, ref in ((r.rel_err_cos, d[key + "_ec"][i]), (r.rel_err_sin, d[key + "_es"][i])):
            if math.isfinite(mine) and math.isfinite(ref) and ref > 0 and mine > 0:
                rat.append((mine / ref, r.scaling_s, i))
    rs = np.array([x[0] for x in rat])
    print(meth, "n", len(rs), "geomean ratio %.3f" % np.exp(np.mean(np.log(rs))), "max %.2f" % rs.max(), "min %.3f" % rs.min())
    print(" worst:", sorted(rat)[-5:])
print(corpus.summary(recs))
