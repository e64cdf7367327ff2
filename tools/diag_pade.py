import numpy as np, os, sys
sys.path.insert(0, os.getcwd())
import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc
from tests._util import rel1, pair_close
g = np.load("tests/golden/pade.npz")
for entry in g["names"]:
    name, prec = str(entry).split("|")
    a = g[f"{name}__a"]
    rep = csm.pade_cos_sin(a, csm.Precision(prec))
    rc, rs = g[f"{name}__cos"], g[f"{name}__sin"]
    print(name, a.shape[0], rep.scaling_exponent, "cos rel1 %.3e" % rel1(rep.result.cos_part, rc), "sin rel1 %.3e" % (rel1(rep.result.sin_part, rs) if orc.norm1(rs) > 0 else 0), pair_close(rep.result.cos_part, rc, rs, 1e-12))
# padded n=65 small norm
rng = np.random.default_rng(1)
for n in (65, 100, 128):
    a = rng.standard_normal((n, n)); a *= 0.05 / orc.norm1(a)
    rep = csm.pade_cos_sin(a); c, s, sc = orc.pade_cos_sin(a)
    print("n", n, "s", sc, rep.scaling_exponent, "%.3e %.3e" % (rel1(rep.result.cos_part, c), rel1(rep.result.sin_part, s)))
