import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2010_00465_b200 as csm
from oracle import cossin_oracle as orc
from tests._util import cfg2_like, rel1
rng = np.random.default_rng(5)
# 1) big batch of tiny matrices (K1, > 65535 matrices)
a = torch.from_numpy(cfg2_like(rng, 70000, n=8)).cuda()
r = csm.cos_sin_batched(a)
idx = [0, 35000, 69999]
ok = all(rel1(r.cos_part[i].cpu().numpy(), orc.cos_sin(a[i].cpu().numpy())[0]) <= 1e-12 for i in idx)
print("70000 x 8^2 K1:", ok)
# 2) tiled path with > 65535 items per launch: 70000 x 65^2 on the side chain? use CSM... n=130 (tiled), batch 4200 -> tiles 9 per matrix -> 37800 items
a = torch.from_numpy(cfg2_like(rng, 4200, n=130)).cuda()
r = csm.cos_sin_batched(a)
ok = all(rel1(r.cos_part[i].cpu().numpy(), orc.cos_sin(a[i].cpu().numpy())[0]) <= 1e-12 for i in (0, 2100, 4199))
print("4200 x 130^2 tiled:", ok)
# 3) one 2048^2 symmetric matrix: symmetry + Pythagorean on the GPU
n = 2048
g = rng.standard_normal((n, n)); h = torch.from_numpy(8.0 * (g + g.T) / (2 * np.sqrt(n))).cuda()
t0 = time.time(); r = csm.cos_sin_batched(h[None]); torch.cuda.synchronize(); dt = time.time() - t0
c, s = r.cos_part[0], r.sin_part[0]
sym = float((c - c.T).abs().max() / c.abs().max())
pyth = float((c @ c + s @ s - torch.eye(n, device="cuda", dtype=torch.float64)).abs().sum(0).max())
print(f"2048^2: k={int(r.k[0])} s={int(r.s[0])} sym={sym:.1e} pyth={pyth:.1e} time={dt:.2f}s")
