"""Single-rank smoke of the symmetric-memory peer path (NCCL, world 1)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
from paper_2010_00465_b200 import distchain
n = 512
g = np.random.default_rng(3).standard_normal((n, n))
a = torch.from_numpy(20.0 * (g + g.T) / (2.0 * np.sqrt(n))).cuda()
c, s, st = distchain.cos_sin_distributed_peer(a)
c1, s1, st1 = distchain.cos_sin_distributed(a)
print("peer == gather:", torch.equal(c, c1), torch.equal(s, s1), st)
dist.destroy_process_group()
