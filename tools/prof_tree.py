"""Short driver for ncu captures of the tree build: three 1M-point builds (configs[2] beam)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1612_04082_b200 as eb
from workloads import geometry as geo

d = geo.config2(n=1_000_000, seed=0)
S, N, W = (torch.from_numpy(d[k]).cuda() for k in ("src", "nrm", "w"))
for _ in range(3):
    tree = eb.fmm_build_tree(S, N, W, max_pts=64, p=6, K=d["K"], G=d["G"])
    del tree
torch.cuda.synchronize()
print("ok")
