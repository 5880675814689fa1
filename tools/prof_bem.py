"""Short driver for ncu captures of the BEM operator: configs[4] cell, a few GMRES iterations
(the near operator is built, then applied once per iteration)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1612_04082_b200 as eb
from workloads import geometry as geo

d = geo.metamaterial_cell(nc=160, level=5, nvoids=64)
verts = torch.from_numpy(d["verts"]).cuda()
bc = torch.from_numpy(d["bc_type"]).cuda()
val = torch.from_numpy(d["bc_val"]).cuda()
op = eb.bem_create(verts, nq=16, max_pts=1536, p=8, K=d["K"], G=d["G"])
x = torch.zeros((d["verts"].shape[0], 3), device="cuda")
x, it, res = eb.bem_gmres_solve(op, bc, val, x, restart=50, max_iter=int(os.environ.get("IT", 3)), tol=1e-6,
                                precond=int(os.environ.get("PRECOND", 2)), check=False)
torch.cuda.synchronize()
print("ok", it, res)
