"""Short driver for ncu captures: build the bench workload's tree, run `reps` matvecs."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1612_04082_b200 as eb
from workloads import geometry as geo

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--p", type=int, default=6)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--direct", action="store_true", help="also run the configs[1] direct P kernel")
a = ap.parse_args()
d = geo.config2(n=a.n)
t = {k: torch.from_numpy(v).cuda() for k, v in d.items() if isinstance(v, np.ndarray)}
tree = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=64, p=a.p, K=d["K"], G=d["G"])
out = torch.empty((d["src"].shape[0], 3), device="cuda")
for _ in range(a.reps):
    eb.fmm_matvec(tree, eb.KERNEL_UP, t["f"], t["g"], out=out)
if a.direct:
    c = geo.config1()
    tc = {k: torch.from_numpy(v).cuda() for k, v in c.items() if isinstance(v, np.ndarray)}
    for _ in range(a.reps):
        eb.bem_kernel_direct(eb.KERNEL_P, tc["src"], tc["src"], nrm=tc["nrm"], w=tc["w"], g=tc["g"], K=c["K"], G=c["G"])
torch.cuda.synchronize()
print("ok")
