"""Per-phase device times (serial, native profiler) of the 1M-point beam matvec at order p."""
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
ap.add_argument("--p", type=int, default=10)
a = ap.parse_args()
d = geo.config2(n=a.n)
t = {k: torch.from_numpy(v).cuda() for k, v in d.items() if isinstance(v, np.ndarray)}
tree = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=64, p=a.p, K=d["K"], G=d["G"])
out = torch.empty((d["src"].shape[0], 3), device="cuda")
for _ in range(2):
    eb.fmm_matvec(tree, eb.KERNEL_UP, t["f"], t["g"], out=out)
eb.fmm_set_profiling(tree, True)
for _ in range(3):
    eb.fmm_matvec(tree, eb.KERNEL_UP, t["f"], t["g"], out=out)
tot = 0
for p in eb.fmm_phase_stats(tree, eb.KERNEL_UP):
    tot += max(p["ms"], 0)
    print(f"{p['name']:8s} {p['ms']:.3f} ms  launches {p['launches']}  gflop {p['flops']/1e9:.2f}")
print("sum", round(tot, 3))
