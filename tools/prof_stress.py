"""configs[3] stress evaluation: per-phase device times (serial, native profiler) and the
overlapped step time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1612_04082_b200 as eb
from workloads import geometry as geo

d = geo.config3()
t = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).cuda() for k, v in d.items() if isinstance(v, np.ndarray)}
tree = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], trg=t["trg"], max_pts=int(os.environ.get("LEAF", 256)), p=8,
                         K=d["K"], G=d["G"])
out = torch.empty((d["trg"].shape[0], 6), device="cuda")
for _ in range(3):
    eb.fmm_eval_stress(tree, eb.KERNEL_DS, t["f"], t["g"], out=out)
eb.fmm_set_profiling(tree, True)
for _ in range(3):
    eb.fmm_eval_stress(tree, eb.KERNEL_DS, t["f"], t["g"], out=out)
for p in eb.fmm_phase_stats(tree, eb.KERNEL_DS):
    print(f"{p['name']:8s} {p['ms']:.3f} ms  launches {p['launches']}  interactions {p['interactions']:.3g}  gflop {p['flops']/1e9:.2f}")
print(eb.fmm_tree_info(tree))
