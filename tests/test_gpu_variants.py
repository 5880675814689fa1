"""Kernel variants selected by process-wide switches (read once per process, so each runs in a
child process): the persistent M2M/L2L level-chain kernel (EBEM_ML_CHAIN=1), the wide
128 x 256 M2L tiles (EBEM_M2L_WIDE=1), the packed FFMA2 near field (EBEM_NEAR_PACKED=1) and the
operand type of the translations (TF32 or FP16 head / remainder splits), the cluster-multicast
M2L (EBEM_M2L_MC = 2 / 4 CTAs sharing the operator tiles).  Each must meet the same bounds against the
fp64 oracle as the default path (the KIFMM sum of Eq. fmm_summation)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.gpu_util import assert_fmm_close, need_gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1612_04082_b200 as eb
from workloads import geometry as geo
d = geo.config2(n=30000)
t = {{k: torch.from_numpy(v).cuda() for k, v in d.items() if isinstance(v, np.ndarray)}}
tree = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=64, p=6, K=d["K"], G=d["G"])
out = eb.fmm_matvec(tree, eb.KERNEL_UP, t["f"], t["g"])
out2 = eb.fmm_matvec(tree, eb.KERNEL_UP, t["f"], t["g"])
torch.cuda.synchronize()
np.save({path!r}, np.stack([out.cpu().numpy(), out2.cpu().numpy()]))
"""

# EBEM_M2L_F16=0: every translation on TF32 operands; EBEM_ML_F16=0: FP16 M2L, TF32 M2M / L2L;
# the default is FP16 operands for M2L, M2M and L2L (tc_gemm.cu, 3xFP16)
VARIANTS = [{}, {"EBEM_ML_CHAIN": "1"}, {"EBEM_M2L_WIDE": "1"}, {"EBEM_NEAR_PACKED": "1"}, {"EBEM_M2L_F16": "0"},
            {"EBEM_ML_F16": "0"}, {"EBEM_M2L_F16": "1"}, {"EBEM_M2L_MC": "2"}, {"EBEM_M2L_MC": "4"},
            {"EBEM_Q2Z_F16": "0"}]


@pytest.fixture(scope="module")
def reference():
    from oracle import cdirect
    from oracle import kernels as KN
    from workloads import geometry as geo
    d = geo.config2(n=30000)
    idx = np.sort(np.random.default_rng(5).choice(d["src"].shape[0], 1500, replace=False))
    ref = cdirect.direct_sum(KN.KERNEL_UP, d["src"][idx], d["src"], d["K"], d["G"], w=d["w"], f=d["f"], g=d["g"],
                             nrm=d["nrm"])
    return idx, ref


@pytest.mark.gpu
@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_variant_matches_oracle(env, reference, tmp_path):
    need_gpu()
    path = str(tmp_path / "out.npy")
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, path=path)], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = np.load(path)
    assert np.array_equal(out[0], out[1]), "repeated matvec not bitwise identical"
    idx, ref = reference
    assert_fmm_close(out[0][idx], ref, 1e-4, label=json.dumps(env))
