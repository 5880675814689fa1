"""The tcgen05 3xTF32 translation path against the fp32 SIMT path (same schedule, same
operators): the two must agree to fp32 rounding, and both against the exact sum."""
import os

import numpy as np
import pytest

from oracle import cdirect
from oracle import kernels as KN
from workloads import geometry as geo
from tests.gpu_util import assert_fmm_close, need_gpu, to_dev, torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eb():
    need_gpu()
    import paper_1612_04082_b200 as eb
    return eb


@pytest.mark.parametrize("p,n", [(4, 6000), (6, 20000), (5, 8000)])
def test_tc_matches_simt(p, n):
    need_gpu()
    import paper_1612_04082_b200 as eb
    d = geo.config2(n=n, seed=11)
    t = to_dev(d)
    os.environ["EBEM_SIMT"] = "1"
    try:
        simt = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=64, p=p, K=d["K"], G=d["G"])
    finally:
        del os.environ["EBEM_SIMT"]
    tc = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=64, p=p, K=d["K"], G=d["G"])
    a = eb.fmm_matvec(simt, eb.KERNEL_UP, t["f"], t["g"]).cpu().numpy().astype(np.float64)
    b = eb.fmm_matvec(tc, eb.KERNEL_UP, t["f"], t["g"]).cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(b))
    diff = KN.rel_l2(b, a)
    ref = cdirect.direct_sum(KN.KERNEL_UP, d["src"], d["src"], d["K"], d["G"], w=d["w"], f=d["f"], g=d["g"],
                             nrm=d["nrm"])
    print(f"p={p}: |tc - simt| {diff:.2e}, tc err {KN.rel_l2(b, ref):.2e}, simt err {KN.rel_l2(a, ref):.2e}")
    assert diff < 1e-5
    # and each path on its own against the fp64 oracle, at the truncation bound of its order
    # (measured on the beam: 3.3e-3 at p = 4, 2.9e-5 at p = 6; p = 5 between)
    bound = {4: 5e-3, 5: 1e-3, 6: 1e-4}[p]
    assert_fmm_close(b, ref, bound, label=f"tc p={p}")
    assert_fmm_close(a, ref, bound, label=f"simt p={p}")


@pytest.mark.parametrize("scale", [1e-12, 1.0, 1e12])
def test_fp16_translations_cover_the_fp32_range(eb, scale):
    """The FP16 operand splits (tc_gemm.cu) scale every state row by a power of two, so the
    5-bit fp16 exponent must not show: densities of magnitude 1e-12 ... 1e12 give the exact sum
    (fp64 oracle, PAPER.md Eq. fmm_summation) within the p = 6 bound, error independent of the
    magnitude."""
    d = geo.config2(n=20000, seed=21)
    f = (d["f"] * scale).astype(np.float32)
    g = (d["g"] * scale).astype(np.float32)
    t = to_dev(d)
    tree = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=64, p=6, K=d["K"], G=d["G"])
    out = eb.fmm_matvec(tree, eb.KERNEL_UP, torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()).cpu().numpy()
    idx = np.sort(np.random.default_rng(3).choice(d["src"].shape[0], 1000, replace=False))
    ref = cdirect.direct_sum(KN.KERNEL_UP, d["src"][idx], d["src"], d["K"], d["G"], w=d["w"],
                             f=f.astype(np.float64), g=g.astype(np.float64), nrm=d["nrm"])
    assert_fmm_close(out[idx], ref, 1e-4, label=f"scale {scale:g}")


def test_fp16_translations_mixed_magnitudes(eb):
    """Densities whose magnitude varies by 1e8 over the surface (a row-wise, not a global,
    scale is needed: one global fp16 scale would flush the weak region's state to zero).  The
    weak half's own field is checked where it dominates: targets in the weak half, with the
    strong half's densities set to zero in a second evaluation, must agree with the oracle."""
    d = geo.config2(n=20000, seed=22)
    weak = d["src"][:, 0] < 2.0
    amp = np.where(weak, 1e-8, 1.0).astype(np.float32)[:, None]
    t = to_dev(d)
    tree = eb.fmm_build_tree(t["src"], t["nrm"], t["w"], max_pts=64, p=6, K=d["K"], G=d["G"])
    idx = np.sort(np.random.default_rng(4).choice(d["src"].shape[0], 1000, replace=False))
    for f, g, label in [(d["f"] * amp, d["g"] * amp, "mixed"),
                        (d["f"] * amp * weak[:, None], d["g"] * amp * weak[:, None], "weak half alone")]:
        f = f.astype(np.float32)
        g = g.astype(np.float32)
        out = eb.fmm_matvec(tree, eb.KERNEL_UP, torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()).cpu().numpy()
        ref = cdirect.direct_sum(KN.KERNEL_UP, d["src"][idx], d["src"], d["K"], d["G"], w=d["w"],
                                 f=f.astype(np.float64), g=g.astype(np.float64), nrm=d["nrm"])
        assert_fmm_close(out[idx], ref, 1e-4, label=label)
