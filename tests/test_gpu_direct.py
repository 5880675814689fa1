"""Parity of bem_kernel_direct (fp32 CUDA) against the fp64 oracle direct sum.
North star: relative L2 error <= 1e-5."""
import numpy as np
import pytest

from oracle import cdirect
from oracle import kernels as KN
from workloads import geometry as geo
from tests.gpu_util import need_gpu, to_dev, torch

pytestmark = pytest.mark.gpu
ALL = (KN.KERNEL_U, KN.KERNEL_P, KN.KERNEL_UP, KN.KERNEL_D, KN.KERNEL_S, KN.KERNEL_DS)


@pytest.fixture(scope="module")
def eb():
    need_gpu()
    import paper_1612_04082_b200 as eb
    return eb


def test_config0_single_layer_sphere(eb):
    d = geo.config0()          # 2048 points, K = 1, G = 0.5
    t = to_dev(d)
    out = eb.bem_kernel_direct(eb.KERNEL_U, t["src"], t["src"], w=t["w"], f=t["f"], K=d["K"], G=d["G"])
    ref = cdirect.direct_sum(KN.KERNEL_U, d["src"], d["src"], d["K"], d["G"], w=d["w"], f=d["f"])
    got = out.cpu().numpy().astype(np.float64)
    assert KN.rel_l2(got, ref) <= 1e-5
    # element by element: fp32 sum of 2047 terms
    assert np.allclose(got, ref, rtol=0, atol=2e-5 * np.abs(ref).max())


def test_config1_double_layer_cube_sampled(eb):
    d = geo.config1()          # 24,576 triangles, all pairs on the GPU
    t = to_dev(d)
    out = eb.bem_kernel_direct(eb.KERNEL_P, t["src"], t["src"], nrm=t["nrm"], w=t["w"], g=t["g"], K=d["K"], G=d["G"])
    got = out.cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(d["src"].shape[0], 1500, replace=False))
    ref = cdirect.direct_sum(KN.KERNEL_P, d["src"][sample], d["src"], d["K"], d["G"], w=d["w"], g=d["g"],
                             nrm=d["nrm"])
    assert KN.rel_l2(got[sample], ref) <= 1e-5


@pytest.mark.parametrize("kern", ALL)
@pytest.mark.parametrize("ntrg,nsrc", [(1, 1), (1, 777), (333, 1), (1000, 5000), (257, 0)])
def test_all_kernels_ragged(eb, kern, ntrg, nsrc):
    rng = np.random.default_rng(ntrg * 7 + nsrc)
    src = rng.uniform(-1, 1, (nsrc, 3)).astype(np.float32)
    trg = rng.uniform(-1, 1, (ntrg, 3)).astype(np.float32)
    if nsrc and ntrg > 1:
        trg[: min(ntrg, nsrc) // 2] = src[: min(ntrg, nsrc) // 2]      # coincident pairs excluded
    nrm = rng.standard_normal((nsrc, 3))
    nrm /= np.maximum(np.linalg.norm(nrm, axis=1, keepdims=True), 1e-30)
    nrm = nrm.astype(np.float32)
    w = rng.uniform(0.5, 2, nsrc).astype(np.float32)
    f = rng.standard_normal((nsrc, 3)).astype(np.float32)
    g = rng.standard_normal((nsrc, 3)).astype(np.float32)
    T = lambda a: torch.from_numpy(a).cuda()
    out = eb.bem_kernel_direct(kern, T(trg), T(src), nrm=T(nrm), w=T(w), f=T(f), g=T(g), K=1.67, G=0.77)
    got = out.cpu().numpy().astype(np.float64)
    ref = cdirect.direct_sum(kern, trg, src, 1.67, 0.77, w=w, f=f, g=g, nrm=nrm)
    if nsrc == 0:
        assert np.all(got == 0)
        return
    assert np.all(np.isfinite(got))
    assert KN.rel_l2(got, ref) <= 1e-5
    # host-pointer path gives the same bits as the device path
    host = eb.bem_kernel_direct(kern, trg, src, nrm=nrm, w=w, f=f, g=g, K=1.67, G=0.77)
    assert np.array_equal(host, out.cpu().numpy())
