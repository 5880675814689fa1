"""Pins for oracle/kifmm.py (reference tree code) and oracle/c/direct_sum.c.

The KIFMM oracle is pinned to the exact O(N^2) sum (itself pinned in
test_oracle_kernels.py): exact equality when the tree is a single leaf (pure near
field), convergence with the multipole order p, and linearity.  The C direct sum is
pinned to the numpy direct sum."""
import numpy as np
import pytest

from oracle import cdirect
from oracle import kernels as KN
from oracle import kifmm as F
from workloads import geometry as geo

ALL = (KN.KERNEL_U, KN.KERNEL_P, KN.KERNEL_UP, KN.KERNEL_D, KN.KERNEL_S, KN.KERNEL_DS)


def _case(n=400, seed=5):
    rng = np.random.default_rng(seed)
    src = rng.uniform(-1, 1, (n, 3))
    trg = np.concatenate([rng.uniform(-1, 1, (n // 2, 3)), src[: n // 4]])
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    return src, trg, nrm, rng.uniform(0.5, 2, n), rng.standard_normal((n, 3)), rng.standard_normal((n, 3))


@pytest.mark.parametrize("kern", ALL)
def test_c_direct_sum_matches_numpy(kern):
    src, trg, nrm, w, f, g = _case()
    a = cdirect.direct_sum(kern, trg, src, 1.67, 0.77, w=w, f=f, g=g, nrm=nrm)
    b = KN.direct_sum(kern, trg, src, 1.67, 0.77, w=w, f=f, g=g, nrm=nrm)
    assert np.allclose(a, b, rtol=1e-12, atol=1e-12 * np.abs(b).max())


@pytest.mark.parametrize("kern", ALL)
def test_single_leaf_is_exact(kern):
    src, trg, nrm, w, f, g = _case(120)
    fm = F.KIFMM(src, trg, 1.0, 0.5, p=4, max_pts=10_000, nrm=nrm)
    assert fm.T.nboxes == 1
    out = fm.evaluate(kern, w=w, f=f, g=g)
    ref = KN.direct_sum(kern, trg, src, 1.0, 0.5, w=w, f=f, g=g, nrm=nrm)
    assert np.allclose(out, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())


@pytest.fixture(scope="module")
def beam():
    d = geo.config2(n=1500, seed=9)
    ref = {k: cdirect.direct_sum(k, d["src"], d["src"], d["K"], d["G"], w=d["w"], f=d["f"], g=d["g"], nrm=d["nrm"])
           for k in (KN.KERNEL_UP, KN.KERNEL_DS)}
    return d, ref


def test_kifmm_converges_in_p(beam):
    """relative L2 error vs the exact sum decreases with p (north star: <= 1e-4 at p = 6)."""
    d, ref = beam
    errs = []
    for p in (4, 6, 8):
        fm = F.KIFMM(d["src"], d["src"], d["K"], d["G"], p=p, max_pts=32, nrm=d["nrm"])
        assert fm.T.level.max() >= 3
        out = fm.evaluate(KN.KERNEL_UP, w=d["w"], f=d["f"], g=d["g"])
        errs.append(KN.rel_l2(out, ref[KN.KERNEL_UP]))
    assert errs[0] > errs[1] > errs[2]
    assert errs[1] < 1e-4 and errs[2] < 5e-6


def test_kifmm_stress_and_linearity(beam):
    d, ref = beam
    fm = F.KIFMM(d["src"], d["src"], d["K"], d["G"], p=6, max_pts=32, nrm=d["nrm"])
    out = fm.evaluate(KN.KERNEL_DS, w=d["w"], f=d["f"], g=d["g"])
    assert KN.rel_l2(out, ref[KN.KERNEL_DS]) < 1e-3
    a = fm.evaluate(KN.KERNEL_UP, w=d["w"], f=d["f"], g=d["g"])
    b = fm.evaluate(KN.KERNEL_UP, w=d["w"], f=2 * d["f"], g=-d["g"])
    c = fm.evaluate(KN.KERNEL_UP, w=d["w"], f=3 * d["f"], g=0 * d["g"])
    # the regularised check->equivalent solve amplifies fp64 rounding to ~1e-8 relative
    assert np.allclose(a + b, c, rtol=0, atol=1e-7 * np.abs(c).max())


def test_kifmm_separate_targets():
    rng = np.random.default_rng(3)
    src = geo.sphere_points(800, seed=4).astype(np.float64)
    trg = rng.uniform(-0.6, 0.6, (500, 3))
    f = rng.standard_normal((800, 3))
    fm = F.KIFMM(src, trg, 1.0, 0.5, p=6, max_pts=24)
    out = fm.evaluate(KN.KERNEL_D, f=f)
    ref = KN.direct_sum(KN.KERNEL_D, trg, src, 1.0, 0.5, f=f)
    assert KN.rel_l2(out, ref) < 1e-4


def test_surface_grid_count():
    for p in (2, 4, 6, 10):
        s = F.surface_grid(p)
        assert s.shape == (6 * (p - 1) ** 2 + 2, 3)
        assert np.all(np.max(np.abs(s), axis=1) == 1.0)
