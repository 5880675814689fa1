"""Collocation BEM operator and GMRES on the GPU against the oracle's dense system
(PAPER.md Eqs. num, num2) and against the exact uniaxial patch test."""
import numpy as np
import pytest

from oracle import bem as OB
from oracle import kernels as KN
from workloads import geometry as geo
from tests.gpu_util import need_gpu, torch

pytestmark = pytest.mark.gpu
E, NU = 1.0, 0.3
G, KB = E / (2 * (1 + NU)), E / (3 * (1 - 2 * NU))


def _problem(nc):
    V0, V1, V2 = geo.cube_voxel_faces(nc)
    c, n, a = geo.panels(V0, V1, V2)
    uex = np.stack([-NU * c[:, 0] / E, -NU * c[:, 1] / E, c[:, 2] / E], 1)
    tex = np.stack([0 * c[:, 0], 0 * c[:, 0], n[:, 2]], 1)
    bc = np.where(c[:, 2] < 1e-9, 0, 1).astype(np.int32)
    val = np.where(bc[:, None] == 0, uex, tex)
    verts = np.stack([V0, V1, V2], 1).astype(np.float32)
    return verts, c, n, a, bc, val, uex, tex, (V0, V1, V2)


@pytest.fixture(scope="module")
def eb():
    need_gpu()
    import paper_1612_04082_b200 as eb
    return eb


@pytest.mark.parametrize("nq", [16, 1])
def test_operator_and_rhs_match_dense_oracle(eb, nq):
    verts, c, n, a, bc, val, uex, tex, V = _problem(3)
    # oracle on the same float32 geometry the GPU sees
    V0, V1, V2 = (verts[:, k].astype(np.float64) for k in range(3))
    c64, n64, a64 = geo.panels(V0, V1, V2)
    U, P = OB.assemble(c64, n64, a64, V0, V1, V2, KB, G, nq=nq)
    A, b = OB.mixed_system(U, P, bc, val.astype(np.float32))
    op = eb.bem_create(torch.from_numpy(verts).cuda(), nq=nq, max_pts=32, p=8, K=KB, G=G)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(3 * len(bc)).astype(np.float32)
    bcd = torch.from_numpy(bc).cuda()
    y = eb.bem_apply(op, bcd, torch.from_numpy(x).cuda().view(-1, 3)).cpu().numpy().reshape(-1)
    assert KN.rel_l2(y, A @ x.astype(np.float64)) < 1e-5
    bg = eb.bem_rhs(op, bcd, torch.from_numpy(val.astype(np.float32)).cuda()).cpu().numpy().reshape(-1)
    assert KN.rel_l2(bg, b) < 1e-5


def test_gmres_matches_dense_solve_and_patch_test(eb):
    verts, c, n, a, bc, val, uex, tex, V = _problem(4)
    V0, V1, V2 = (verts[:, k].astype(np.float64) for k in range(3))
    c64, n64, a64 = geo.panels(V0, V1, V2)
    U, P = OB.assemble(c64, n64, a64, V0, V1, V2, KB, G, nq=16)
    A, b = OB.mixed_system(U, P, bc, val.astype(np.float32))
    xref = np.linalg.solve(A, b)
    op = eb.bem_create(torch.from_numpy(verts).cuda(), nq=16, max_pts=32, p=8, K=KB, G=G)
    x = torch.zeros((len(bc), 3), device="cuda")
    x, it, res = eb.bem_gmres_solve(op, torch.from_numpy(bc).cuda(), torch.from_numpy(val.astype(np.float32)).cuda(),
                                    x, restart=50, max_iter=300, tol=1e-6)
    print("GMRES iterations", it, "residual", res)
    assert res <= 1e-6 and 0 < it < 300
    xs = x.cpu().numpy().astype(np.float64)
    assert KN.rel_l2(xs.reshape(-1), xref) < 1e-4
    m = bc == 1
    assert np.linalg.norm(xs[m] - uex[m]) / np.linalg.norm(uex[m]) < 0.05      # patch test
    assert np.linalg.norm(xs[~m] - tex[~m]) / np.linalg.norm(tex[~m]) < 0.05
    # the same system stopped early reports non-convergence but still returns an iterate
    x2 = torch.zeros_like(x)
    x2, it2, res2 = eb.bem_gmres_solve(op, torch.from_numpy(bc).cuda(),
                                       torch.from_numpy(val.astype(np.float32)).cuda(), x2, restart=5, max_iter=3,
                                       tol=1e-6, check=False)
    assert it2 == 3 and res2 > 1e-6
