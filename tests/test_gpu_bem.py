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


@pytest.mark.parametrize("precond", [0, 1, 2])
def test_gmres_matches_dense_solve_and_patch_test(eb, precond):
    """the paper's GMRES (precond = 0) and the right-preconditioned ones (precond = 1: 3x3
    block-Jacobi, 2: leaf-block Jacobi; the same residual |b - A x| / |b|) against dense LU of
    the oracle system."""
    verts, c, n, a, bc, val, uex, tex, V = _problem(4)
    V0, V1, V2 = (verts[:, k].astype(np.float64) for k in range(3))
    c64, n64, a64 = geo.panels(V0, V1, V2)
    U, P = OB.assemble(c64, n64, a64, V0, V1, V2, KB, G, nq=16)
    A, b = OB.mixed_system(U, P, bc, val.astype(np.float32))
    xref = np.linalg.solve(A, b)
    op = eb.bem_create(torch.from_numpy(verts).cuda(), nq=16, max_pts=32, p=8, K=KB, G=G)
    x = torch.zeros((len(bc), 3), device="cuda")
    x, it, res = eb.bem_gmres_solve(op, torch.from_numpy(bc).cuda(), torch.from_numpy(val.astype(np.float32)).cuda(),
                                    x, restart=50, max_iter=300, tol=1e-6, precond=precond)
    print("GMRES precond", precond, "iterations", it, "residual", res)
    est, true = eb.bem_gmres_history(op)
    assert len(est) == it and est[-1] <= 1e-6 and true[0] == 1.0
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
                                       tol=1e-6, precond=precond, check=False)
    assert it2 == 3 and res2 > 1e-6
    # a warm start (nonzero initial guess: the dense solution perturbed by 1%) takes the
    # r0 = b - A x0 branch and reaches the same solution
    rng = np.random.default_rng(3)
    x0 = (xref.reshape(-1, 3) * (1 + 0.01 * rng.standard_normal((len(bc), 3)))).astype(np.float32)
    x3 = torch.from_numpy(x0).cuda()
    x3, it3, res3 = eb.bem_gmres_solve(op, torch.from_numpy(bc).cuda(),
                                       torch.from_numpy(val.astype(np.float32)).cuda(), x3, restart=50,
                                       max_iter=300, tol=1e-6, precond=precond)
    est3, true3 = eb.bem_gmres_history(op)
    print("warm start: iterations", it3, "first true residual", true3[0])
    assert res3 <= 1e-6 and 1e-6 < true3[0] < 1.0
    assert KN.rel_l2(x3.cpu().numpy().reshape(-1).astype(np.float64), xref) < 1e-4


def test_gmres_solver_setting_of_configs4_matches_dense_oracle(eb):
    """configs[4]'s solver setting -- block-Jacobi right preconditioner, tol 1e-6 (so the
    full-chain tensor-core M2L), the near operator held in HBM, sources grouped per leaf by
    panel type, p = 8 -- on a small voided cell (unit cube 6 x 6 cells per face + two
    icosphere voids: 1024 panels, 16384 quadrature sources) with 64 sources per leaf, so the
    tree has several levels and every list kind, against dense LU of the oracle's system
    (PAPER.md Eqs. num, num2; l. 181 GMRES, l. 187 16-point quadrature)."""
    d = geo.metamaterial_cell(nc=6, level=1, nvoids=2, seed=5)
    verts = d["verts"]
    V0, V1, V2 = (verts[:, k].astype(np.float64) for k in range(3))
    c64, n64, a64 = geo.panels(V0, V1, V2)
    U, P = OB.assemble(c64, n64, a64, V0, V1, V2, d["K"], d["G"], nq=16)
    A, b = OB.mixed_system(U, P, d["bc_type"], d["bc_val"])
    xref = np.linalg.solve(A, b)
    op = eb.bem_create(torch.from_numpy(verts).cuda(), nq=16, max_pts=64, p=8, K=d["K"], G=d["G"])
    bc, val = torch.from_numpy(d["bc_type"]).cuda(), torch.from_numpy(d["bc_val"]).cuda()
    # the operator itself (bem_apply) and the right-hand side against the dense system
    rng = np.random.default_rng(2)
    xr = rng.standard_normal(A.shape[0]).astype(np.float32)
    y = eb.bem_apply(op, bc, torch.from_numpy(xr).cuda().view(-1, 3)).cpu().numpy().reshape(-1)
    assert KN.rel_l2(y, A @ xr.astype(np.float64)) < 1e-5
    bg = eb.bem_rhs(op, bc, val).cpu().numpy().reshape(-1)
    assert KN.rel_l2(bg, b) < 1e-5
    x = torch.zeros((verts.shape[0], 3), device="cuda")
    x, it, res = eb.bem_gmres_solve(op, bc, val, x, restart=50, max_iter=400, tol=1e-6, precond=1)
    err = KN.rel_l2(x.cpu().numpy().reshape(-1).astype(np.float64), xref)
    print("voided cell: iterations", it, "residual", res, "solution rel-L2 vs dense LU", err,
          "cond", np.linalg.cond(A))
    assert res <= 1e-6 and err < 1e-4
    # true residual of the returned solution against the oracle's own matrix
    xs = x.cpu().numpy().reshape(-1).astype(np.float64)
    assert np.linalg.norm(b - A @ xs) / np.linalg.norm(b) < 1e-4
    # the leaf-block Jacobi preconditioner (precond = 2): the same solution in fewer
    # iterations (its blocks are A's own diagonal blocks over each leaf's panels)
    x2 = torch.zeros((verts.shape[0], 3), device="cuda")
    x2, it2, res2 = eb.bem_gmres_solve(op, bc, val, x2, restart=50, max_iter=400, tol=1e-6, precond=2)
    err2 = KN.rel_l2(x2.cpu().numpy().reshape(-1).astype(np.float64), xref)
    print("leaf-block Jacobi: iterations", it2, "residual", res2, "solution rel-L2 vs dense LU", err2)
    assert res2 <= 1e-6 and err2 < 1e-4 and it2 < it


def test_near_operator_matches_near_kernel(eb, monkeypatch):
    """The BEM near field held in HBM (bem_near.cu: per-leaf 3x3 blocks of the summed
    quadrature-point kernels), the S2M / S2L check-potential operators built the same way, and
    the per-leaf grouping of sources by panel type (one-layer check-potential loops) against
    the pair-by-pair near-field and check-potential kernels and the combined loop:
    same solve to fp32 rounding, on a cell with voids (leaves straddling panels, direct X/W
    entries); the stored operator is reused for the same boundary conditions and rebuilt
    when they change (the grouping then changes too)."""
    d = geo.metamaterial_cell(nc=24, level=2, nvoids=4, seed=3)
    verts = torch.from_numpy(d["verts"]).cuda()
    val = torch.from_numpy(d["bc_val"]).cuda()
    op = eb.bem_create(verts, nq=16, max_pts=256, p=6, K=d["K"], G=d["G"])

    def solve(bc_np):
        bc = torch.from_numpy(bc_np).cuda()
        x = torch.zeros((d["verts"].shape[0], 3), device="cuda")
        x, it, res = eb.bem_gmres_solve(op, bc, val, x, restart=30, max_iter=300, tol=1e-6, precond=1, check=False)
        return x.cpu().numpy().reshape(-1), it, res

    bc0 = d["bc_type"].astype(np.int32)
    bc1 = bc0.copy()
    bc1[: len(bc1) // 7] = 0          # more Dirichlet panels: the blocks change kind
    ref = []
    monkeypatch.setenv("EBEM_BEM_NEARMAT", "0")
    monkeypatch.setenv("EBEM_BEM_SPLIT", "0")       # and the combined U+P check-potential loop
    for bc in (bc0, bc1):
        ref.append(solve(bc))
    monkeypatch.setenv("EBEM_BEM_NEARMAT", "1")
    monkeypatch.setenv("EBEM_BEM_SPLIT", "1")       # sources grouped by panel type per leaf
    for checkmat in ("0", "1"):                     # near operator alone; + S2M / S2L operators
        monkeypatch.setenv("EBEM_BEM_CHECKMAT", checkmat)
        for k, bc in enumerate((bc0, bc0, bc1)):      # build, reuse, rebuild
            x, it, res = solve(bc)
            xr, itr, resr = ref[0 if k < 2 else 1]
            print("near operator, check operators", checkmat, k, "iterations", it, itr, "residual", res, resr)
            assert res <= 1e-6 and abs(it - itr) <= 3
            assert KN.rel_l2(x, xr) < 1e-4      # both stop at residual 1e-6; a wrong block is O(1)


def test_near_operator_memory_fallback_and_nq1(eb, monkeypatch):
    """When the near operator does not fit its memory budget the solve runs the near-field
    kernel instead (same answer); with one quadrature point per panel (nq = 1) the stored
    operator holds one point per block and matches the kernel path too."""
    verts, c, n, a, bc, val, uex, tex, V = _problem(4)
    bcd, vald = torch.from_numpy(bc).cuda(), torch.from_numpy(val.astype(np.float32)).cuda()
    for nq in (16, 1):
        sols = []
        for frac in ("0.6", "1e-12"):          # 1e-12: nothing fits, the kernel path runs
            monkeypatch.setenv("EBEM_BEM_NEARMAT_FRAC", frac)
            op2 = eb.bem_create(torch.from_numpy(verts).cuda(), nq=nq, max_pts=32, p=8, K=KB, G=G)
            x = torch.zeros((len(bc), 3), device="cuda")
            x, it, res = eb.bem_gmres_solve(op2, bcd, vald, x, restart=50, max_iter=300, tol=1e-6)
            assert res <= 1e-6
            sols.append(x.cpu().numpy().reshape(-1))
        print("nq", nq, "near operator vs kernel:", KN.rel_l2(sols[0], sols[1]))
        assert KN.rel_l2(sols[0], sols[1]) < 1e-4
