"""Pins for oracle/bem.py: singular self-integrals against a closed form and an independent
Duffy-transformed 2-D quadrature, the CPV term against symmetry and a second formula,
GMRES against dense LU, and the collocation system against the exact uniaxial patch test."""
import numpy as np
import pytest

from oracle import bem as B
from oracle import kernels as KN
from workloads import geometry as geo

RNG = np.random.default_rng(5)


def _rand_tri():
    """a random, not too degenerate triangle (perturbed equilateral, random pose)"""
    V = np.array([[0, 0, 0], [1, 0, 0], [0.5, np.sqrt(3) / 2, 0.0]]) + 0.25 * RNG.standard_normal((3, 3))
    R = np.linalg.qr(RNG.standard_normal((3, 3)))[0]
    return V @ R.T + RNG.standard_normal(3)


def test_self_U_equilateral_closed_form():
    G, nu = 0.77, 0.3
    s = 0.7
    V = np.array([[0, 0, 0], [s, 0, 0], [s / 2, s * np.sqrt(3) / 2, 0.0]])
    R = np.linalg.qr(RNG.standard_normal((3, 3)))[0]      # arbitrary rotation
    V = V @ R.T + RNG.standard_normal(3)
    n = np.cross(V[1] - V[0], V[2] - V[0])
    n /= np.linalg.norm(n)
    got = B.self_U_polar(V, G, nu)
    assert np.allclose(got, B.self_U_closed_equilateral(s, n, G, nu), rtol=1e-12, atol=1e-15)


def test_self_U_matches_duffy_quadrature():
    """independent 2-D evaluation: Duffy map of each sub-triangle (xi, A, B),
    x = xi + u (a + v (b - a)), Jacobian u |a x b|, Gauss-Legendre in u and v."""
    G, nu = 0.5, 0.25
    g, w = np.polynomial.legendre.leggauss(64)
    s, ws = 0.5 * (g + 1), 0.5 * w
    for _ in range(3):
        V = _rand_tri()
        xi = V.mean(0)
        tot = np.zeros((3, 3))
        for k in range(3):
            a, b = V[k] - xi, V[(k + 1) % 3] - xi
            cr = np.linalg.norm(np.cross(a, b))
            U, Vv = np.meshgrid(s, s, indexing="ij")
            W = np.outer(ws, ws)
            X = xi + U[..., None] * (a + Vv[..., None] * (b - a))
            K = KN.kernel_U(xi[None, None, :], X, G, nu)
            tot += np.einsum("uv,uvij->ij", W * U * cr, K)
        assert np.allclose(B.self_U_polar(V, G, nu), tot, rtol=1e-9, atol=1e-13)


def test_self_P_cpv_symmetry_and_second_formula():
    nu = 0.3
    s = 1.3
    V = np.array([[0, 0, 0], [s, 0, 0], [s / 2, s * np.sqrt(3) / 2, 0.0]])
    assert np.abs(B.self_P_cpv(V, nu)).max() < 1e-14          # 3-fold symmetry
    # general triangle: divergence-theorem (edges) vs polar CPV int r(theta) ln R(theta) dtheta
    g, w = np.polynomial.legendre.leggauss(80)
    for _ in range(3):
        V = _rand_tri()
        xi = V.mean(0)
        n = np.cross(V[1] - V[0], V[2] - V[0])
        n /= np.linalg.norm(n)
        I = np.zeros(3)       # CPV int e(theta)/rho dS, e = (x - xi)/rho
        for k in range(3):
            a, b = V[k] - xi, V[(k + 1) % 3] - xi
            s_ = 0.5 * (g + 1)
            P = a + s_[:, None] * (b - a)
            R = np.linalg.norm(P, axis=1)
            dth = np.linalg.norm(np.cross(a, b)) / R ** 2 * 0.5 * w
            I += np.sum((P / R[:, None]) * (np.log(R) * dth)[:, None], axis=0)
        # r = (xi - x)/rho = -e
        c = -(1 - 2 * nu) / (8 * np.pi * (1 - nu))
        ref = c * ((-I)[:, None] * n[None, :] - n[:, None] * (-I)[None, :])
        assert np.allclose(B.self_P_cpv(V, nu), ref, rtol=1e-10, atol=1e-14)


def test_quadrature_rule():
    V0, V1, V2 = (RNG.standard_normal((5, 3)) for _ in range(3))
    qp, qw = B.quadrature(V0, V1, V2, 16)
    area = 0.5 * np.linalg.norm(np.cross(V1 - V0, V2 - V0), axis=1)
    assert np.allclose(qw.sum(1), area, rtol=1e-13)
    # degree-3 exactness on each sub-triangle => exact for cubic polynomials
    f = lambda x: x[..., 0] ** 3 - 2 * x[..., 1] ** 2 * x[..., 2] + x[..., 0] * x[..., 2] + 1
    # reference: same integral by a 1-level finer 16-point rule (exact for cubics too)
    M01, M12, M20 = (V0 + V1) / 2, (V1 + V2) / 2, (V2 + V0) / 2
    ref = 0
    for A, Bv, C in ((V0, M01, M20), (M01, V1, M12), (M20, M12, V2), (M01, M12, M20)):
        q2, w2 = B.quadrature(A, Bv, C, 16)
        ref = ref + np.sum(f(q2) * w2, 1)
    assert np.allclose(np.sum(f(qp) * qw, 1), ref, rtol=1e-12)


def test_gmres_against_lu():
    n = 60
    A = np.eye(n) * 4 + RNG.standard_normal((n, n)) / np.sqrt(n)
    b = RNG.standard_normal(n)
    x, it, hist = B.gmres(lambda v: A @ v, b, restart=20, tol=1e-12, max_iter=500)
    assert np.allclose(x, np.linalg.solve(A, b), rtol=1e-9, atol=1e-10)
    x, it, _ = B.gmres(lambda v: v, b, tol=1e-12)
    assert it == 1 and np.allclose(x, b)
    x, it, _ = B.gmres(lambda v: A @ v, np.zeros(n))
    assert it == 0 and np.all(x == 0)


def _patch(nc, nq):
    E, nu = 1.0, 0.3
    G, Kb = E / (2 * (1 + nu)), E / (3 * (1 - 2 * nu))
    V0, V1, V2 = geo.cube_voxel_faces(nc)
    c, n, a = geo.panels(V0, V1, V2)
    uex = np.stack([-nu * c[:, 0] / E, -nu * c[:, 1] / E, c[:, 2] / E], 1)   # sigma = e_z e_z
    tex = np.stack([0 * c[:, 0], 0 * c[:, 0], n[:, 2]], 1)
    bc = np.where(c[:, 2] < 1e-9, 0, 1)      # Dirichlet on z = 0, Neumann elsewhere
    val = np.where(bc[:, None] == 0, uex, tex)
    U, P = B.assemble(c, n, a, V0, V1, V2, Kb, G, nq=nq)
    A, b = B.mixed_system(U, P, bc, val)
    return A, b, bc, uex, tex, P


def test_patch_test_uniaxial():
    """PAPER.md Sec. 3 benchmark material (E = 1, nu = 0.3) under uniform tension: the exact
    solution is linear; the 16-point collocation BEM reproduces it to a few percent."""
    A, b, bc, uex, tex, P = _patch(3, 16)
    x = np.linalg.solve(A, b).reshape(-1, 3)
    m = bc == 1
    assert np.linalg.norm(x[m] - uex[m]) / np.linalg.norm(uex[m]) < 0.05
    assert np.linalg.norm(x[~m] - tex[~m]) / np.linalg.norm(tex[~m]) < 0.05
    # rigid translation is (nearly) annihilated by (1/2 I + P)
    one = np.tile([0.0, 1.0, 0.0], len(bc))
    assert np.abs(P @ one).max() < 0.02
    # GMRES reaches the LU solution
    xg, it, hist = B.gmres(lambda v: A @ v, b, restart=50, tol=1e-10, max_iter=300)
    assert np.allclose(xg, x.reshape(-1), rtol=1e-7, atol=1e-9)
