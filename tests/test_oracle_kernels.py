"""Pins for oracle/kernels.py against the mathematics (not against itself).

Each pin names what fixes the expected value: a hand-evaluated closed form, the
reciprocity symmetry, the Navier equilibrium equation, the rigid-translation
identity of the double layer over a closed sphere, the Somigliana identity
(PAPER.md Eq. BIE with c = 1 inside), Betti reciprocity, the constitutive law
C_ijkl eps_kl (PAPER.md Eq. elast) by finite differences and by sympy.
"""
import itertools

import numpy as np
import pytest

from oracle import kernels as K

RNG = np.random.default_rng(1234)


def sphere_quadrature(R=1.0, center=(0.0, 0.0, 0.0), nt=48, nph=96):
    """Gauss-Legendre in cos(theta) x trapezoid in phi: exponentially accurate for
    integrands smooth on the sphere (used to integrate the kernels over a closed surface)."""
    mu, wmu = np.polynomial.legendre.leggauss(nt)
    ph = (np.arange(nph) + 0.5) * 2 * np.pi / nph
    MU, PH = np.meshgrid(mu, ph, indexing="ij")
    st = np.sqrt(1 - MU ** 2)
    nrm = np.stack([st * np.cos(PH), st * np.sin(PH), MU], -1).reshape(-1, 3)
    w = (wmu[:, None] * np.full(nph, 2 * np.pi / nph)[None, :]).reshape(-1) * R * R
    pts = np.asarray(center) + R * nrm
    return pts, nrm, w


# ---------------------------------------------------------------- material
def test_moduli_identities():
    # E = 2G(1+nu) = 3K(1-2nu): two independent isotropic identities
    for Kb, G in [(1.0, 0.5), (1.67, 0.77), (10.0, 1.0)]:
        nu = K.poisson_ratio(Kb, G)
        E = K.young_modulus(Kb, G)
        assert abs(E - 2 * G * (1 + nu)) < 1e-12 * E
        assert abs(E - 3 * Kb * (1 - 2 * nu)) < 1e-12 * E
    # PAPER.md Sec. 3 benchmark: E = 1, nu = 0.3  ->  G = 1/2.6, K = 1/1.2
    assert abs(K.poisson_ratio(1 / 1.2, 1 / 2.6) - 0.3) < 1e-14


def test_stiffness_is_isotropic_hooke():
    # C_ijkl eps_kl must equal lambda tr(eps) d_ij + 2 G eps_ij, lambda = K - 2G/3
    Kb, G = 1.67, 0.77
    C = K.stiffness(Kb, G)
    eps = RNG.standard_normal((3, 3))
    eps = eps + eps.T
    sig = np.einsum("ijkl,kl->ij", C, eps)
    lam = Kb - 2 * G / 3
    assert np.allclose(sig, lam * np.trace(eps) * np.eye(3) + 2 * G * eps, atol=1e-13)


# ---------------------------------------------------------------- U closed forms
def test_U_hand_values():
    # nu = 0.3, G = 1, r-vector (1,0,0): U_11 = (3 - 1.2 + 1)/(16 pi 0.7), U_22 = U_33 = 1.8/(16 pi 0.7)
    nu, G = 0.3, 1.0
    U = K.kernel_U(np.array([1.0, 0, 0]), np.zeros(3), G, nu)
    expect = np.diag([2.8, 1.8, 1.8]) / (16 * np.pi * 0.7)
    assert np.allclose(U, expect, rtol=0, atol=1e-15)
    # along the diagonal (1,1,1)/sqrt3 at r = 2: U_12 = (1/3)/(16 pi 0.7 * 2)
    U = K.kernel_U(np.array([1.0, 1, 1]) * 2 / np.sqrt(3), np.zeros(3), G, nu)
    assert abs(U[0, 1] - (1 / 3) / (16 * np.pi * 0.7 * 2)) < 1e-15
    assert abs(U[0, 0] - (1.8 + 1 / 3) / (16 * np.pi * 0.7 * 2)) < 1e-15


def test_U_reciprocity_and_homogeneity():
    x = RNG.standard_normal((50, 3))
    y = RNG.standard_normal((50, 3))
    G, nu = 0.77, 0.3
    Uxy = K.kernel_U(x, y, G, nu)
    Uyx = K.kernel_U(y, x, G, nu)
    assert np.allclose(Uxy, np.swapaxes(Uyx, -1, -2), rtol=1e-14, atol=0)
    # homogeneity of degree -1 (U), -2 (P, D), -3 (S)
    n = RNG.standard_normal((50, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    lam = 2.5
    assert np.allclose(K.kernel_U(lam * x, lam * y, G, nu), Uxy / lam, rtol=1e-13)
    assert np.allclose(K.kernel_P(lam * x, lam * y, n, nu), K.kernel_P(x, y, n, nu) / lam ** 2, rtol=1e-13)
    assert np.allclose(K.kernel_D(lam * x, lam * y, nu), K.kernel_D(x, y, nu) / lam ** 2, rtol=1e-13)
    assert np.allclose(K.kernel_S(lam * x, lam * y, n, G, nu), K.kernel_S(x, y, n, G, nu) / lam ** 3, rtol=1e-13)


def _fd_grad(fun, x, h):
    """central differences d/dx_n of fun(x) -> array with a trailing axis n."""
    out = []
    for a in range(3):
        e = np.zeros(3)
        e[a] = h
        out.append((fun(x + e) - fun(x - e)) / (2 * h))
    return np.stack(out, -1)


def test_U_satisfies_navier_equilibrium():
    # G lap u + (lambda + G) grad div u = 0 away from the source, u_m = U_mk e_k
    Kb, G = 1.67, 0.77
    nu = K.poisson_ratio(Kb, G)
    lam = Kb - 2 * G / 3
    y = np.zeros(3)
    h = 1e-3
    for _ in range(5):
        x = RNG.standard_normal(3)
        x *= 1.3 / np.linalg.norm(x)
        e = RNG.standard_normal(3)
        u = lambda p: K.kernel_U(p, y, G, nu) @ e
        grad = lambda p: _fd_grad(u, p, h)                 # [m, n] = du_m/dx_n
        H = _fd_grad(grad, x, h)                           # [m, n, l]
        lap = np.einsum("mnn->m", H)
        graddiv = np.einsum("nnm->m", H)
        res = G * lap + (lam + G) * graddiv
        scale = G * np.abs(np.einsum("mnn->m", np.abs(H))).max()
        assert np.abs(res).max() < 1e-5 * scale


# ---------------------------------------------------------------- P: rigid translation
@pytest.mark.parametrize("nu", [0.0, 0.3, 0.2857142857142857, 0.45])
def test_P_rigid_translation_identity_sphere(nu):
    """int_{sphere} P_ij(xi, x) dGamma_x = -delta_ij for xi inside, 0 outside
    (rigid translation u = e, p = 0 in PAPER.md Eq. BIE, with c = 1 inside, 0 outside)."""
    pts, nrm, w = sphere_quadrature(R=1.3, center=(0.2, -0.1, 0.3))
    for xi, expect in [((0.2, -0.1, 0.3), -np.eye(3)), ((0.5, 0.1, 0.6), -np.eye(3)),
                       ((0.0, -0.4, 0.1), -np.eye(3)), ((3.0, 2.0, -1.0), np.zeros((3, 3))),
                       ((0.2, -0.1, 2.5), np.zeros((3, 3)))]:
        P = K.kernel_P(np.asarray(xi)[None, :], pts, nrm, nu)
        integral = np.einsum("sij,s->ij", P, w)
        assert np.allclose(integral, expect, atol=1e-10), (xi, integral)


def _kelvin_state(xf, e, pts, nrm, Kb, G):
    """displacement and traction on (pts, nrm) of the Kelvin solution of a unit force e at xf.
    The traction uses D (stress of a point force) -- pinned independently by the FD tests."""
    nu = K.poisson_ratio(Kb, G)
    u = np.einsum("sij,j->si", K.kernel_U(pts, xf[None, :], G, nu), e)
    sig = np.einsum("skij,k->sij", K.kernel_D(pts, xf[None, :], nu), e)
    t = np.einsum("sij,sj->si", sig, nrm)
    return u, t


def test_somigliana_identity_interior():
    """PAPER.md Eq. BIE with c_ij = delta_ij at an interior point:
    u_i(xi) = int U_ij p_j - int P_ij u_j for a regular state (force outside the sphere)."""
    Kb, G = 1.67, 0.77
    nu = K.poisson_ratio(Kb, G)
    pts, nrm, w = sphere_quadrature(R=1.0, nt=64, nph=128)
    xf = np.array([2.1, -1.4, 0.7])
    e = np.array([0.3, -1.0, 0.6])
    u, t = _kelvin_state(xf, e, pts, nrm, Kb, G)
    for xi in [np.zeros(3), np.array([0.3, 0.2, -0.4]), np.array([-0.5, 0.1, 0.2])]:
        lhs = K.kernel_U(xi, xf, G, nu) @ e
        Uq = K.kernel_U(xi[None, :], pts, G, nu)
        Pq = K.kernel_P(xi[None, :], pts, nrm, nu)
        rhs = np.einsum("sij,sj,s->i", Uq, t, w) - np.einsum("sij,sj,s->i", Pq, u, w)
        assert np.allclose(rhs, lhs, rtol=1e-9, atol=1e-12), (rhs, lhs)
        # and the exterior version is 0 (c = 0)
    xo = np.array([0.0, 0.0, 1.8])
    Uq = K.kernel_U(xo[None, :], pts, G, nu)
    Pq = K.kernel_P(xo[None, :], pts, nrm, nu)
    rhs = np.einsum("sij,sj,s->i", Uq, t, w) - np.einsum("sij,sj,s->i", Pq, u, w)
    # the force point itself lies outside; a point outside Gamma but not the force point sees
    # the exterior integral of a state regular inside -> 0
    assert np.abs(rhs).max() < 1e-9


def test_betti_reciprocity():
    """int t1 . u2 = int t2 . u1 over a closed surface for two states regular inside."""
    Kb, G = 1.0, 0.5
    pts, nrm, w = sphere_quadrature(R=1.0, nt=64, nph=128)
    u1, t1 = _kelvin_state(np.array([1.9, 0.4, -0.3]), np.array([1.0, 0.2, 0.0]), pts, nrm, Kb, G)
    u2, t2 = _kelvin_state(np.array([-0.6, 2.2, 1.1]), np.array([0.0, -0.5, 1.0]), pts, nrm, Kb, G)
    a = np.sum(np.sum(t1 * u2, 1) * w)
    b = np.sum(np.sum(t2 * u1, 1) * w)
    assert abs(a - b) < 1e-10 * max(abs(a), 1e-3)


# ---------------------------------------------------------------- D, S: constitutive law
def _stress_from_displacement(kfun, x, Cmat, h=1e-5):
    """sigma_ij[k] = C_ijmn d_n u_m for u_m = kfun(x)[m, k] (central differences)."""
    grad = _fd_grad(kfun, x, h)                 # [m, k, n]
    return np.einsum("ijmn,mkn->kij", Cmat, grad)


@pytest.mark.parametrize("Kb,G", [(1.0, 0.5), (1.67, 0.77)])
def test_D_is_C_grad_U(Kb, G):
    nu = K.poisson_ratio(Kb, G)
    C = K.stiffness(Kb, G)
    y = RNG.standard_normal(3)
    for _ in range(4):
        x = y + RNG.standard_normal(3)
        fd = _stress_from_displacement(lambda p: K.kernel_U(p, y, G, nu), x, C)
        D = K.kernel_D(x, y, nu)
        assert np.allclose(D, fd, rtol=1e-6, atol=1e-8 * np.abs(D).max())


@pytest.mark.parametrize("Kb,G", [(1.0, 0.5), (1.67, 0.77)])
def test_S_is_C_grad_P(Kb, G):
    nu = K.poisson_ratio(Kb, G)
    C = K.stiffness(Kb, G)
    y = RNG.standard_normal(3)
    n = RNG.standard_normal(3)
    n /= np.linalg.norm(n)
    for _ in range(4):
        x = y + RNG.standard_normal(3)
        fd = _stress_from_displacement(lambda p: K.kernel_P(p, y, n, nu), x, C)
        S = K.kernel_S(x, y, n, G, nu)
        assert np.allclose(S, fd, rtol=1e-6, atol=1e-8 * np.abs(S).max())


def test_D_S_equilibrium_and_symmetry():
    Kb, G = 1.67, 0.77
    nu = K.poisson_ratio(Kb, G)
    y = np.zeros(3)
    n = np.array([0.48, 0.6, 0.64])
    for _ in range(3):
        x = RNG.standard_normal(3)
        D = K.kernel_D(x, y, nu)
        S = K.kernel_S(x, y, n, G, nu)
        assert np.allclose(D, np.swapaxes(D, 1, 2), atol=1e-15)
        assert np.allclose(S, np.swapaxes(S, 1, 2), atol=1e-15)
        r = np.linalg.norm(x)
        # FD truncation is O(h^2 f'''); compare with the gradient scale |f| / r
        divD = np.einsum("kijj->ki", _fd_grad(lambda p: K.kernel_D(p, y, nu), x, 1e-4 * r))
        divS = np.einsum("kijj->ki", _fd_grad(lambda p: K.kernel_S(p, y, n, G, nu), x, 1e-4 * r))
        assert np.abs(divD).max() < 1e-6 * np.abs(D).max() / r
        assert np.abs(divS).max() < 1e-6 * np.abs(S).max() / r


def test_D_S_symbolic():
    """sympy differentiates Eq. disp_1 / disp_2 and applies C_ijkl: an independent derivation."""
    sp = pytest.importorskip("sympy")
    xs = sp.symbols("x0:3", real=True)
    ns = sp.symbols("n0:3", real=True)
    Gs, nus = sp.Rational(77, 100), sp.Rational(3, 10)
    r = sp.sqrt(sum(v ** 2 for v in xs))
    dl = lambda i, j: 1 if i == j else 0
    rh = [v / r for v in xs]
    U = [[((3 - 4 * nus) * dl(i, j) + rh[i] * rh[j]) / (16 * sp.pi * (1 - nus) * Gs * r) for j in range(3)] for i in range(3)]
    drdn = sum(rh[i] * ns[i] for i in range(3))
    P = [[(drdn * ((1 - 2 * nus) * dl(i, j) + 3 * rh[i] * rh[j]) - (1 - 2 * nus) * (rh[i] * ns[j] - rh[j] * ns[i]))
          / (8 * sp.pi * (1 - nus) * r ** 2) for j in range(3)] for i in range(3)]
    lam = 2 * Gs * nus / (1 - 2 * nus)
    Cf = lambda i, j, k, l: lam * dl(i, j) * dl(k, l) + Gs * (dl(i, k) * dl(j, l) + dl(i, l) * dl(j, k))
    xv = np.array([0.3, -0.7, 0.45])
    nv = np.array([0.48, 0.6, 0.64])
    sub = {xs[0]: xv[0], xs[1]: xv[1], xs[2]: xv[2], ns[0]: nv[0], ns[1]: nv[1], ns[2]: nv[2]}
    D = K.kernel_D(xv, np.zeros(3), 0.3)
    S = K.kernel_S(xv, np.zeros(3), nv, 0.77, 0.3)
    for k, i, j in itertools.product(range(3), range(3), range(3)):
        sd = sum(Cf(i, j, m, q) * sp.diff(U[m][k], xs[q]) for m in range(3) for q in range(3))
        ss = sum(Cf(i, j, m, q) * sp.diff(P[m][k], xs[q]) for m in range(3) for q in range(3))
        assert abs(float(sd.subs(sub)) - D[k, i, j]) < 1e-13
        assert abs(float(ss.subs(sub)) - S[k, i, j]) < 1e-13


def test_stress_somigliana_interior():
    """PAPER.md Eq. stress_1: sigma_ij(p) = -int u_k S_kij + int t_k D_kij, checked against
    the stress of the Kelvin state evaluated directly."""
    Kb, G = 1.67, 0.77
    nu = K.poisson_ratio(Kb, G)
    pts, nrm, w = sphere_quadrature(R=1.0, nt=64, nph=128)
    xf = np.array([-1.7, 1.2, 0.9])
    e = np.array([0.2, 0.9, -0.4])
    u, t = _kelvin_state(xf, e, pts, nrm, Kb, G)
    for p in [np.zeros(3), np.array([0.2, -0.3, 0.25])]:
        expect = np.einsum("kij,k->ij", K.kernel_D(p, xf, nu), e)
        Dq = K.kernel_D(p[None, :], pts, nu)
        Sq = K.kernel_S(p[None, :], pts, nrm, G, nu)
        got = np.einsum("skij,sk,s->ij", Dq, t, w) - np.einsum("skij,sk,s->ij", Sq, u, w)
        assert np.allclose(got, expect, rtol=1e-8, atol=1e-11)


# ---------------------------------------------------------------- direct sum
def test_direct_sum_matches_pair_loop():
    """pure-Python pair loop on a tiny case (the plain definition of Eq. fmm_summation)."""
    Kb, G = 1.0, 0.5
    nu = K.poisson_ratio(Kb, G)
    src = RNG.standard_normal((7, 3))
    trg = np.concatenate([RNG.standard_normal((4, 3)), src[:2]])   # two coincident points
    nrm = RNG.standard_normal((7, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    w = RNG.uniform(0.5, 1.5, 7)
    f = RNG.standard_normal((7, 3))
    g = RNG.standard_normal((7, 3))
    for kern in (K.KERNEL_U, K.KERNEL_P, K.KERNEL_UP, K.KERNEL_D, K.KERNEL_S, K.KERNEL_DS):
        got = K.direct_sum(kern, trg, src, Kb, G, w=w, f=f, g=g, nrm=nrm)
        ref = np.zeros_like(got)
        for i in range(trg.shape[0]):
            for j in range(7):
                if np.all(trg[i] == src[j]):
                    continue
                if kern in (K.KERNEL_U, K.KERNEL_P, K.KERNEL_UP):
                    v = np.zeros(3)
                    if kern != K.KERNEL_P:
                        v += K.kernel_U(trg[i], src[j], G, nu) @ f[j]
                    if kern != K.KERNEL_U:
                        v += K.kernel_P(trg[i], src[j], nrm[j], nu) @ g[j]
                else:
                    s = np.zeros((3, 3))
                    if kern != K.KERNEL_S:
                        s += np.einsum("kij,k->ij", K.kernel_D(trg[i], src[j], nu), f[j])
                    if kern != K.KERNEL_D:
                        s += np.einsum("kij,k->ij", K.kernel_S(trg[i], src[j], nrm[j], G, nu), g[j])
                    v = np.array([s[a, b] for a, b in K.VOIGT])
                ref[i] += w[j] * v
        assert np.allclose(got, ref, rtol=1e-13, atol=1e-14)
