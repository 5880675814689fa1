"""Oracle: collocation BEM system of PAPER.md Eqs. (BIE), (num), (coef), (num2) and the
restarted GMRES that solves it.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product path.

Discretisation: piecewise-constant u and p on flat triangles,
collocation at centroids.  Off-diagonal panel integrals use the paper's rule, "Each
triangular element contains 16 quadrature points ... (the element is subdivided into four
equal triangular parts, and the 4-node Gauss quadrature is used for each part)" (l. 187),
or (nq = 1) the centroid rule of the benchmark configs (reading R9).  The singular
own-panel integrals are evaluated exactly ("The singular integrals over triangles are
evaluated analytically", l. 179):
    U_self = int_T U(xi, x) dS          (weakly singular; polar coordinates about xi)
    P_self = CPV int_T P(xi, x) dS      (in-plane: only the (1-2nu)(r_i n_j - r_j n_i) term)
and the free term of Eq. (BIE) is 1/2 I (smooth point).  Row i of Eq. (num):
    (1/2 I + P_self_i) u_i + sum_{j != i} P(xi_i, x_j) a_j u_j
        = U_self_i p_i + sum_{j != i} U(xi_i, x_j) a_j p_j.
Mixed BVP (Eq. elast): on Dirichlet panels u is given and p unknown, on Neumann panels
p is given and u unknown; moving the unknowns to the left gives A x = b (Eq. num2).
"""
from __future__ import annotations

import numpy as np

from . import kernels as KN


# ------------------------------------------------------------------ self integrals
def _edge_pieces(V, xi):
    """for each edge (A,B) of triangle V: foot distance h, unit in-plane directions."""
    out = []
    for k in range(3):
        A, B = V[k], V[(k + 1) % 3]
        out.append((A, B))
    return out


def self_U_polar(V, G, nu, nq=64):
    """int_T U(xi, x) dS at the centroid xi in polar coordinates about xi over the three
    sub-triangles (xi, A, B): U r dr dtheta = f(theta) dr, so the radial integral is
    R(theta) f(theta) and the remaining angular integral (smooth) uses Gauss-Legendre along
    each edge."""
    V = np.asarray(V, np.float64)
    xi = V.mean(axis=0)
    g, w = np.polynomial.legendre.leggauss(nq)
    total = np.zeros((3, 3))
    for A, B in _edge_pieces(V, xi):
        a, b = A - xi, B - xi
        # points on segment AB: a + s (b - a), s in [0,1]; map to polar angle via the segment
        s = 0.5 * (g + 1.0)
        P = a[None, :] + s[:, None] * (b - a)[None, :]         # boundary points
        R = np.linalg.norm(P, axis=1)
        e = P / R[:, None]
        # d(theta)/ds = |a x b| / R^2 (in-plane), so int dtheta int_0^R f(e) (1/r) r dr
        #   = int ds |a x b| / R^2 * R * f(e)  for f homogeneous of degree -1 (U)
        cross = np.linalg.norm(np.cross(a, b))
        jac = 0.5 * w * cross / R ** 2
        # U(xi, x) with r-vector xi - x = -rho e: U depends on e e^T only (even)
        c = 1.0 / (16.0 * np.pi * (1.0 - nu) * G)
        f = c * ((3.0 - 4.0 * nu) * np.eye(3)[None] + e[:, :, None] * e[:, None, :])
        total += np.einsum("q,qij->ij", jac * R, f)
    return total


def self_U_closed_equilateral(side, n, G, nu):
    """closed form for an equilateral triangle (centroid): int 1/r dS = 6 h ln(2+sqrt3),
    h = side/(2 sqrt3) the inradius, and by in-plane isotropy
    int r_i r_j / r dS = 1/2 (delta_ij - n_i n_j) int 1/r dS."""
    h = side / (2.0 * np.sqrt(3.0))
    I1 = 6.0 * h * np.log(2.0 + np.sqrt(3.0))
    n = np.asarray(n, np.float64)
    c = 1.0 / (16.0 * np.pi * (1.0 - nu) * G)
    return c * ((3.0 - 4.0 * nu) * I1 * np.eye(3) + 0.5 * I1 * (np.eye(3) - np.outer(n, n)))


def self_P_cpv(V, nu, nq=64):
    """CPV int_T P(xi, x) dS at the centroid of a flat triangle.  With xi in the plane,
    dr/dn = 0 and P_ij = -(1-2nu)(r_i n_j - r_j n_i) / (8 pi (1-nu) rho^2), r = (xi - x)/rho.
    In the plane, e/rho^2 = grad_x(-1/rho) with e = (x - xi)/rho, and by the divergence
    theorem on T minus a small disk, CPV int_T e/rho^2 dS = -sum_edges int_edge nu_edge/rho ds
    (the disk term is int e dtheta = 0)."""
    V = np.asarray(V, np.float64)
    xi = V.mean(axis=0)
    cr = np.cross(V[1] - V[0], V[2] - V[0])
    n = cr / np.linalg.norm(cr)
    g, w = np.polynomial.legendre.leggauss(nq)
    J = np.zeros(3)       # CPV int_T e / rho^2 dS
    for k in range(3):
        A, B = V[k], V[(k + 1) % 3]
        L = np.linalg.norm(B - A)
        t = (B - A) / L
        nu_e = np.cross(t, n)          # outward in-plane normal of the edge (CCW about n)
        s = 0.5 * (g + 1.0)
        P = A[None, :] + s[:, None] * (B - A)[None, :]
        J -= nu_e * np.sum(0.5 * w * L / np.linalg.norm(P - xi, axis=1))
    # CPV int r_i / rho^2 dS with r = (xi - x)/rho = -e  is  -J_i
    Ir = -J
    c = -(1.0 - 2.0 * nu) / (8.0 * np.pi * (1.0 - nu))
    return c * (Ir[:, None] * n[None, :] - n[:, None] * Ir[None, :])


# ------------------------------------------------------------------ quadrature
TRI4 = ((1 / 3, 1 / 3, 1 / 3, -27 / 48), (0.6, 0.2, 0.2, 25 / 48), (0.2, 0.6, 0.2, 25 / 48),
        (0.2, 0.2, 0.6, 25 / 48))   # the 4-point degree-3 Gauss rule on a triangle (Strang-Fix)


def quadrature(V0, V1, V2, nq=16):
    """quadrature points (n, nq, 3) and weights (n, nq) of every panel: nq = 16 is PAPER.md
    l. 187 (midpoint subdivision into 4 congruent triangles x the 4-point rule), nq = 1 the
    centroid with the panel area."""
    V0, V1, V2 = (np.asarray(v, np.float64) for v in (V0, V1, V2))
    area = 0.5 * np.linalg.norm(np.cross(V1 - V0, V2 - V0), axis=1)
    if nq == 1:
        return ((V0 + V1 + V2) / 3.0)[:, None, :], area[:, None]
    M01, M12, M20 = (V0 + V1) / 2, (V1 + V2) / 2, (V2 + V0) / 2
    pts, wts = [], []
    for A, B, C in ((V0, M01, M20), (M01, V1, M12), (M20, M12, V2), (M01, M12, M20)):
        for l1, l2, l3, w in TRI4:
            pts.append(l1 * A + l2 * B + l3 * C)
            wts.append(w * area / 4.0)
    return np.stack(pts, 1), np.stack(wts, 1)


# ------------------------------------------------------------------ dense system
def assemble(cent, nrm, area, V0, V1, V2, K, G, nq=16):
    """dense matrices Umat, Pmat (3n x 3n) of Eq. (num): Pmat includes 1/2 I + P_self,
    Umat includes U_self; off-diagonal blocks by the nq-point panel rule."""
    nu = KN.poisson_ratio(K, G)
    cent = np.asarray(cent, np.float64)
    nrm = np.asarray(nrm, np.float64)
    n = cent.shape[0]
    qp, qw = quadrature(V0, V1, V2, nq)
    X = cent[:, None, :]
    off = ~np.eye(n, dtype=bool)
    Ub = np.zeros((n, n, 3, 3))
    Pb = np.zeros((n, n, 3, 3))
    for q in range(qp.shape[1]):
        Y = qp[None, :, q, :]
        Ys = np.where(off[..., None], Y, X + 1.0)
        wq = (qw[None, :, q] * off)[..., None, None]
        Ub += KN.kernel_U(X, Ys, G, nu) * wq
        Pb += KN.kernel_P(X, Ys, nrm[None, :, :], nu) * wq
    for i in range(n):
        V = np.stack([V0[i], V1[i], V2[i]]).astype(np.float64)
        Ub[i, i] = self_U_polar(V, G, nu)
        Pb[i, i] = 0.5 * np.eye(3) + self_P_cpv(V, nu)
    Umat = Ub.transpose(0, 2, 1, 3).reshape(3 * n, 3 * n)
    Pmat = Pb.transpose(0, 2, 1, 3).reshape(3 * n, 3 * n)
    return Umat, Pmat


def mixed_system(Umat, Pmat, bc_type, bc_val):
    """A x = b of Eq. (num2): Pmat u = Umat p with u known on Dirichlet panels (bc_type 0),
    p known on Neumann panels (bc_type 1).  x holds p on Dirichlet, u on Neumann panels."""
    n = len(bc_type)
    dir_ = np.repeat(np.asarray(bc_type) == 0, 3)
    val = np.asarray(bc_val, np.float64).reshape(-1)
    # columns: unknown p (Dirichlet) enters as -Umat, unknown u (Neumann) as +Pmat
    A = np.where(dir_[None, :], -Umat, Pmat)
    b = np.where(dir_, 0.0, 0.0)
    known = np.where(dir_[None, :], Pmat, -Umat)      # moved to the right-hand side
    b = -known @ val
    return A, b


# ------------------------------------------------------------------ GMRES (Saad)
def gmres(matvec, b, x0=None, restart=50, tol=1e-6, max_iter=1000):
    """restarted GMRES(m), Saad Alg. 6.9 / 6.11: Arnoldi with modified Gram-Schmidt, Givens
    rotations on the Hessenberg matrix, stop when |r| / |b| <= tol.
    Returns (x, iterations, relative residual history)."""
    b = np.asarray(b, np.float64)
    n = b.shape[0]
    x = np.zeros(n) if x0 is None else np.asarray(x0, np.float64).copy()
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return np.zeros(n), 0, [0.0]
    hist = []
    it = 0
    while it < max_iter:
        r = b - matvec(x)
        beta = np.linalg.norm(r)
        hist.append(beta / bn)
        if beta / bn <= tol:
            break
        m = restart
        Vb = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        Vb[0] = r / beta
        k_done = 0
        for j in range(m):
            w = matvec(Vb[j])
            for i in range(j + 1):
                H[i, j] = np.dot(w, Vb[i])
                w = w - H[i, j] * Vb[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] > 0:
                Vb[j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            it += 1
            k_done = j + 1
            hist.append(abs(g[j + 1]) / bn)
            if abs(g[j + 1]) / bn <= tol or it >= max_iter:
                break
        y = np.linalg.solve(np.triu(H[:k_done, :k_done]), g[:k_done])
        x = x + Vb[:k_done].T @ y
        if hist[-1] <= tol:
            break
    return x, it, hist
