"""Oracle: the four elastostatic fundamental solutions and their O(N^2) direct sum.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product path.

All arithmetic is fp64 numpy, written term by term from PAPER.md Sec. 2.1.

Notation.  A *target* is the point where a value is
wanted (the paper's collocation point xi, or interior point p); a *source* is an
integration point x on Gamma with outward unit normal n.  Throughout

    d = target - source,   r = |d|,   rh = d / r      (the paper's r_{,i})

Reading R1: the paper writes r_{,i} without fixing the
direction.  Taking r_{,i} = (xi_i - x_i)/r (target minus source) makes Eq.
disp_2 exactly the classical Kelvin traction kernel, which is what the BIE Eq.
(BIE) needs: the rigid-translation identity  int_Gamma P_ij dGamma = -delta_ij
for a target inside a closed surface (pinned in tests/test_oracle_kernels.py).

Reading R2: Eq. stress_2 as extracted reads (1-2nu)/(2 pi (1-nu) r^2)(...).  The
constitutive law of Eq. (elast), sigma_ij = C_ijkl eps_kl applied to the
displacement of Eq. disp_1, fixes the prefactor to -1/(8 pi (1-nu) r^2) in the
r_{,i} direction of R1 (pinned by finite differences and by sympy).

Reading R3: Eq. stress_3 as extracted omits the shear modulus G that a
displacement-to-stress kernel must carry; C_ijkl applied to Eq. disp_2 fixes
S_kij = G * (printed expression).  (PAPER.md's examples use G = 1, where the two
agree.)

Material: the paper states the problem with bulk modulus K and shear modulus G
(Eq. elast, line 37) and writes the kernels with G and Poisson's ratio nu;
nu = (3K - 2G) / (2 (3K + G)) (isotropic elasticity identity).
"""
from __future__ import annotations

import numpy as np

PI = np.pi

# kernel identifiers shared (by value, not by code) with include/elastobem.h
KERNEL_U = 0        # single layer, displacement out (Eq. disp_1)
KERNEL_P = 1        # double layer, displacement out (Eq. disp_2)
KERNEL_UP = 2       # U f + P g in one sum
KERNEL_D = 3        # single layer, stress out (Eq. stress_2, reading R2)
KERNEL_S = 4        # double layer, stress out (Eq. stress_3, reading R3)
KERNEL_DS = 5       # D f + S g in one sum

VOIGT = ((0, 0), (1, 1), (2, 2), (0, 1), (1, 2), (0, 2))   # stress output order


def poisson_ratio(K: float, G: float) -> float:
    """nu from bulk and shear moduli (PAPER.md Eq. elast uses K, G; kernels use G, nu)."""
    return (3.0 * K - 2.0 * G) / (2.0 * (3.0 * K + G))


def young_modulus(K: float, G: float) -> float:
    return 9.0 * K * G / (3.0 * K + G)


def stiffness(K: float, G: float) -> np.ndarray:
    """C_ijkl of PAPER.md Eq. (elast), line 43, written out literally."""
    d = np.eye(3)
    C = np.zeros((3, 3, 3, 3))
    for i in range(3):
        for j in range(3):
            for k in range(3):
                for l in range(3):
                    C[i, j, k, l] = (K * d[i, j] * d[k, l]
                                     + G * (d[i, k] * d[j, l] + d[i, l] * d[j, k]
                                            - 2.0 / 3.0 * d[i, j] * d[k, l]))
    return C


def _geom(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    dvec = x - y
    r = np.sqrt(np.sum(dvec * dvec, axis=-1))
    rh = dvec / r[..., None]
    return r, rh


def kernel_U(x, y, G, nu):
    """U_ij(xi, x), PAPER.md Eq. disp_1 (line 94):
    U_ij = ((3 - 4 nu) delta_ij + r_i r_j) / (16 pi (1 - nu) G r).   shape (..., 3, 3)"""
    r, rh = _geom(x, y)
    I = np.eye(3)
    c = 1.0 / (16.0 * PI * (1.0 - nu) * G * r)
    return c[..., None, None] * ((3.0 - 4.0 * nu) * I + rh[..., :, None] * rh[..., None, :])


def kernel_P(x, y, n, nu):
    """P_ij(xi, x), PAPER.md Eq. disp_2 (line 98), reading R1 for r_{,i}:
    P_ij = [dr/dn ((1-2nu) d_ij + 3 r_i r_j) - (1-2nu)(r_i n_j - r_j n_i)] / (8 pi (1-nu) r^2)
    with dr/dn = r_k n_k and n the unit normal at the source.   shape (..., 3, 3)"""
    r, rh = _geom(x, y)
    n = np.broadcast_to(np.asarray(n, dtype=np.float64), rh.shape)
    I = np.eye(3)
    drdn = np.sum(rh * n, axis=-1)
    a = 1.0 - 2.0 * nu
    br = (drdn[..., None, None] * (a * I + 3.0 * rh[..., :, None] * rh[..., None, :])
          - a * (rh[..., :, None] * n[..., None, :] - rh[..., None, :] * n[..., :, None]))
    return br / (8.0 * PI * (1.0 - nu) * r * r)[..., None, None]


def kernel_D(x, y, nu):
    """D_kij(p, x), PAPER.md Eq. stress_2 (line 109) under reading R2:
    D_kij = -[(1-2nu)(d_ki r_j + d_kj r_i - d_ij r_k) + 3 r_i r_j r_k] / (8 pi (1-nu) r^2)
    sigma_ij at the target due to a unit force in direction k at the source.  shape (..., 3, 3, 3)"""
    r, rh = _geom(x, y)
    I = np.eye(3)
    a = 1.0 - 2.0 * nu
    t = (a * (I[:, :, None] * rh[..., None, None, :]          # d_ki r_j
              + I[:, None, :] * rh[..., None, :, None]        # d_kj r_i
              - I[None, :, :] * rh[..., :, None, None])       # d_ij r_k
         + 3.0 * rh[..., None, :, None] * rh[..., None, None, :] * rh[..., :, None, None])
    return -t / (8.0 * PI * (1.0 - nu) * r * r)[..., None, None, None]


def kernel_S(x, y, n, G, nu):
    """S_kij(p, x), PAPER.md Eq. stress_3 (lines 113-116) under reading R3 (factor G):
    S_kij = G/(4 pi (1-nu) r^3) { 3 dr/dn [ (1-2nu) d_ij r_k + nu (d_ki r_j + d_kj r_i) - 5 r_i r_j r_k ]
            + 3 nu (n_i r_j r_k + n_j r_i r_k) + (1-2nu)(3 n_k r_i r_j + n_j d_ki + n_i d_kj)
            - (1-4nu) n_k d_ij }
    which is the paper's bracket with (3-6nu) = 3(1-2nu) and (1-2nu) multiplied through.
    shape (..., 3, 3, 3), index order [k, i, j]."""
    r, rh = _geom(x, y)
    n = np.broadcast_to(np.asarray(n, dtype=np.float64), rh.shape)
    I = np.eye(3)
    drdn = np.sum(rh * n, axis=-1)
    a = 1.0 - 2.0 * nu
    rk = rh[..., :, None, None]
    ri = rh[..., None, :, None]
    rj = rh[..., None, None, :]
    nk = n[..., :, None, None]
    ni = n[..., None, :, None]
    nj = n[..., None, None, :]
    dki = I[:, :, None]
    dkj = I[:, None, :]
    dij = I[None, :, :]
    t1 = 3.0 * drdn[..., None, None, None] * (a * dij * rk + nu * (dki * rj + dkj * ri) - 5.0 * ri * rj * rk)
    t2 = 3.0 * nu * (ni * rj * rk + nj * ri * rk)
    t3 = a * (3.0 * nk * ri * rj + nj * dki + ni * dkj)
    t4 = -(1.0 - 4.0 * nu) * nk * dij
    return (G / (4.0 * PI * (1.0 - nu) * r ** 3))[..., None, None, None] * (t1 + t2 + t3 + t4)


def direct_sum(kernel, trg, src, K, G, w=None, f=None, g=None, nrm=None, chunk=64, schunk=4096):
    """O(N^2) evaluation of PAPER.md Eq. fmm_summation (line 154),
        t_i = sum_j w_j K(x_i, y_j, n_j) s_j,
    for kernel in {U, P, UP, D, S, DS}.  f is the single-layer density (traction-like,
    used with U/D), g the double-layer density (displacement-like, used with P/S);
    w the panel weights (1 if None).  Pairs with r == 0 are skipped (self-interaction
    exclusion: the own-panel contribution is handled separately).
    Returns (ntrg, 3) for U/P/UP, (ntrg, 6) Voigt (xx,yy,zz,xy,yz,xz) for D/S/DS."""
    trg = np.asarray(trg, np.float64).reshape(-1, 3)
    src = np.asarray(src, np.float64).reshape(-1, 3)
    ns = src.shape[0]
    nu = poisson_ratio(K, G)
    w = np.ones(ns) if w is None else np.asarray(w, np.float64).reshape(ns)
    use_sl = kernel in (KERNEL_U, KERNEL_UP, KERNEL_D, KERNEL_DS)
    use_dl = kernel in (KERNEL_P, KERNEL_UP, KERNEL_S, KERNEL_DS)
    stress = kernel in (KERNEL_D, KERNEL_S, KERNEL_DS)
    if use_sl:
        fw = np.asarray(f, np.float64).reshape(ns, 3) * w[:, None]
    if use_dl:
        gw = np.asarray(g, np.float64).reshape(ns, 3) * w[:, None]
        nrm = np.asarray(nrm, np.float64).reshape(ns, 3)
    out = np.zeros((trg.shape[0], 6 if stress else 3))
    for t0 in range(0, trg.shape[0], chunk):
        x = trg[t0:t0 + chunk, None, :]
        acc = np.zeros((x.shape[0], 3)) if not stress else np.zeros((x.shape[0], 3, 3))
        for s0 in range(0, ns, schunk):
            sl = slice(s0, s0 + schunk)
            dd = x - src[None, sl, :]
            self_pair = np.all(dd == 0.0, axis=-1)
            # move coincident sources away so the kernel stays finite; their terms are zeroed
            ys = np.where(self_pair[..., None], x + 1.0, src[None, sl, :])
            mask = (~self_pair).astype(np.float64)
            if not stress:
                if use_sl:
                    acc += np.einsum('tsij,sj,ts->ti', kernel_U(x, ys, G, nu), fw[sl], mask)
                if use_dl:
                    acc += np.einsum('tsij,sj,ts->ti', kernel_P(x, ys, nrm[None, sl, :], nu), gw[sl], mask)
            else:
                if use_sl:
                    acc += np.einsum('tskij,sk,ts->tij', kernel_D(x, ys, nu), fw[sl], mask)
                if use_dl:
                    acc += np.einsum('tskij,sk,ts->tij', kernel_S(x, ys, nrm[None, sl, :], G, nu), gw[sl], mask)
        if stress:
            acc = np.stack([acc[:, a, b] for a, b in VOIGT], axis=-1)
        out[t0:t0 + chunk] = acc
    return out


def rel_l2(a, b):
    """relative L2 error ||a - b|| / ||b|| (the north-star metric)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
