"""Oracle: kernel-independent FMM (reference tree code), fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the product path.

Follows PAPER.md Sec. 2.2, "Kernel-independent fast multipole method" (lines 131-151),
step by step and in the paper's order:

  1. "Generation of an octree partitioning of the domain into boxes"   -> oracle.tree
  2. "Fine-to-coarse tree traversal to compute compact representations of the
     far-field potential of a box ... combining expansions of descendant boxes ...
     using linear M2M translation operators"                          -> upward()
  3. "a coarse-to-fine pass, that computes local expansions for each box ...
     obtained ... by combining the parent's local expansion (using an L2L operator)
     with multipole expansions of boxes that are not in the far zone of the parent,
     but are in the far zones of the descendants. Multipole expansions are converted
     to local using M2L operators"                                     -> downward()
  4. "At the finest level of the tree, the complete integrals are computed by adding
     the contributions of points in the near zone using direct summation" -> evaluate()

  "it represents the far-field (multipole) and local approximations of the integrals
  with a density phi defined at samples x_i of an equivalent surface, so that the
  approximation at a point y has the form sum_i phi_i K(x_i, y)" (line 147), and
  "The M2M, L2L and M2L operators ... are represented by matrices mapping density
  values on different equivalent surfaces to each other, and are computed
  automatically for each needed kernel" (line 149).

Reading R6 fixes what the paper leaves to its references:
  * surfaces: the boundary of the cube [-1,1]^3 sampled on a p x p x p grid
    (6 (p-1)^2 + 2 points; "multipole order p"), scaled by the box half-width r and
    radius factors  upward-equivalent 1.05, upward-check 2.95, downward-equivalent
    2.95, downward-check 1.05;
  * equivalent densities are single-layer (kernel U) 3-vectors for every source kernel
    (the field of double-layer sources outside a surface is a single-layer field);
    targets asking for stress read them through D;
  * check surfaces are sampled one point per edge finer than the equivalent
    surfaces (p+1 per edge), and the check-to-equivalent solve is the Tikhonov-
    regularised least-squares pseudo-inverse  V diag(s/(s^2 + a^2)) U^T,
    a = rcond * s_max, rcond = max(1e-9, 10^-(p+1)) by default;
  * the X list (S2L) and W list (M2T) of the adaptive KIFMM complete the far field.
"""
from __future__ import annotations

import numpy as np

from . import kernels as KN
from . import tree as TR

RAD_UE, RAD_UC, RAD_DE, RAD_DC = 1.05, 2.95, 2.95, 1.05


def surface_grid(p: int) -> np.ndarray:
    """points of the p^3 grid on [-1,1]^3 that lie on the cube boundary, lexicographic
    (i slowest); 6 (p-1)^2 + 2 of them."""
    t = np.linspace(-1.0, 1.0, p)
    out = []
    for i in range(p):
        for j in range(p):
            for k in range(p):
                if i in (0, p - 1) or j in (0, p - 1) or k in (0, p - 1):
                    out.append((t[i], t[j], t[k]))
    return np.array(out)


def U_matrix(X, Y, G, nu):
    """dense (3 nx, 3 ny) matrix of kernel U: rows (target i, component a),
    columns (source j, component b)."""
    M = KN.kernel_U(X[:, None, :], Y[None, :, :], G, nu)       # (nx, ny, 3, 3)
    return M.transpose(0, 2, 1, 3).reshape(3 * X.shape[0], 3 * Y.shape[0])


def pinv(A, rcond):
    """Tikhonov-regularised pseudo-inverse  argmin |A x - b|^2 + a^2 |x|^2,  a = rcond s_max."""
    u, s, vt = np.linalg.svd(A, full_matrices=False)
    a = rcond * s[0]
    return (vt.T * (s / (s * s + a * a))) @ u.T


def default_rcond(p: int) -> float:
    return max(1e-9, 10.0 ** (-(p + 1)))


class KIFMM:
    def __init__(self, src, trg, K, G, p=6, max_pts=64, nrm=None, rcond=None, pc=None):
        self.src = np.asarray(src, np.float64).reshape(-1, 3)
        self.trg = np.asarray(trg, np.float64).reshape(-1, 3)
        self.nrm = None if nrm is None else np.asarray(nrm, np.float64).reshape(-1, 3)
        self.K, self.G = K, G
        self.nu = KN.poisson_ratio(K, G)
        self.p = p
        self.T = TR.build_tree(self.src, self.trg, max_pts)
        self.L = TR.build_lists(self.T)
        rcond = default_rcond(p) if rcond is None else rcond
        self.s = surface_grid(p)                          # equivalent surfaces
        self.sc = surface_grid(p + 1 if pc is None else pc)   # check surfaces
        # check -> equivalent solves at unit half-width; at half-width r the kernel
        # matrix is U/r (U is homogeneous of degree -1), so the solve is r * pinv.
        self.uc2ue = pinv(U_matrix(RAD_UC * self.sc, RAD_UE * self.s, G, self.nu), rcond)
        self.dc2de = pinv(U_matrix(RAD_DC * self.sc, RAD_DE * self.s, G, self.nu), rcond)
        self.side = self.T.side
        self._cache = {}

    # ---------------------------------------------------------------- helpers
    def surf(self, b, rad):
        return self.T.center(b) + rad * self.T.half_width(b) * self.s

    def csurf(self, b, rad):
        return self.T.center(b) + rad * self.T.half_width(b) * self.sc

    def trans(self, b, rad_b, a, rad_a):
        """U_matrix(csurf(b, rad_b), surf(a, rad_a)).  It depends only on the two box
        levels, their relative anchor position and the radii, so it is memoised on those
        (evaluated in coordinates relative to box a's centre)."""
        T = self.T
        la, lb = int(T.level[a]), int(T.level[b])
        L = max(la, lb)
        off = T.anchor[b] * (1 << (L - lb)) * 2 + (1 << (L - lb)) - (T.anchor[a] * (1 << (L - la)) * 2 + (1 << (L - la)))
        key = (la, lb, tuple(int(v) for v in off), rad_b, rad_a)
        M = self._cache.get(key)
        if M is None:
            unit = self.side / 2.0 ** (L + 1)          # half-width at the finer level
            X = off * unit + rad_b * T.half_width(b) * self.sc
            Y = rad_a * T.half_width(a) * self.s
            M = U_matrix(X, Y, self.G, self.nu)
            self._cache[key] = M
        return M

    def _src_sum(self, kernel, X, b, dens):
        """direct sum from the sources of box b to the points X (displacement kernels)."""
        T = self.T
        idx = T.src_perm[T.src_begin[b]:T.src_end[b]]
        if idx.size == 0:
            return np.zeros((X.shape[0], 3))
        f = None if dens["f"] is None else dens["f"][idx]
        g = None if dens["g"] is None else dens["g"][idx]
        nrm = None if self.nrm is None else self.nrm[idx]
        return KN.direct_sum(kernel, X, self.src[idx], self.K, self.G, w=dens["w"][idx], f=f, g=g, nrm=nrm)

    def _equiv_eval(self, Y, phi, X, stress):
        """potential (or stress) at X of the single-layer density phi on the points Y."""
        kern = KN.KERNEL_D if stress else KN.KERNEL_U
        return KN.direct_sum(kern, X, Y, self.K, self.G, f=phi.reshape(-1, 3))

    # ---------------------------------------------------------------- passes
    def upward(self, kernel, dens):
        """fine-to-coarse: phi_u of every box (multipole equivalent densities)."""
        T = self.T
        phi = np.zeros((T.nboxes, 3 * self.s.shape[0]))
        for b in range(T.nboxes - 1, -1, -1):          # children have larger ids than parents
            r = T.half_width(b)
            xc = self.csurf(b, RAD_UC)
            if T.leaf[b]:
                q = self._src_sum(kernel, xc, b, dens).reshape(-1)           # S2M check potential
            else:
                q = np.zeros(3 * xc.shape[0])
                for c in T.child[b]:
                    if c >= 0:                                               # M2M
                        q += self.trans(b, RAD_UC, c, RAD_UE) @ phi[c]
            phi[b] = r * (self.uc2ue @ q)
        return phi

    def downward(self, kernel, dens, phi_u):
        """coarse-to-fine: phi_d of every box (local equivalent densities)."""
        T = self.T
        phi = np.zeros_like(phi_u)
        for b in range(T.nboxes):                        # parents before children
            if T.level[b] < 2:
                continue
            r = T.half_width(b)
            xc = self.csurf(b, RAD_DC)
            q = np.zeros(3 * xc.shape[0])
            for a in self.L["V"][b]:                     # M2L
                q += self.trans(b, RAD_DC, a, RAD_UE) @ phi_u[a]
            for a in self.L["X"][b]:                     # S2L
                q += self._src_sum(kernel, xc, a, dens).reshape(-1)
            par = T.parent[b]
            if T.level[par] >= 2:                        # L2L
                q += self.trans(b, RAD_DC, par, RAD_DE) @ phi[par]
            phi[b] = r * (self.dc2de @ q)
        return phi

    def evaluate(self, kernel, w=None, f=None, g=None):
        """t(x_i) = sum_j w_j K(x_i, y_j) s_j for every target (Eq. fmm_summation).
        kernel in {U, P, UP} -> (ntrg, 3); {D, S, DS} -> (ntrg, 6) Voigt."""
        stress = kernel in (KN.KERNEL_D, KN.KERNEL_S, KN.KERNEL_DS)
        src_kernel = {KN.KERNEL_D: KN.KERNEL_U, KN.KERNEL_S: KN.KERNEL_P,
                      KN.KERNEL_DS: KN.KERNEL_UP}.get(kernel, kernel)
        ns = self.src.shape[0]
        dens = dict(w=np.ones(ns) if w is None else np.asarray(w, np.float64).reshape(ns),
                    f=None if f is None else np.asarray(f, np.float64).reshape(ns, 3),
                    g=None if g is None else np.asarray(g, np.float64).reshape(ns, 3))
        phi_u = self.upward(src_kernel, dens)
        phi_d = self.downward(src_kernel, dens, phi_u)
        T = self.T
        out = np.zeros((self.trg.shape[0], 6 if stress else 3))
        for b in np.nonzero(T.leaf)[0]:
            tidx = T.trg_perm[T.trg_begin[b]:T.trg_end[b]]
            if tidx.size == 0:
                continue
            X = self.trg[tidx]
            acc = np.zeros((X.shape[0], out.shape[1]))
            if T.level[b] >= 2:                                            # L2T
                acc += self._equiv_eval(self.surf(b, RAD_DE), phi_d[b], X, stress)
            for a in self.L["W"][b]:                                       # M2T
                acc += self._equiv_eval(self.surf(a, RAD_UE), phi_u[a], X, stress)
            for a in self.L["U"][b]:                                       # near field
                idx = T.src_perm[T.src_begin[a]:T.src_end[a]]
                if idx.size == 0:
                    continue
                acc += KN.direct_sum(kernel, X, self.src[idx], self.K, self.G, w=dens["w"][idx],
                                     f=None if dens["f"] is None else dens["f"][idx],
                                     g=None if dens["g"] is None else dens["g"][idx],
                                     nrm=None if self.nrm is None else self.nrm[idx])
            out[tidx] = acc
        return out
