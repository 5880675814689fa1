/*
 * elastobem.h -- C ABI of the B200-native elastostatic BEM / KIFMM hot path.
 *
 * What it computes (PAPER.md = arXiv:1612.04082 as extracted, line numbers cited):
 *   the sums of Eq. fmm_summation (line 154)
 *       t_i = sum_j w_j K(x_i, y_j, n_j) s_j
 *   for the four fundamental solutions of Sec. 2.1 -- U (Eq. disp_1, line 94),
 *   P (Eq. disp_2, line 98), D (Eq. stress_2), S (Eq. stress_3)
 *   -- by direct summation or by the kernel-independent FMM of Sec. 2.2 (lines
 *   131-151), and the GMRES solve of the collocation system Eq. num2 (line 175) whose
 *   matrix-vector products that FMM supplies (lines 181-189).
 *   Readings of garbled passages (signs/prefactors of P, D, S) are R1-R3 in DESIGN.md.
 *
 * Conventions shared by every entry point
 *   - Points, normals, densities are float32, 3 per item, packed xyzxyz... (AoS).
 *   - A target is where a value is wanted (the paper's collocation point xi or
 *     interior point p); a source is an integration point y_j with outward unit
 *     normal n_j and weight w_j (panel area x quadrature weight).
 *     r-vector = target - source (reading R1).
 *   - f_j: single-layer density (traction-like, PAPER.md p_j in Eq. BIE), used by U/D.
 *     g_j: double-layer density (displacement-like, u_j in Eq. BIE), used by P/S.
 *   - Displacement outputs are 3 floats per target; stress outputs 6 floats per
 *     target in Voigt order (xx, yy, zz, xy, yz, xz).
 *   - Pairs with r == 0 are excluded (the own panel's singular
 *     contribution is the job of the local pass, not of the sum).
 *   - Empty inputs: nsrc = 0 gives zero outputs, ntrg = 0 writes nothing; a tree
 *     needs nsrc + ntrg >= 1 (either may be 0).  Coincident points are allowed: the
 *     tree stops refining at level 20 and such a leaf may exceed max_pts.
 *   - Material: bulk modulus K > 0 and shear modulus G > 0 (PAPER.md Eq. elast,
 *     line 37); the kernels use nu = (3K - 2G) / (2 (3K + G)).
 *   - Memory: unless stated otherwise, array arguments of one call must be either
 *     all device pointers (the call is asynchronous on `stream`) or all host pointers
 *     (the call stages them through device memory and returns after completion); a
 *     call that mixes the two kinds returns EBEM_ERR_ARG before touching any array.
 *     The library never takes ownership of caller arrays.
 *   - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Errors: every int-returning call returns 0 on success and a negative code on
 *     failure; ebem_last_error() gives a thread-local message.  On failure outputs
 *     are unspecified.  No call ever falls back to a CPU computation.
 */
#ifndef ELASTOBEM_H
#define ELASTOBEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* kernel identifiers */
enum ebem_kernel {
    EBEM_U = 0,   /* single layer, displacement out:      sum w U f           */
    EBEM_P = 1,   /* double layer, displacement out:      sum w P g           */
    EBEM_UP = 2,  /* both layers, displacement out:       sum w (U f + P g)   */
    EBEM_D = 3,   /* single layer, stress out:            sum w D f           */
    EBEM_S = 4,   /* double layer, stress out:            sum w S g           */
    EBEM_DS = 5   /* both layers, stress out:             sum w (D f + S g)   */
};

enum ebem_status {
    EBEM_OK = 0,
    EBEM_ERR_ARG = -1,      /* invalid argument                          */
    EBEM_ERR_CUDA = -2,     /* CUDA runtime error (message has details)  */
    EBEM_ERR_STATE = -3,    /* invalid handle / state                    */
    EBEM_ERR_NOCONV = -4    /* GMRES did not reach the tolerance          */
};

/* thread-local description of the last failure ("" if none) */
const char *ebem_last_error(void);

/*
 * bem_kernel_direct -- O(N^2) evaluation of Eq. fmm_summation (
 * "an iterative solution scheme would require O(N^2) operations", line 125).
 *   kernel   one of enum ebem_kernel
 *   trg      [ntrg*3]  target points
 *   src      [nsrc*3]  source points
 *   nrm      [nsrc*3]  unit normals at the sources (required iff the kernel has a
 *                      double layer: P, UP, S, DS; else may be NULL)
 *   w        [nsrc]    weights (NULL = all 1)
 *   f        [nsrc*3]  single-layer density (required iff U, UP, D, DS)
 *   g        [nsrc*3]  double-layer density (required iff P, UP, S, DS)
 *   out      [ntrg*3] (U, P, UP) or [ntrg*6] (D, S, DS), overwritten
 * fp32 arithmetic (FFMA + rsqrt), one pass over all pairs.
 */
int bem_kernel_direct(int kernel, const float *trg, int64_t ntrg, const float *src,
                      const float *nrm, const float *w, const float *f, const float *g,
                      int64_t nsrc, double K, double G, float *out, void *stream);

/* opaque FMM tree + plan: geometry, octree, interaction lists, translation operators */
typedef struct ebem_tree ebem_tree;

/*
 * fmm_build_tree -- build the octree of PAPER.md Sec. 2.2 ("Generation of an octree
 * partitioning of the domain into boxes", line 135) on the device: Morton codes of
 * sources U targets, radix sort, level-by-level adaptive refinement (a box splits iff
 * it holds more than max_pts sources or more than max_pts targets; reading R5),
 * the U/V/W/X interaction lists, and the KIFMM translation operators for multipole
 * order p (surface grid of p points per cube edge, 6(p-1)^2+2 points; reading R6).
 *   src/nrm/w [nsrc*3]/[nsrc*3]/[nsrc]  sources, normals (NULL allowed if only
 *             single-layer kernels will be used), weights (NULL = 1)
 *   trg       [ntrg*3] targets (may alias src)
 *   max_pts   leaf capacity (>= 1), p in [3, 12], K, G material
 *   *tree     receives the handle (free with fmm_tree_free)
 * The tree copies what it needs; caller arrays may be released afterwards.
 * Synchronises `stream` (output sizes are data dependent).
 */
int fmm_build_tree(const float *src, const float *nrm, const float *w, int64_t nsrc,
                   const float *trg, int64_t ntrg, int max_pts, int p, double K, double G,
                   ebem_tree **tree, void *stream);

/*
 * fmm_matvec -- KIFMM evaluation of Eq. fmm_summation with displacement output
 * (kernel U, P or UP): upward pass (S2M, M2M), downward pass (M2L, S2L, L2L),
 * leaf evaluation (L2T, M2T) and near field (P2P over the U list); PAPER.md
 * lines 131-151.  f/g [nsrc*3] in the caller's source order (NULL where unused),
 * out [ntrg*3] in the caller's target order, overwritten.
 * Device pointers: asynchronous, no allocation, capturable in a CUDA graph.
 */
int fmm_matvec(ebem_tree *tree, int kernel, const float *f, const float *g, float *out,
               void *stream);

/*
 * fmm_eval_stress -- the same FMM with stress output (kernel D, S or DS): PAPER.md
 * Eq. stress_1 (line 104) evaluated "via fast summation of the kernels" (line 194).
 * out [ntrg*6], Voigt order.  Returns sum w (D f + S g); the caller applies the signs
 * of Eq. stress_1 (sigma = sum D t - sum S u).
 */
int fmm_eval_stress(ebem_tree *tree, int kernel, const float *f, const float *g, float *out,
                    void *stream);

int fmm_tree_free(ebem_tree *tree);

/*
 * Native phase profiler.  fmm_set_profiling(tree, mode): 0 off; 1 "solo" -- every later
 * evaluation runs its phases one after another on the caller's stream, each bracketed by
 * CUDA events; 2 "in situ" -- the normal overlapped two-stream schedule, each phase
 * bracketed by CUDA events on the (internal) stream it is launched on, so a phase's time
 * includes the slowdown from whatever runs beside it.  Switching the mode resets the record.
 * fmm_phase_stats fills up to `cap` entries (returns the number of phases) with, per phase
 * and for the given kernel id: kernel launches per evaluation, ALGORITHMIC work per
 * evaluation (flops: pair interactions x flops per interaction of the kernel as written in
 * elastic.cuh, or 2 M K per GEMM column; bytes: operands read once + results written
 * once), its arithmetic precision and the MEAN device time over the evaluations profiled
 * since the mode was set (at most the last 64; ms, -1 if none; synchronises the device).
 * Phases: prep, S2M, Q2Z_up, M2M, S2L, Q2Z_dn, M2L, L2L, PHI, NEAR, FAR (near field:
 * U list and the directly summed X/W/V entries; far field: L2T + M2T and the scatter).
 * Returns EBEM_ERR_ARG for a mode outside 0..2.
 */
typedef struct ebem_phase_stat {
    char name[16];
    int32_t launches;
    int32_t fp64;          /* 1 if the phase computes (partly) in fp64 */
    double flops;          /* algorithmic floating-point operations per evaluation */
    double flops_fp64;     /* the part of `flops` computed in fp64 */
    double interactions;   /* kernel pair evaluations per evaluation (0 for GEMM phases) */
    double bytes;          /* algorithmic DRAM bytes per evaluation */
    double ms;             /* device time of the last profiled evaluation */
} ebem_phase_stat;

int fmm_set_profiling(ebem_tree *tree, int on);
int fmm_phase_stats(ebem_tree *tree, int kernel, ebem_phase_stat *out, int cap);

/* number of CUDA kernel launches issued by this library since it was loaded */
int64_t ebem_launch_count(void);

/*
 * Device memory the library keeps: released long-lived buffers of >= 1 MB (tree workspace,
 * operators) stay cached for reuse by the next tree or solve of the same sizes, up to
 * EBEM_CACHE_MB (environment, default 16384) MB in total; an allocation that fails returns
 * the cache to the driver and retries.  ebem_trim_cache returns every cached block to the
 * driver now (for a caller that needs the memory elsewhere) and reports the bytes freed.
 */
int64_t ebem_trim_cache(void);

typedef struct ebem_tree_info {
    int64_t nsrc, ntrg, nboxes, nleaves;
    int32_t nlevels, p, max_pts, n_equiv;   /* n_equiv = 6(p-1)^2+2 surface points */
    int64_t n_u, n_v, n_w, n_x;             /* total entries of each interaction list */
    double origin[3], side;                 /* root cube */
    int64_t device_bytes;                   /* device memory held by the handle */
} ebem_tree_info;

int fmm_tree_info(const ebem_tree *tree, ebem_tree_info *info);

/*
 * fmm_tree_export -- copy one tree array to HOST memory (parity tests).
 *   what: 0 point Morton keys in sorted order   int64[nsrc+ntrg]
 *         1 sorted position -> original point index (sources 0..nsrc-1, then
 *           targets nsrc..)                      int32[nsrc+ntrg]
 *         2 box level                            int32[nboxes]
 *         3 box anchor (ix,iy,iz)                int32[nboxes*3]
 *         4 box parent (-1 root)                 int32[nboxes]
 *         5 box point range [begin,end)          int32[nboxes*2]
 *         6..9 list U,V,W,X offsets (CSR)        int32[nboxes+1]
 *         10..13 list U,V,W,X entries            int32[n_list]
 *   buf/cap: destination and its capacity in bytes.  Returns bytes written (>= 0)
 *   or a negative error.
 */
int64_t fmm_tree_export(const ebem_tree *tree, int what, void *buf, int64_t cap);

/*
 * Collocation BEM operator of PAPER.md Eqs. (num), (coef), (num2) (l. 159-191): piecewise-
 * constant displacement u and traction p on flat triangles, collocation at centroids,
 * off-diagonal panel integrals by the panels' quadrature points as FMM sources ("Each
 * triangular element contains 16 quadrature points", l. 187; nq = 1: centroid rule), and
 * the "second, local, pass" (l. 189): own-panel quadrature contributions replaced by the
 * singular integrals ("evaluated analytically", l. 179) and the free term 1/2 I.
 *
 * bem_create -- vertices [npanels*9]: v0, v1, v2 (xyz each) per flat triangle, ordered
 *   counter-clockwise seen from outside the material (outward normal by the right-hand
 *   rule); nq in {1, 16}; max_pts, p: FMM leaf size and order; K, G material.
 *   Builds quadrature points, the FMM tree over them (targets = centroids), and the local
 *   3x3 correction blocks.  Synchronises `stream`.
 * bem_apply  -- y = A x for the mixed BVP with per-panel bc_type (0 = displacement
 *   prescribed / traction unknown, 1 = traction prescribed / displacement unknown);
 *   x, y [npanels*3].
 * bem_rhs    -- b = right-hand side of Eq. num2 for prescribed values bc_val [npanels*3].
 * bem_gmres_solve -- restarted GMRES(restart) (Saad) with device-side
 *   Arnoldi (classical Gram-Schmidt + one re-orthogonalisation, fp64 Krylov basis on the
 *   device, Givens rotations on the host), every A v through bem_apply (one KIFMM matvec).
 *   x [npanels*3]: initial guess in, solution out (traction on Dirichlet panels,
 *   displacement on Neumann panels).  Stops at |b - A x| / |b| <= tol or max_iter;
 *   returns EBEM_ERR_NOCONV (x still written) if the tolerance was not reached.
 *   precond: 0 = none (the paper's solver, l. 181, "In the future this shortcoming should be
 *   addressed with ... the appropriate preconditioner", l. 369); 1 = block-Jacobi right
 *   preconditioner with the panels' own 3x3 blocks (-U_self on Dirichlet panels,
 *   1/2 I + P_self on Neumann panels); 2 = leaf-block Jacobi right preconditioner: the
 *   diagonal blocks of A over the panels whose collocation points share an octree leaf (at
 *   most 52 panels per block), formed in fp64 as the operator applies them and inverted
 *   once per solve (they may take up to half of the free device memory; precond 1 is used
 *   when they do not fit).  The solution of A x = b is the same; any other value is
 *   EBEM_ERR_ARG.
 *   iters_out / resid_out (host, may be NULL): iterations and final relative residual.
 *   restart in [1, 63] (EBEM_ERR_ARG otherwise): the Krylov basis is (restart + 1) fp64
 *   vectors of npanels*3 on the device.
 *   Inside the solve the operator is the same map re-associated for the B200 (results equal
 *   to fp32 rounding): the near field is held in device memory as one 3x3 block per target
 *   and near panel (built at the first solve, rebuilt when bc_type changes, kept by the
 *   handle until bem_free; it may take up to 60% of the free device memory, and the
 *   pair-kernel near field is used when it does not fit), and the sources of every leaf are
 *   grouped by the bc_type of their panel (a permutation inside each leaf).  The handle must
 *   not be used from two streams at once.
 * Array arguments of bem_apply / bem_rhs / bem_gmres_solve must be device pointers
 * (EBEM_ERR_ARG otherwise, checked for every array argument).
 */
typedef struct ebem_bem ebem_bem;

int bem_create(const float *vertices, int64_t npanels, int nq, int max_pts, int p, double K,
               double G, ebem_bem **bem, void *stream);
int bem_apply(ebem_bem *bem, const int32_t *bc_type, const float *x, float *y, void *stream);
int bem_rhs(ebem_bem *bem, const int32_t *bc_type, const float *bc_val, float *b, void *stream);
int bem_gmres_solve(ebem_bem *bem, const int32_t *bc_type, const float *bc_val, float *x,
                    int restart, int max_iter, double tol, int precond, int32_t *iters_out,
                    double *resid_out, void *stream);
/*
 * bem_gmres_history -- residual history of the last bem_gmres_solve on this handle (host).
 *   what 0: the Arnoldi estimate |g_{j+1}| / |b| after every iteration (one entry per
 *           iteration: the GMRES least-squares residual);
 *   what 1: the true relative residual |b - A x| / |b| at the start of every restart cycle
 *           and after the last one (computed by one extra operator application).
 *   The gap between the two measures the inexactness of the fp32 operator (R12).
 *   Copies min(n, cap) doubles to buf and returns n (>= 0), or a negative error.
 */
int bem_gmres_history(const ebem_bem *bem, int what, double *buf, int cap);
int bem_free(ebem_bem *bem);

#ifdef __cplusplus
}
#endif
#endif /* ELASTOBEM_H */
