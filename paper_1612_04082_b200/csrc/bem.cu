// Collocation BEM operator and restarted GMRES with device-side Arnoldi
// (Sec. 2.2, "Discretization of BIE" and "Matrix-vector products", l. 159-191).
//
// Row i of Eq. (num) (piecewise-constant u, p on flat triangles, collocation at centroids):
//   (1/2 I + P_self_i) u_i + sum_{j} sum_{q in j, y_q != xi_i} w_q P(xi_i, y_q) u_j
//       = U_self_i p_i + sum_{j} sum_{q in j, y_q != xi_i} w_q U(xi_i, y_q) p_j
// The double sum is one KIFMM evaluation with the panels' quadrature points as sources
// (l. 186-187: 16 points per triangle; or the centroid rule, reading R9) and the centroids
// as targets.  The "second, local, pass" (l. 189) subtracts the own panel's quadrature
// contributions and adds the singular integrals: per panel two 3x3 blocks
//   CU_i = U_self_i - sum_{q in i} w_q U(xi_i, y_q),
//   CP_i = 1/2 I + P_self_i - sum_{q in i} w_q P(xi_i, y_q),
// with U_self (weakly singular) and the CPV P_self evaluated in polar coordinates about the
// centroid (radial integral in closed form, angular integral by Gauss-Legendre along the
// edges: "evaluated analytically", l. 179).
// The mixed BVP moves the unknowns (p on Dirichlet panels, u on Neumann panels) to the left:
// A x = b (Eq. num2), applied matrix-free as L(u, p) = P u - U p.
#include <chrono>
#include <cmath>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "bem_near.cuh"
#include "bem_prec.cuh"
#include "fmm.cuh"
#include "p2p.cuh"

namespace ebem {

constexpr int NGL = 32;   // Gauss-Legendre points per edge for the self integrals
__constant__ double c_gl_x[NGL], c_gl_w[NGL];

static void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
    x.resize(n);
    w.resize(n);
    for (int i = 0; i < n; ++i) {
        double z = std::cos(3.14159265358979323846 * (i + 0.75) / (n + 0.5)), pp = 0;
        for (int it = 0; it < 100; ++it) {
            double p1 = 1, p2 = 0;
            for (int k = 1; k <= n; ++k) {
                double p3 = p2;
                p2 = p1;
                p1 = ((2.0 * k - 1.0) * z * p2 - (k - 1.0) * p3) / k;
            }
            pp = n * (z * p1 - p2) / (z * z - 1.0);
            double z1 = z;
            z = z1 - p1 / pp;
            if (std::fabs(z - z1) < 1e-16) break;
        }
        x[i] = z;
        w[i] = 2.0 / ((1.0 - z * z) * pp * pp);
    }
}

struct Bem {
    int64_t n = 0;          // panels
    int nq = 16;
    Material mat{};
    Tree* tree = nullptr;
    DBuf<float> cent, nrm, area, qpts, qnrm, qw;
    DBuf<float> CU, CP;     // [n x 9] local correction blocks (row-major 3x3)
    DBuf<double> DU, DP;    // [n x 9] diagonal blocks U_self, 1/2 I + P_self (preconditioner)
    DBuf<float> f, g, y;    // expanded densities [n nq x 3], FMM output [n x 3]
    DBuf<double> yd;        // FMM output in fp64 (the operator inside GMRES)
    NearMat nm;             // near-field operator of the last solve's boundary conditions
    PanelOp s2m_op, s2l_op; // check-potential operators (S2M of the source leaves, S2L of the X lists)
    // residual history of the last bem_gmres_solve (bem_gmres_history): the Arnoldi estimate
    // |g_{j+1}| / |b| after every iteration, and the true |b - A x| / |b| at every restart
    std::vector<double> hist_est, hist_true;
    ~Bem() { delete tree; }
};

// ------------------------------------------------------------------ geometry
__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

// centroid, unit normal (right-hand rule), area, and the nq quadrature points / weights:
// nq = 16: midpoint subdivision into 4 congruent triangles x the 4-point degree-3 rule
// (barycentric (1/3,1/3,1/3) weight -27/48, (3/5,1/5,1/5) x 3 weight 25/48); the middle
// sub-triangle's centre point is the panel centroid itself and is copied bit-exactly so
// the FMM's r == 0 exclusion removes it.
__global__ void panels_kernel(const float* __restrict__ V, int64_t n, int nq, float* cent, float* nrm, float* area,
                              float* qp, float* qn, float* qw) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v[3][3];
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) v[a][c] = V[9 * i + 3 * a + c];
    double e1[3], e2[3], cr[3];
    for (int c = 0; c < 3; ++c) {
        e1[c] = v[1][c] - v[0][c];
        e2[c] = v[2][c] - v[0][c];
    }
    cross3(e1, e2, cr);
    const double a2 = sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
    float ctr[3], nn[3];
    for (int c = 0; c < 3; ++c) {
        ctr[c] = (float)((v[0][c] + v[1][c] + v[2][c]) / 3.0);
        nn[c] = (float)(cr[c] / a2);
        cent[3 * i + c] = ctr[c];
        nrm[3 * i + c] = nn[c];
    }
    const double A = 0.5 * a2;
    area[i] = (float)A;
    if (nq == 1) {
        for (int c = 0; c < 3; ++c) {
            qp[3 * i + c] = ctr[c];
            qn[3 * i + c] = nn[c];
        }
        qw[i] = (float)A;
        return;
    }
    double m01[3], m12[3], m20[3];
    for (int c = 0; c < 3; ++c) {
        m01[c] = 0.5 * (v[0][c] + v[1][c]);
        m12[c] = 0.5 * (v[1][c] + v[2][c]);
        m20[c] = 0.5 * (v[2][c] + v[0][c]);
    }
    const double* sub[4][3] = {{v[0], m01, m20}, {m01, v[1], m12}, {m20, m12, v[2]}, {m01, m12, m20}};
    const double bary[4][4] = {{1.0 / 3, 1.0 / 3, 1.0 / 3, -27.0 / 48},
                               {0.6, 0.2, 0.2, 25.0 / 48},
                               {0.2, 0.6, 0.2, 25.0 / 48},
                               {0.2, 0.2, 0.6, 25.0 / 48}};
    int q = 0;
    for (int t = 0; t < 4; ++t)
        for (int k = 0; k < 4; ++k, ++q) {
            const int64_t o = i * 16 + q;
            for (int c = 0; c < 3; ++c) {
                const double x = bary[k][0] * sub[t][0][c] + bary[k][1] * sub[t][1][c] + bary[k][2] * sub[t][2][c];
                qp[3 * o + c] = (t == 3 && k == 0) ? ctr[c] : (float)x;
                qn[3 * o + c] = nn[c];
            }
            qw[o] = (float)(bary[k][3] * A / 4.0);
        }
}

// local correction blocks CU, CP (see the file header), fp64
__global__ void self_terms_kernel(const float* __restrict__ V, int64_t n, int nq, const float* __restrict__ qp,
                                  const float* __restrict__ qw, const float* __restrict__ cent,
                                  const float* __restrict__ nrm, double G, double nu, float* CU, float* CP,
                                  double* DU, double* DP) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double PI = 3.14159265358979323846;
    double v[3][3], xi[3], nn[3];
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) v[a][c] = V[9 * i + 3 * a + c];
    for (int c = 0; c < 3; ++c) {
        xi[c] = (v[0][c] + v[1][c] + v[2][c]) / 3.0;
        nn[c] = nrm[3 * i + c];
    }
    const double cU = 1.0 / (16.0 * PI * (1.0 - nu) * G), a1 = 3.0 - 4.0 * nu;
    double Us[9] = {0}, Ie[3] = {0};   // int U dS ; int e ln R dtheta (= CPV int e / rho^2 dS)
    for (int k = 0; k < 3; ++k) {
        double a[3], b[3], ab[3];
        for (int c = 0; c < 3; ++c) {
            a[c] = v[k][c] - xi[c];
            b[c] = v[(k + 1) % 3][c] - xi[c];
        }
        cross3(a, b, ab);
        const double cr = sqrt(ab[0] * ab[0] + ab[1] * ab[1] + ab[2] * ab[2]);
        for (int q = 0; q < NGL; ++q) {
            const double s = 0.5 * (c_gl_x[q] + 1.0), w = 0.5 * c_gl_w[q];
            double P[3];
            for (int c = 0; c < 3; ++c) P[c] = a[c] + s * (b[c] - a[c]);
            const double R = sqrt(P[0] * P[0] + P[1] * P[1] + P[2] * P[2]);
            const double e[3] = {P[0] / R, P[1] / R, P[2] / R};
            const double dth = w * cr / (R * R);          // d theta
            // int_0^R U rho drho = R U(e) rho -> U(e) (homogeneous of degree -1)
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) Us[3 * r + c] += dth * R * cU * ((r == c ? a1 : 0.0) + e[r] * e[c]);
            for (int c = 0; c < 3; ++c) Ie[c] += dth * log(R) * e[c];
        }
    }
    // CPV P_self: r = -e, P_ij = -(1-2nu)(r_i n_j - r_j n_i) / (8 pi (1-nu) rho^2)
    const double cp = -(1.0 - 2.0 * nu) / (8.0 * PI * (1.0 - nu));
    double Ps[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) Ps[3 * r + c] = cp * (-Ie[r] * nn[c] + Ie[c] * nn[r]) + (r == c ? 0.5 : 0.0);
    for (int k = 0; k < 9; ++k) {
        DU[9 * i + k] = Us[k];
        DP[9 * i + k] = Ps[k];
    }
    // subtract what the FMM adds from the panel's own quadrature points (y_q != xi)
    const float cx = cent[3 * i], cy = cent[3 * i + 1], cz = cent[3 * i + 2];
    for (int q = 0; q < nq; ++q) {
        const int64_t o = i * nq + q;
        const double dx = (double)(cx - qp[3 * o]), dy = (double)(cy - qp[3 * o + 1]), dz = (double)(cz - qp[3 * o + 2]);
        const double r2 = dx * dx + dy * dy + dz * dz;
        if (r2 == 0.0) continue;
        const double rr = sqrt(r2), w = qw[o];
        const double e[3] = {dx / rr, dy / rr, dz / rr};
        const double dn = e[0] * nn[0] + e[1] * nn[1] + e[2] * nn[2];
        const double a = 1.0 - 2.0 * nu;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                Us[3 * r + c] -= w * cU / rr * ((r == c ? a1 : 0.0) + e[r] * e[c]);
                Ps[3 * r + c] -= w / (8.0 * PI * (1.0 - nu) * r2) *
                                 (dn * ((r == c ? a : 0.0) + 3.0 * e[r] * e[c]) - a * (e[r] * nn[c] - e[c] * nn[r]));
            }
    }
    for (int k = 0; k < 9; ++k) {
        CU[9 * i + k] = (float)Us[k];
        CP[9 * i + k] = (float)Ps[k];
    }
}

// ------------------------------------------------------------------ operator L(u, p) = P u - U p
// mode 0 (A x): p = x on Dirichlet panels, u = x on Neumann panels
// mode 1 (rhs): u = value on Dirichlet panels, p = value on Neumann panels
template <class XT>
__device__ __forceinline__ void split_up(int mode, int bc, const XT* xv, XT* u, XT* p) {
    const bool dir = bc == 0;
    const bool is_p = mode == 0 ? dir : !dir;
    for (int c = 0; c < 3; ++c) {
        u[c] = is_p ? XT(0) : xv[c];
        p[c] = is_p ? xv[c] : XT(0);
    }
}

// FMM source densities of the quadrature points (fp32: the FMM's input precision)
template <class XT>
__global__ void expand_kernel(int mode, const int32_t* __restrict__ bc, const XT* __restrict__ x, int64_t n, int nq,
                              float* __restrict__ f, float* __restrict__ g) {
    const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (o >= n * nq) return;
    const int64_t j = o / nq;
    XT u[3], p[3];
    split_up(mode, bc[j], x + 3 * j, u, p);
    for (int c = 0; c < 3; ++c) {
        f[3 * o + c] = (float)-p[c];      // single layer enters as - U p
        g[3 * o + c] = (float)u[c];       // double layer as + P u
    }
}

// out = sign (y + CP u - CU p): the local pass of l. 189 in fp64 (x and y fp32 outside GMRES,
// fp64 inside)
template <class XT, class YT, class T>
__global__ void local_kernel(int mode, double sign, const int32_t* __restrict__ bc, const XT* __restrict__ x,
                             int64_t n, const float* __restrict__ CU, const float* __restrict__ CP,
                             const YT* __restrict__ y, T* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    XT u[3], p[3];
    split_up(mode, bc[i], x + 3 * i, u, p);
    for (int r = 0; r < 3; ++r) {
        double s = y[3 * i + r];
        for (int c = 0; c < 3; ++c)
            s += (double)CP[9 * i + 3 * r + c] * (double)u[c] - (double)CU[9 * i + 3 * r + c] * (double)p[c];
        out[3 * i + r] = (T)(sign * s);
    }
}

// L(u, p) of the panel vector x.  y64: the FMM result in fp64 (B.yd; GMRES), else fp32 (B.y)
template <class XT, class T>
static void apply_L(Bem& B, int mode, double sign, const int32_t* bc, const XT* x, T* out, cudaStream_t s,
                    bool y64 = false, bool expand = true) {
    const int64_t n = B.n;
    if (expand) {   // (not needed when stored operators replace every pass over the quadrature points)
        expand_kernel<XT><<<ceil_div(n * B.nq, 256), 256, 0, s>>>(mode, bc, x, n, B.nq, B.f.p, B.g.p);
        EB_CHECK_LAUNCH();
    }
    static const bool prof = std::getenv("EBEM_BEM_PROFILE") != nullptr;   // diagnostics: phase times to stderr
    if (prof) set_profiling(*B.tree, 1);
    if (y64) {
        if (!B.yd.p) B.yd.alloc(3 * n);
        B.tree->out_d = B.yd.p;
    }
    struct OutGuard {
        Tree& t;
        ~OutGuard() { t.out_d = nullptr; }
    } out_guard{*B.tree};
    fmm_evaluate(*B.tree, K_UP, B.f.p, B.g.p, B.y.p, s);
    if (prof) {
        EB_CUDA(cudaStreamSynchronize(s));
        ebem_phase_stat st[Tree::NPHASE];
        const int np = phase_stats(*B.tree, K_UP, st, Tree::NPHASE);
        double tot = 0;
        for (int i = 0; i < np; ++i) {
            std::fprintf(stderr, "%s %.2f", st[i].name, st[i].ms);
            if (st[i].interactions > 0) std::fprintf(stderr, " (%.2f G pairs)", st[i].interactions / 1e9);
            std::fprintf(stderr, "  ");
            tot += st[i].ms;
        }
        std::fprintf(stderr, "| total %.2f ms\n", tot);
    }
    if (y64) local_kernel<XT, double, T><<<ceil_div(n, 256), 256, 0, s>>>(mode, sign, bc, x, n, B.CU.p, B.CP.p, B.yd.p, out);
    else local_kernel<XT, float, T><<<ceil_div(n, 256), 256, 0, s>>>(mode, sign, bc, x, n, B.CU.p, B.CP.p, B.y.p, out);
    EB_CHECK_LAUNCH();
}

Bem* bem_create(const float* verts, int64_t n, int nq, int max_pts, int p, const Material& m, cudaStream_t s) {
    EB_REQUIRE(nq == 1 || nq == 16, "nq must be 1 or 16");
    static bool gl_ready = false;
    if (!gl_ready) {
        std::vector<double> x, w;
        gauss_legendre(NGL, x, w);
        EB_CUDA(cudaMemcpyToSymbol(c_gl_x, x.data(), sizeof(double) * NGL));
        EB_CUDA(cudaMemcpyToSymbol(c_gl_w, w.data(), sizeof(double) * NGL));
        gl_ready = true;
    }
    auto B = std::make_unique<Bem>();
    B->n = n;
    B->nq = nq;
    B->mat = m;
    const int64_t ns = n * nq;
    B->cent.alloc(3 * n);
    B->nrm.alloc(3 * n);
    B->area.alloc(n);
    B->qpts.alloc(3 * ns);
    B->qnrm.alloc(3 * ns);
    B->qw.alloc(ns);
    panels_kernel<<<ceil_div(n, 128), 128, 0, s>>>(verts, n, nq, B->cent.p, B->nrm.p, B->area.p, B->qpts.p, B->qnrm.p,
                                                   B->qw.p);
    EB_CHECK_LAUNCH();
    B->CU.alloc(9 * n);
    B->CP.alloc(9 * n);
    B->DU.alloc(9 * n);
    B->DP.alloc(9 * n);
    self_terms_kernel<<<ceil_div(n, 128), 128, 0, s>>>(verts, n, nq, B->qpts.p, B->qw.p, B->cent.p, B->nrm.p, m.G, m.nu,
                                                       B->CU.p, B->CP.p, B->DU.p, B->DP.p);
    EB_CHECK_LAUNCH();
    // W boxes with fewer than 16 n_e quadrature sources are summed directly (R11): in the BEM
    // the far field is fp64 (M2T ~7 ps per target-equivalent point pair) while a direct entry
    // costs one fp32 pair, or 36 B of the near operator per target and panel (measured on
    // configs[4]: 99 -> 90 ms per iteration)
    B->tree = build_tree(B->qpts.p, B->qnrm.p, B->qw.p, ns, B->cent.p, n, max_pts, p, m, s, 16.0);
    // GMRES needs an operator linear to ~1e-8: fp64 far field and the precise (drained)
    // tensor-core accumulation (see fmm.cu)
    tree_precise(*B->tree, s);
    B->f.alloc(3 * ns);
    B->g.alloc(3 * ns);
    B->y.alloc(3 * n);
    EB_CUDA(cudaStreamSynchronize(s));
    return B.release();
}

void bem_free(Bem* B) { delete B; }

void bem_apply(Bem& B, const int32_t* bc, const float* x, float* y, cudaStream_t s) {
    apply_L<float, float>(B, 0, 1.0, bc, x, y, s);
}

void bem_rhs(Bem& B, const int32_t* bc, const float* val, float* b, cudaStream_t s) {
    apply_L<float, float>(B, 1, -1.0, bc, val, b, s);
}

// ------------------------------------------------------------------ GMRES (fp64 Krylov basis)
// h[j] = V_j . w (j < k) over n: DOT_BLOCKS blocks each reduce a contiguous slice for 8 basis
// vectors at a time (w read once per 8), partial sums combined in a fixed order by
// dots_finish (deterministic).  One block per vector left most SMs idle: 17 ms of every
// GMRES iteration on the 1.9 M-panel cell.
constexpr int DOT_BLOCKS = 592, DOT_T = 256, DOT_J = 8;
__global__ void __launch_bounds__(DOT_T)
dots_partial(const double* __restrict__ V, int64_t ld, int k, const double* __restrict__ w, int64_t n,
             double* __restrict__ part) {
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t i0 = blockIdx.x * per, i1 = min(n, i0 + per);
    __shared__ double red[DOT_T / 32][DOT_J];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j0 = 0; j0 < k; j0 += DOT_J) {
        double acc[DOT_J];
#pragma unroll
        for (int q = 0; q < DOT_J; ++q) acc[q] = 0.0;
        for (int64_t i = i0 + threadIdx.x; i < i1; i += DOT_T) {
            const double wi = w[i];
#pragma unroll
            for (int q = 0; q < DOT_J; ++q)
                if (j0 + q < k) acc[q] = fma(V[(int64_t)(j0 + q) * ld + i], wi, acc[q]);
        }
#pragma unroll
        for (int q = 0; q < DOT_J; ++q) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
        }
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < DOT_J; ++q) red[warp][q] = acc[q];
        __syncthreads();
        if (threadIdx.x < DOT_J && j0 + threadIdx.x < k) {
            double t = 0.0;
            for (int wv = 0; wv < DOT_T / 32; ++wv) t += red[wv][threadIdx.x];
            part[(int64_t)blockIdx.x * 64 + j0 + threadIdx.x] = t;
        }
        __syncthreads();
    }
}

__global__ void dots_finish(const double* __restrict__ part, int nblocks, int k, double* __restrict__ h) {
    const int j = threadIdx.x;
    if (j >= k) return;
    double t = 0.0;
    for (int b = 0; b < nblocks; ++b) t += part[(int64_t)b * 64 + j];
    h[j] = t;
}

// h[0..k) = V_j . w; part: DOT_BLOCKS x 64 scratch (k <= 64)
static void dots(const double* V, int64_t ld, int k, const double* w, int64_t n, double* part, double* h,
                 cudaStream_t s) {
    EB_REQUIRE(k <= 64, "GMRES restart length above 63");
    const int nb = (int)std::min<int64_t>(DOT_BLOCKS, std::max<int64_t>(1, n / 1024));
    dots_partial<<<nb, DOT_T, 0, s>>>(V, ld, k, w, n, part);
    EB_CHECK_LAUNCH();
    dots_finish<<<1, 64, 0, s>>>(part, nb, k, h);
    EB_CHECK_LAUNCH();
}

__global__ void axpy_basis(const double* __restrict__ V, int64_t ld, int k, const double* __restrict__ h, double sgn,
                           double* __restrict__ w, int64_t n) {
    // w += sgn * sum_{j<k} h[j] V_j
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0;
    for (int j = 0; j < k; ++j) s += h[j] * V[j * ld + i];
    w[i] += sgn * s;
}

__global__ void scale_copy(const double* __restrict__ a, double sc, double* __restrict__ b, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = sc * a[i];
}
__global__ void to_f32_kernel(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = (float)a[i];
}
__global__ void to_f64_kernel(const float* __restrict__ a, double* __restrict__ b, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = (double)a[i];
}
__global__ void add_kernel(const double* __restrict__ a, double* __restrict__ b, int64_t n) {   // b += a
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] += a[i];
}
// diagnostics: a deterministic pseudo-random vector in [-1, 1) (EBEM_GMRES_PROBE)
__global__ void hash_fill(double* __restrict__ a, int64_t n, double sc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    a[i] = sc * ((double)(z >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0);
}

__global__ void sub_kernel(const double* __restrict__ a, double* __restrict__ b, int64_t n) {   // b = a - b
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i] - b[i];
}

// block-Jacobi right preconditioner: M_i = diagonal block of A (-U_self on Dirichlet panels,
// 1/2 I + P_self on Neumann panels); Minv_i by 3x3 cofactors in fp64
__global__ void prec_setup(const int32_t* __restrict__ bc, const double* __restrict__ DU,
                           const double* __restrict__ DP, int64_t n, double* __restrict__ Minv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double a[9];
    const bool dir = bc[i] == 0;
    for (int k = 0; k < 9; ++k) a[k] = dir ? -DU[9 * i + k] : DP[9 * i + k];
    const double c00 = a[4] * a[8] - a[5] * a[7], c01 = a[5] * a[6] - a[3] * a[8], c02 = a[3] * a[7] - a[4] * a[6];
    const double det = a[0] * c00 + a[1] * c01 + a[2] * c02;
    const double id = 1.0 / det;
    double* m = Minv + 9 * i;
    m[0] = c00 * id;
    m[3] = c01 * id;
    m[6] = c02 * id;
    m[1] = (a[2] * a[7] - a[1] * a[8]) * id;
    m[4] = (a[0] * a[8] - a[2] * a[6]) * id;
    m[7] = (a[1] * a[6] - a[0] * a[7]) * id;
    m[2] = (a[1] * a[5] - a[2] * a[4]) * id;
    m[5] = (a[2] * a[3] - a[0] * a[5]) * id;
    m[8] = (a[0] * a[4] - a[1] * a[3]) * id;
}

__global__ void prec_apply(const double* __restrict__ Minv, const double* __restrict__ v, int64_t n,
                           double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int r = 0; r < 3; ++r)
        out[3 * i + r] = Minv[9 * i + 3 * r] * v[3 * i] + Minv[9 * i + 3 * r + 1] * v[3 * i + 1] +
                         Minv[9 * i + 3 * r + 2] * v[3 * i + 2];
}

static double dnorm(const double* v, int64_t n, double* tmp, double* part, cudaStream_t s) {
    dots(v, 0, 1, v, n, part, tmp, s);
    double h = 0;
    d2h(&h, tmp, 1, s);
    EB_CUDA(cudaStreamSynchronize(s));
    return std::sqrt(h);
}

int bem_gmres(Bem& B, const int32_t* bc, const float* val, float* x, int m, int max_iter, double tol, int32_t* iters,
              double* resid, int precond, cudaStream_t s) {
    const int64_t n3 = 3 * B.n;
    B.hist_est.clear();
    B.hist_true.clear();
    static const bool trace = std::getenv("EBEM_GMRES_TRACE") != nullptr;   // diagnostics: history to stderr
    // M2L accumulation for this solve: the full-chain (fast) kernel for tolerances no tighter
    // than 1e-6 (the operator's linearity probe is 2.4e-7 with it: configs[4] with the paper's
    // unpreconditioned solver converged in 1295 iterations / 80.7 s against 1405 / 96.7 s with
    // the drained kernel, reading R12); the drained kernel for tighter tolerances and
    // for bem_apply outside a solve.
    struct M2LMode {
        Tree& t;
        cudaStream_t s;
        ~M2LMode() { tree_m2l_fast(t, false, s); }
    } mode{*B.tree, s};
    // (EBEM_BEM_M2L=fast|precise overrides; EBEM_BEM_PRECISE_M2L=1 = precise)
    bool m2l_fast = tol >= 1e-6 && !std::getenv("EBEM_BEM_PRECISE_M2L");
    if (const char* e = std::getenv("EBEM_BEM_M2L")) m2l_fast = std::strcmp(e, "fast") == 0;
    tree_m2l_fast(*B.tree, m2l_fast, s);
    DBuf<double> V((size_t)(m + 1) * n3), w(n3), b(n3), xd(n3), hd(m + 2), Minv, tp, part((size_t)DOT_BLOCKS * 64);
    struct SplitGuard {
        Tree& t;
        ~SplitGuard() { t.split_mode = 0; }
    } split_guard{*B.tree};
    // right-hand side b = -L(known values), with the combined single + double layer loops (the
    // per-leaf grouping below is only set up once a solve is needed)
    B.tree->split_mode = 0;
    apply_L<float, double>(B, 1, -1.0, bc, val, b.p, s, true);
    const double bn = dnorm(b.p, n3, hd.p, part.p, s);
    if (bn == 0.0) {   // x = 0 solves it; nothing else (near operator, grouping) is set up
        EB_CUDA(cudaMemsetAsync(x, 0, sizeof(float) * n3, s));
        EB_CUDA(cudaStreamSynchronize(s));
        if (iters) *iters = 0;
        if (resid) *resid = 0;
        return EBEM_OK;
    }
    to_f64_kernel<<<ceil_div(n3, 256), 256, 0, s>>>(x, xd.p, n3);
    EB_CHECK_LAUNCH();
    bool x_zero = dnorm(xd.p, n3, hd.p, part.p, s) == 0.0;   // r0 = b without a matvec
    if (precond) {
        Minv.alloc(9 * B.n);
        tp.alloc(n3);
        prec_setup<<<ceil_div(B.n, 256), 256, 0, s>>>(bc, B.DU.p, B.DP.p, B.n, Minv.p);
        EB_CHECK_LAUNCH();
    }
    // sources grouped per leaf by panel type: each then carries one layer only, and the check
    // potentials run one-kernel pair loops (EBEM_BEM_SPLIT=0: the combined U+P loop)
    const bool split = !(std::getenv("EBEM_BEM_SPLIT") && std::atoi(std::getenv("EBEM_BEM_SPLIT")) == 0);
    if (split) tree_partition_sources(*B.tree, bc, B.nq, s);
    B.tree->split_mode = split ? 1 : 0;   // A x: Dirichlet panels carry p (single layer)
    // near field, and the S2M / S2L check potentials, from operators held in HBM (bem_near.cu)
    // when they fit (built in that order: the near operator saves the most per byte)
    Tree& T = *B.tree;
    const bool use_nm = near_matrix_enabled() && near_matrix_build(T, B.nq, B.n, bc, B.mat, B.nm, s);
    const bool use_cm = use_nm && T.use_tc && check_matrix_enabled() &&
                        panel_op_build(T, PanelOp::S2M, B.nq, B.n, bc, B.mat, B.s2m_op, s);
    const bool use_cl = use_cm && (T.n_s2l == 0 || panel_op_build(T, PanelOp::S2L, B.nq, B.n, bc, B.mat, B.s2l_op, s));
    // precond = 2: leaf-block Jacobi (bem_prec.cu), built after the HBM operators (they save
    // more per byte); the 3x3 blocks when the inverses do not fit
    LeafBlockPrec lbp;
    const auto t_lb = std::chrono::steady_clock::now();
    const bool use_lb = precond == 2 &&
                        leafblock_build(T, B.n, B.nq, B.cent.p, B.qpts.p, B.qnrm.p, B.qw.p, bc, B.DU.p, B.DP.p, B.mat,
                                        lbp, s);
    if (precond == 2 && std::getenv("EBEM_BEM_PROFILE"))
        std::fprintf(stderr, "[bem] leaf-block preconditioner: %s, %d blocks, %.2f GB, built in %.1f ms\n",
                     use_lb ? "on" : "did not fit / singular (3x3 blocks)", lbp.nblocks, lbp.entries * 8e-9,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_lb).count());
    auto prec = [&](const double* v, double* out) {     // out = M^-1 v
        if (use_lb) {
            leafblock_apply(T, lbp, v, out, s);
        } else {
            prec_apply<<<ceil_div(B.n, 256), 256, 0, s>>>(Minv.p, v, B.n, out);
            EB_CHECK_LAUNCH();
        }
    };
    struct HookGuard {
        Tree& t;
        ~HookGuard() {
            t.near_hook = t.s2m_hook = t.s2l_hook = nullptr;
            t.near_f64 = false;
            t.force_serial = false;
        }
    } hook_guard{T};
    // one stream inside the solve: the HBM-bound near operator beside the tensor-core M2L was
    // slower than the two back to back (configs[4]: 82 vs 77.5 ms per iteration)
    T.force_serial = !(std::getenv("EBEM_BEM_CONC") && std::atoi(std::getenv("EBEM_BEM_CONC")));
    if (use_nm && B.tree->near_sorted_d.n < (size_t)3 * B.tree->ntrg) B.tree->near_sorted_d.alloc(3 * B.tree->ntrg);
    // out = A v, fp64 in and out: the near operator reads v in fp64 and accumulates in fp64,
    // the local pass is fp64 and the FMM returns its sum in fp64; only the far field's
    // sources (the quadrature-point densities) are fp32 (the FMM's own precision)
    auto matvec = [&](const double* v, double* out) {
        if (use_nm) {
            T.near_hook = [&, v](cudaStream_t st) { near_matrix_apply(T, B.nm, v, T.near_sorted_d.p, st); };
            T.near_f64 = true;
        }
        if (use_cm)
            T.s2m_hook = [&, v](cudaStream_t st) {
                panel_op_apply(T, B.s2m_op, v, nullptr, T.Qb.p, T.Qs.p, T.plan->ldc, st);
            };
        if (use_cl && T.n_s2l)
            T.s2l_hook = [&, v](cudaStream_t st) {
                panel_op_apply(T, B.s2l_op, v, nullptr, T.Qdb.p, T.Qds.p, T.plan->ldc, st);
            };
        apply_L<double, double>(B, 0, 1.0, bc, v, out, s, true, !(use_nm && use_cl));
        T.near_hook = T.s2m_hook = T.s2l_hook = nullptr;
        T.near_f64 = false;
    };
    auto pmatvec = [&](const double* v, double* out) {  // out = A M^-1 v (right preconditioning)
        if (!precond) return matvec(v, out);
        prec(v, tp.p);
        matvec(tp.p, out);
    };
    int it = 0;
    double rel = 1.0;
    std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), h(m + 1), h2(m + 1);
    while (true) {
        if (x_zero) {
            EB_CUDA(cudaMemcpyAsync(w.p, b.p, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s));
            x_zero = false;
        } else {
            matvec(xd.p, w.p);
            sub_kernel<<<ceil_div(n3, 256), 256, 0, s>>>(b.p, w.p, n3);   // w = b - A x
            EB_CHECK_LAUNCH();
        }
        const double beta = dnorm(w.p, n3, hd.p, part.p, s);
        rel = beta / bn;
        B.hist_true.push_back(rel);
        if (trace) std::fprintf(stderr, "[gmres] it %d true residual %.3e\n", it, rel);
        if (rel <= tol || it >= max_iter) break;
        scale_copy<<<ceil_div(n3, 256), 256, 0, s>>>(w.p, 1.0 / beta, V.p, n3);
        EB_CHECK_LAUNCH();
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int k = 0;
        for (int j = 0; j < m; ++j) {
            pmatvec(V.p + (int64_t)j * n3, w.p);
            // classical Gram-Schmidt with one re-orthogonalisation, on the device
            for (int pass = 0; pass < 2; ++pass) {
                dots(V.p, n3, j + 1, w.p, n3, part.p, hd.p, s);
                axpy_basis<<<ceil_div(n3, 256), 256, 0, s>>>(V.p, n3, j + 1, hd.p, -1.0, w.p, n3);
                EB_CHECK_LAUNCH();
                d2h((pass ? h2 : h).data(), hd.p, j + 1, s);
            }
            const double hn = dnorm(w.p, n3, hd.p, part.p, s);
            for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = h[i] + h2[i];
            H[(size_t)(j + 1) * m + j] = hn;
            if (hn > 0) {
                scale_copy<<<ceil_div(n3, 256), 256, 0, s>>>(w.p, 1.0 / hn, V.p + (int64_t)(j + 1) * n3, n3);
                EB_CHECK_LAUNCH();
            }
            for (int i = 0; i < j; ++i) {   // previous Givens rotations
                const double a = H[(size_t)i * m + j], c = H[(size_t)(i + 1) * m + j];
                H[(size_t)i * m + j] = cs[i] * a + sn[i] * c;
                H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * c;
            }
            const double a = H[(size_t)j * m + j], c = H[(size_t)(j + 1) * m + j];
            const double den = std::hypot(a, c);
            cs[j] = a / den;
            sn[j] = c / den;
            H[(size_t)j * m + j] = den;
            H[(size_t)(j + 1) * m + j] = 0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            ++it;
            k = j + 1;
            rel = std::fabs(g[j + 1]) / bn;
            B.hist_est.push_back(rel);
            if (trace) std::fprintf(stderr, "[gmres] it %d estimate %.3e\n", it, rel);
            if (rel <= tol || it >= max_iter || hn == 0) break;
        }
        // y = H^-1 g (upper triangular), x += V y
        std::vector<double> y(k);
        for (int i = k - 1; i >= 0; --i) {
            double sum = g[i];
            for (int l = i + 1; l < k; ++l) sum -= H[(size_t)i * m + l] * y[l];
            y[i] = sum / H[(size_t)i * m + i];
        }
        h2d(hd.p, y.data(), k, s);
        if (precond) {     // x += M^-1 (V y)
            EB_CUDA(cudaMemsetAsync(w.p, 0, sizeof(double) * n3, s));
            axpy_basis<<<ceil_div(n3, 256), 256, 0, s>>>(V.p, n3, k, hd.p, 1.0, w.p, n3);
            prec(w.p, tp.p);
            add_kernel<<<ceil_div(n3, 256), 256, 0, s>>>(tp.p, xd.p, n3);
        } else {
            axpy_basis<<<ceil_div(n3, 256), 256, 0, s>>>(V.p, n3, k, hd.p, 1.0, xd.p, n3);
        }
        EB_CHECK_LAUNCH();
        if (it >= max_iter) {
            // true residual of the final iterate
            matvec(xd.p, w.p);
            sub_kernel<<<ceil_div(n3, 256), 256, 0, s>>>(b.p, w.p, n3);
            EB_CHECK_LAUNCH();
            rel = dnorm(w.p, n3, hd.p, part.p, s) / bn;
            B.hist_true.push_back(rel);
            if (trace) std::fprintf(stderr, "[gmres] it %d true residual %.3e (final)\n", it, rel);
            break;
        }
    }
    if (std::getenv("EBEM_GMRES_PROBE")) {
        // linearity of the operator as GMRES applies it: |A(x + y) - A x - A y| / |A (x + y)|
        // for the solution x and a pseudo-random y of the same norm (rounding noise that
        // bounds the attainable residual)
        DBuf<double> y(n3), xy(n3), Ax(n3), Ay(n3), Axy(n3);
        const double xn = dnorm(xd.p, n3, hd.p, part.p, s);
        hash_fill<<<ceil_div(n3, 256), 256, 0, s>>>(y.p, n3, 1.0);
        const double yn = dnorm(y.p, n3, hd.p, part.p, s);
        hash_fill<<<ceil_div(n3, 256), 256, 0, s>>>(y.p, n3, xn / yn);
        EB_CUDA(cudaMemcpyAsync(xy.p, xd.p, sizeof(double) * n3, cudaMemcpyDeviceToDevice, s));
        add_kernel<<<ceil_div(n3, 256), 256, 0, s>>>(y.p, xy.p, n3);
        matvec(xd.p, Ax.p);
        matvec(y.p, Ay.p);
        matvec(xy.p, Axy.p);
        add_kernel<<<ceil_div(n3, 256), 256, 0, s>>>(Ay.p, Ax.p, n3);      // Ax += Ay
        const double den = dnorm(Axy.p, n3, hd.p, part.p, s);
        sub_kernel<<<ceil_div(n3, 256), 256, 0, s>>>(Axy.p, Ax.p, n3);     // Ax = Axy - (Ax + Ay)
        const double num = dnorm(Ax.p, n3, hd.p, part.p, s);
        std::fprintf(stderr, "[gmres probe] eps_linearity %.3e  |x| %.4e  |b| %.4e\n", num / den, xn, bn);
    }
    to_f32_kernel<<<ceil_div(n3, 256), 256, 0, s>>>(xd.p, x, n3);
    EB_CHECK_LAUNCH();
    EB_CUDA(cudaStreamSynchronize(s));
    if (iters) *iters = it;
    if (resid) *resid = rel;
    return rel <= tol ? EBEM_OK : EBEM_ERR_NOCONV;
}

int bem_history(const Bem& B, int what, double* buf, int cap) {
    const std::vector<double>& h = what == 0 ? B.hist_est : B.hist_true;
    const int n = (int)h.size();
    for (int i = 0; i < std::min(n, cap); ++i) buf[i] = h[i];
    return n;
}

}  // namespace ebem
