// KIFMM operator precomputation (fp64, on the device): "The M2M, L2L
// and M2L operators needed in the algorithm, in the case of KIFMM are represented by
// matrices mapping density values on different equivalent surfaces to each other, and
// are computed automatically for each needed kernel."
//
// Reading R6: cube surfaces with p points per edge (equivalent) and p+1
// (check); radii 1.05 / 2.95; Tikhonov-regularised check->equivalent solve with
// a = rcond * s_max(K), rcond = max(1e-9, 10^-(p+1)).  The solve is factored as
// [K; a I] = Q R (classical Gram-Schmidt with one full re-orthogonalisation, fp64), so
// the Tikhonov pseudo-inverse is R^-1 Q_1^T (Q_1 = first 3 n_c rows of Q).
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>

#include "elastic.cuh"
#include "fmm.cuh"

namespace ebem {

static std::vector<double> surface_grid(int p) {
    std::vector<double> out;
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j)
            for (int k = 0; k < p; ++k)
                if (i == 0 || i == p - 1 || j == 0 || j == p - 1 || k == 0 || k == p - 1) {
                    double t[3] = {-1.0 + 2.0 * i / (p - 1), -1.0 + 2.0 * j / (p - 1), -1.0 + 2.0 * k / (p - 1)};
                    out.insert(out.end(), t, t + 3);
                }
    return out;
}

// K[b] (3nx x 3ny, row-major, ld = ldk) with X_i = xo[b] + xs sx_i, Y_j = yo[b] + ys sy_j,
// U kernel (PAPER.md Eq. disp_1), times scale.
__global__ void kmat_kernel(const double* __restrict__ sx, int nx, double xs, const double* __restrict__ sy,
                            int ny, double ys, const double* __restrict__ xo, const double* __restrict__ yo,
                            double cU, double a1, double scale, double* __restrict__ K, int64_t strideK) {
    const int b = blockIdx.y;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)nx * ny) return;
    const int i = (int)(e / ny), j = (int)(e % ny);
    double dx = xo[3 * b] + xs * sx[3 * i] - (yo[3 * b] + ys * sy[3 * j]);
    double dy = xo[3 * b + 1] + xs * sx[3 * i + 1] - (yo[3 * b + 1] + ys * sy[3 * j + 1]);
    double dz = xo[3 * b + 2] + xs * sx[3 * i + 2] - (yo[3 * b + 2] + ys * sy[3 * j + 2]);
    double r = sqrt(dx * dx + dy * dy + dz * dz);
    double d[3] = {dx / r, dy / r, dz / r};
    double c = scale * cU / r;
    double* Kb = K + b * strideK;
    const int ld = 3 * ny;
    for (int a = 0; a < 3; ++a)
        for (int q = 0; q < 3; ++q)
            Kb[(int64_t)(3 * i + a) * ld + 3 * j + q] = c * ((a == q ? a1 : 0.0) + d[a] * d[q]);
}

static void kmat(const Plan& P, const DBuf<double>& sx, int nx, double xs, const DBuf<double>& sy, int ny,
                 double ys, const std::vector<double>& xo, const std::vector<double>& yo, double scale,
                 double* K, int batch, cudaStream_t s) {
    DBuf<double> dxo(3 * batch), dyo(3 * batch);
    h2d(dxo.p, xo.data(), 3 * batch, s);
    h2d(dyo.p, yo.data(), 3 * batch, s);
    dim3 grid(ceil_div((int64_t)nx * ny, 256), batch);
    kmat_kernel<<<grid, 256, 0, s>>>(sx.p, nx, xs, sy.p, ny, ys, dxo.p, dyo.p, P.mat.cU, P.mat.a1, scale, K,
                                     (int64_t)9 * nx * ny);
    EB_CHECK_LAUNCH();
    EB_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ CGS2 QR
// One cooperative kernel for the whole factorisation (grid-wide barriers between the steps of
// each column): a launch per step and column took ~3 n launches (≈ 1500 at p = 4, 4400 at
// p = 10) -- one-time work, but it filled every launch list with plan kernels.
// Column j: v = a_j; two passes of r = Q_{<j}^T v, v -= Q_{<j} r, R_{<j, j} += r (classical
// Gram-Schmidt with one full re-orthogonalisation); R_jj = |v|, q_j = v / R_jj.  Every
// reduction has a fixed order (deterministic).
namespace cg = cooperative_groups;

constexpr int PT = 256;

__device__ __forceinline__ double block_sum(double x, double* sh) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = x;
    __syncthreads();
    double t = 0.0;
    for (int k = 0; k < PT / 32; ++k) t += sh[k];
    return t;
}

__global__ void __launch_bounds__(PT)
cgs2_coop(double* __restrict__ Q, int m, int n, double* __restrict__ R, double* __restrict__ v,
          double* __restrict__ r, double* __restrict__ part) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[PT / 32];
    const int64_t gt = (int64_t)blockIdx.x * PT + threadIdx.x, gs = (int64_t)gridDim.x * PT;
    for (int j = 0; j < n; ++j) {
        for (int64_t i = gt; i < m; i += gs) v[i] = Q[(int64_t)j * m + i];
        grid.sync();
        for (int pass = 0; pass < 2 && j > 0; ++pass) {
            for (int k = blockIdx.x; k < j; k += gridDim.x) {          // r_k = q_k . v
                double x = 0.0;
                for (int i = threadIdx.x; i < m; i += PT) x += Q[(int64_t)k * m + i] * v[i];
                x = block_sum(x, sh);
                if (threadIdx.x == 0) r[k] = x;
            }
            grid.sync();
            for (int64_t i = gt; i < m; i += gs) {                    // v -= Q r
                double x = 0.0;
                for (int k = 0; k < j; ++k) x += Q[(int64_t)k * m + i] * r[k];
                v[i] -= x;
            }
            for (int64_t k = gt; k < j; k += gs) R[(int64_t)j * n + k] += r[k];
            grid.sync();
        }
        double x = 0.0;                                                // |v|^2, block partials
        for (int64_t i = gt; i < m; i += gs) x += v[i] * v[i];
        x = block_sum(x, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = x;
        grid.sync();
        double nn = 0.0;
        for (int b = 0; b < (int)gridDim.x; ++b) nn += part[b];
        const double nrm = sqrt(nn);
        for (int64_t i = gt; i < m; i += gs) Q[(int64_t)j * m + i] = v[i] / nrm;
        if (gt == 0) R[(int64_t)j * n + j] = nrm;
        grid.sync();
    }
}

static int coop_grid(const void* fn) {
    int per = 0;
    EB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, PT, 0));
    return std::max(1, std::min(per, 2)) * num_sms();
}

// A (m x n) column-major in Q on entry; on exit Q has orthonormal columns and R (n x n,
// column-major, upper) satisfies A = Q R.
static void cgs2_qr(double* Q, int m, int n, double* R, cudaStream_t s) {
    const int grid = coop_grid((const void*)cgs2_coop);
    DBuf<double> v(m), r(n), part(grid);
    EB_CUDA(cudaMemsetAsync(R, 0, sizeof(double) * n * n, s));
    void* args[] = {&Q, &m, &n, &R, &v.p, &r.p, &part.p};
    EB_CUDA(cudaLaunchCooperativeKernel((const void*)cgs2_coop, grid, PT, args, 0, s));
    EB_CHECK_LAUNCH();
    EB_CUDA(cudaStreamSynchronize(s));
}

// X = R^-1 (both n x n; R column-major upper, X row-major upper): a warp per column j of X,
// back substitution X[i, j] = (delta_ij - sum_{i<k<=j} R[i,k] X[k, j]) / R[i,i] from i = j
// down to 0, the column kept in shared memory (one launch for all columns)
constexpr int TI_W = 4;
__global__ void __launch_bounds__(32 * TI_W)
trinv_cols(const double* __restrict__ R, int n, double* __restrict__ X) {
    extern __shared__ double col_all[];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int j = blockIdx.x * TI_W + w;
    if (j >= n) return;
    double* col = col_all + (size_t)w * n;
    for (int i = j; i >= 0; --i) {
        double x = 0.0;
        for (int k = i + 1 + l; k <= j; k += 32) x += R[(int64_t)k * n + i] * col[k];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (l == 0) col[i] = ((i == j ? 1.0 : 0.0) - x) / R[(int64_t)i * n + i];
        __syncwarp();
    }
    for (int i = l; i < n; i += 32) X[(int64_t)i * n + j] = i <= j ? col[i] : 0.0;
}

// largest singular value of K (row-major m x n): 60 power iterations on K^T K in one
// cooperative launch (v <- K^T K v / |K^T K v|, sigma = sqrt|K^T K v| at the end)
__global__ void __launch_bounds__(PT)
power_coop(const double* __restrict__ K, int m, int n, double* __restrict__ v, double* __restrict__ t,
           double* __restrict__ part, double* __restrict__ sig) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double sh[PT / 32];
    const int64_t gt = (int64_t)blockIdx.x * PT + threadIdx.x, gs = (int64_t)gridDim.x * PT;
    for (int64_t j = gt; j < n; j += gs) v[j] = 1.0 / sqrt((double)n);
    grid.sync();
    double nrm = 1.0;
    for (int it = 0; it < 60; ++it) {
        for (int64_t i = gt; i < m; i += gs) {            // t = K v
            double x = 0.0;
            for (int j = 0; j < n; ++j) x += K[i * n + j] * v[j];
            t[i] = x;
        }
        grid.sync();
        double ss = 0.0;
        for (int64_t j = gt; j < n; j += gs) {            // w = K^T t (into v after the norm)
            double x = 0.0;
            for (int i = 0; i < m; ++i) x += K[(int64_t)i * n + j] * t[i];
            ss += x * x;
        }
        ss = block_sum(ss, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = ss;
        grid.sync();
        double nn = 0.0;
        for (int b = 0; b < (int)gridDim.x; ++b) nn += part[b];
        nrm = sqrt(nn);
        for (int64_t j = gt; j < n; j += gs) {
            double x = 0.0;
            for (int i = 0; i < m; ++i) x += K[(int64_t)i * n + j] * t[i];
            v[j] = x / nrm;
        }
        grid.sync();
    }
    if (gt == 0) *sig = sqrt(nrm);
}

static double sigma_max(const double* K, int m, int n, cudaStream_t s) {
    const int grid = coop_grid((const void*)power_coop);
    DBuf<double> v(n), t(m), part(grid), sig(1);
    void* args[] = {&K, &m, &n, &v.p, &t.p, &part.p, &sig.p};
    EB_CUDA(cudaLaunchCooperativeKernel((const void*)power_coop, grid, PT, args, 0, s));
    EB_CHECK_LAUNCH();
    double h = 0;
    d2h(&h, sig.p, 1, s);
    EB_CUDA(cudaStreamSynchronize(s));
    return h;
}

__global__ void build_aug(const double* __restrict__ K, int mc, int me, double alpha, double* __restrict__ A) {
    // A column-major (mc+me) x me = [K; alpha I]
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int m = mc + me;
    if (e >= (int64_t)m * me) return;
    const int col = (int)(e / m), row = (int)(e % m);
    A[e] = row < mc ? K[(int64_t)row * me + col] : (row - mc == col ? alpha : 0.0);
}

__global__ void extract_q1t(const double* __restrict__ Q, int m, int mc, int me, double* __restrict__ Q1T) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)me * mc) return;
    const int i = (int)(e / mc), k = (int)(e % mc);
    Q1T[e] = Q[(int64_t)i * m + k];
}

// fp64 [rows x cols] (dense) -> fp32 [rows x ldb]
__global__ void cast_f32(const double* __restrict__ a, float* __restrict__ b, int64_t rows, int cols, int ldb) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * cols) return;
    const int64_t r = i / cols;
    const int c = (int)(i % cols);
    b[r * ldb + c] = (float)a[i];
}

static void to_f32(const double* a, float* b, int64_t rows, int cols, int ldb, cudaStream_t s) {
    cast_f32<<<ceil_div(rows * cols, 256), 256, 0, s>>>(a, b, rows, cols, ldb);
    EB_CHECK_LAUNCH();
}

// Factor one check->equivalent solve: returns Q1T (me x mc, fp64) and Rinv (me x me).
static void factor_solve(const Plan& P, const DBuf<double>& sc, double rc, const DBuf<double>& se,
                         double re, DBuf<double>& Q1T, DBuf<double>& Rinv, cudaStream_t s) {
    const int mc = P.mc, me = P.me, m = mc + me;
    DBuf<double> K((size_t)mc * me);
    std::vector<double> zero(3, 0.0);
    kmat(P, sc, P.nc, rc, se, P.ne, re, zero, zero, 1.0, K.p, 1, s);
    const double alpha = P.rcond * sigma_max(K.p, mc, me, s);
    DBuf<double> Q((size_t)m * me), R((size_t)me * me);
    build_aug<<<ceil_div((int64_t)m * me, 256), 256, 0, s>>>(K.p, mc, me, alpha, Q.p);
    EB_CHECK_LAUNCH();
    cgs2_qr(Q.p, m, me, R.p, s);
    Rinv.alloc((size_t)me * me);
    const size_t tsm = sizeof(double) * me * TI_W;
    if (tsm > 48 * 1024) EB_CUDA(cudaFuncSetAttribute(trinv_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
    trinv_cols<<<ceil_div(me, TI_W), 32 * TI_W, tsm, s>>>(R.p, me, Rinv.p);
    EB_CHECK_LAUNCH();
    Q1T.alloc((size_t)me * mc);
    extract_q1t<<<ceil_div((int64_t)me * mc, 256), 256, 0, s>>>(Q.p, m, mc, me, Q1T.p);
    EB_CHECK_LAUNCH();
    EB_CUDA(cudaStreamSynchronize(s));
}

// composites C[b] = Q1T * (Kb * Rinv) for a batch of kernel matrices Kb (mc x me)
static void composites(const Plan& P, const DBuf<double>& Q1T, const DBuf<double>& Rinv, const DBuf<double>& sx,
                       double xs, const DBuf<double>& sy, double ys, const std::vector<double>& xo,
                       const std::vector<double>& yo, double scale, float* out, cudaStream_t s) {
    const int mc = P.mc, me = P.me;
    const int nb = (int)xo.size() / 3;
    // operators per batch: as many as ~2 GB of fp64 scratch allows (all 316 M2L operators in one
    // batch up to p = 7, a handful of batches at p = 10)
    const double per = 8.0 * (2.0 * mc * me + (double)me * me);
    const int chunk = std::max(1, std::min(nb, (int)(2e9 / per)));
    DBuf<double> K((size_t)chunk * mc * me), T((size_t)chunk * mc * me), C((size_t)chunk * me * me);
    for (int b0 = 0; b0 < nb; b0 += chunk) {
        const int nbc = std::min(chunk, nb - b0);
        std::vector<double> xoc(xo.begin() + 3 * b0, xo.begin() + 3 * (b0 + nbc));
        std::vector<double> yoc(yo.begin() + 3 * b0, yo.begin() + 3 * (b0 + nbc));
        kmat(P, sx, P.nc, xs, sy, P.ne, ys, xoc, yoc, scale, K.p, nbc, s);
        gemm_f64(mc, me, me, 1.0, K.p, (int64_t)mc * me, me, Rinv.p, 0, me, 0.0, T.p, (int64_t)mc * me, me, nbc, s);
        gemm_f64(me, me, mc, 1.0, Q1T.p, 0, mc, T.p, (int64_t)mc * me, me, 0.0, C.p, (int64_t)me * me, me, nbc, s);
        to_f32(C.p, out + (int64_t)b0 * me * P.lde, (int64_t)nbc * me, me, P.lde, s);
    }
    EB_CUDA(cudaStreamSynchronize(s));
}

static std::shared_ptr<Plan> make_plan(int p, const Material& m, cudaStream_t s) {
    auto P = std::make_shared<Plan>();
    P->p = p;
    P->pc = p + 1;
    P->mat = m;
    P->rcond = std::max(1e-9, std::pow(10.0, -(p + 1)));
    if (const char* e = std::getenv("EBEM_RCOND")) P->rcond = std::atof(e);   // diagnostics (A/B of reading R6)
    std::vector<double> se = surface_grid(p), sc = surface_grid(P->pc);
    P->ne = (int)se.size() / 3;
    P->nc = (int)sc.size() / 3;
    P->me = 3 * P->ne;
    P->mc = 3 * P->nc;
    P->lde = (P->me + 3) & ~3;
    P->ldc = (P->mc + 3) & ~3;
    P->s_e64.alloc(se.size());
    P->s_c64.alloc(sc.size());
    h2d(P->s_e64.p, se.data(), se.size(), s);
    h2d(P->s_c64.p, sc.data(), sc.size(), s);
    std::vector<float> sef(se.begin(), se.end()), scf(sc.begin(), sc.end());
    P->s_e.alloc(sef.size());
    P->s_c.alloc(scf.size());
    h2d(P->s_e.p, sef.data(), sef.size(), s);
    h2d(P->s_c.p, scf.data(), scf.size(), s);
    std::vector<float4> se4(P->ne);
    for (int k = 0; k < P->ne; ++k) se4[k] = make_float4((float)se[3 * k], (float)se[3 * k + 1], (float)se[3 * k + 2], 0.f);
    P->s_e4.alloc(P->ne);
    h2d(P->s_e4.p, se4.data(), P->ne, s);

    DBuf<double> Qu1T, Qd1T;
    factor_solve(*P, P->s_c64, RAD_UC, P->s_e64, RAD_UE, Qu1T, P->Ruinv, s);
    factor_solve(*P, P->s_c64, RAD_DC, P->s_e64, RAD_DE, Qd1T, P->Rdinv, s);
    P->Qu1T.alloc((size_t)P->me * P->ldc);
    P->Qd1T.alloc((size_t)P->me * P->ldc);
    P->Qu1T.zero(s);
    P->Qd1T.zero(s);
    to_f32(Qu1T.p, P->Qu1T.p, P->me, P->mc, P->ldc, s);
    to_f32(Qd1T.p, P->Qd1T.p, P->me, P->mc, P->ldc, s);

    // M2M_c = Q_u1^T (1/2 K(uc_P, ue_C)) R_u^-1 (parent half-width 1; child centre o_c)
    // L2L_c = Q_d1^T K(dc_C, de_P) R_d^-1
    std::vector<double> oc, zero8(24, 0.0);
    for (int c = 0; c < 8; ++c) {
        oc.push_back(((c >> 2) & 1) - 0.5);
        oc.push_back(((c >> 1) & 1) - 0.5);
        oc.push_back((c & 1) - 0.5);
    }
    P->M2M.alloc((size_t)8 * P->me * P->lde);
    P->L2L.alloc((size_t)8 * P->me * P->lde);
    P->M2M.zero(s);
    P->L2L.zero(s);
    composites(*P, Qu1T, P->Ruinv, P->s_c64, RAD_UC, P->s_e64, 0.5 * RAD_UE, zero8, oc, 0.5, P->M2M.p, s);
    composites(*P, Qd1T, P->Rdinv, P->s_c64, 0.5 * RAD_DC, P->s_e64, RAD_DE, oc, zero8, 1.0, P->L2L.p, s);

    // M2L_o = Q_d1^T K(dc_B, ue_A) R_u^-1, target box B at the origin, source box A at 2o
    std::vector<double> xo, yo;
    int idx = 0;
    for (int i = 0; i < 343; ++i) P->off_index[i] = -1;
    for (int ox = -3; ox <= 3; ++ox)
        for (int oy = -3; oy <= 3; ++oy)
            for (int oz = -3; oz <= 3; ++oz) {
                if (std::max(std::abs(ox), std::max(std::abs(oy), std::abs(oz))) < 2) continue;
                P->off_index[(ox + 3) * 49 + (oy + 3) * 7 + (oz + 3)] = idx++;
                xo.insert(xo.end(), {0.0, 0.0, 0.0});
                yo.insert(yo.end(), {2.0 * ox, 2.0 * oy, 2.0 * oz});
            }
    P->M2L.alloc((size_t)NV_OFFSETS * P->me * P->lde);
    P->M2L.zero(s);
    composites(*P, Qd1T, P->Ruinv, P->s_c64, RAD_DC, P->s_e64, RAD_UE, xo, yo, 1.0, P->M2L.p, s);

    // exact-TF32 head / remainder splits and TMA maps for the tensor-core path
    auto split = [&](const DBuf<float>& X, int nops, int K, int ld, DBuf<float>& Xb, DBuf<float>& Xs, CUtensorMap* mb,
                     CUtensorMap* ms) {
        Xb.alloc(X.n);
        Xs.alloc(X.n);
        Xb.zero(s);
        Xs.zero(s);
        tc_split_rows(X.p, ld, 0, (int64_t)nops * P->me, K, Xb.p, Xs.p, s);
        tc_make_map_a(mb, Xb.p, nops, P->me, K, ld);
        tc_make_map_a(ms, Xs.p, nops, P->me, K, ld);
    };
    split(P->Qu1T, 1, P->mc, P->ldc, P->Qu1T_b, P->Qu1T_s, &P->mQu1T_b, &P->mQu1T_s);
    split(P->Qd1T, 1, P->mc, P->ldc, P->Qd1T_b, P->Qd1T_s, &P->mQd1T_b, &P->mQd1T_s);
    split(P->M2M, 8, P->me, P->lde, P->M2M_b, P->M2M_s, &P->mM2M_b, &P->mM2M_s);
    split(P->L2L, 8, P->me, P->lde, P->L2L_b, P->L2L_s, &P->mL2L_b, &P->mL2L_s);
    split(P->M2L, NV_OFFSETS, P->me, P->lde, P->M2L_b, P->M2L_s, &P->mM2L_b, &P->mM2L_s);
    // scaled FP16 copies of the M2L / M2M / L2L operators (3xFP16 translations, tc_gemm.cu)
    P->ldh = (P->me + 7) & ~7;
    auto split_h = [&](const DBuf<float>& X, int nops, DBuf<__half>& Xh, DBuf<__half>& Xr, CUtensorMap* mh,
                       CUtensorMap* mr) {
        Xh.alloc((size_t)nops * P->me * P->ldh);
        Xr.alloc((size_t)nops * P->me * P->ldh);
        Xh.zero(s);
        Xr.zero(s);
        const float inv = tc_split_ops_h(X.p, P->lde, (int64_t)nops * P->me, P->me, Xh.p, Xr.p, P->ldh, s);
        tc_make_map_a_h(mh, Xh.p, nops, P->me, P->me, P->ldh);
        tc_make_map_a_h(mr, Xr.p, nops, P->me, P->me, P->ldh);
        return inv;
    };
    P->m2l_hinv = split_h(P->M2L, NV_OFFSETS, P->M2L_hb, P->M2L_hs, &P->mM2L_hb, &P->mM2L_hs);
    P->m2m_hinv = split_h(P->M2M, 8, P->M2M_hb, P->M2M_hs, &P->mM2M_hb, &P->mM2M_hs);
    P->l2l_hinv = split_h(P->L2L, 8, P->L2L_hb, P->L2L_hs, &P->mL2L_hb, &P->mL2L_hs);
    // the upward check-potential rotation Q_u1^T ([me x mc], rows of mc check values)
    P->ldch = (P->mc + 7) & ~7;
    P->Qu1T_hb.alloc((size_t)P->me * P->ldch);
    P->Qu1T_hs.alloc((size_t)P->me * P->ldch);
    P->Qu1T_hb.zero(s);
    P->Qu1T_hs.zero(s);
    P->qu_hinv = tc_split_ops_h(P->Qu1T.p, P->ldc, P->me, P->mc, P->Qu1T_hb.p, P->Qu1T_hs.p, P->ldch, s);
    tc_make_map_a_h(&P->mQu1T_hb, P->Qu1T_hb.p, 1, P->me, P->mc, P->ldch);
    tc_make_map_a_h(&P->mQu1T_hs, P->Qu1T_hs.p, 1, P->me, P->mc, P->ldch);
    EB_CUDA(cudaStreamSynchronize(s));
    return P;
}

std::shared_ptr<Plan> get_plan(int p, const Material& m, cudaStream_t s) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, double, double>, std::shared_ptr<Plan>> cache;
    int dev = 0;
    EB_CUDA(cudaGetDevice(&dev));
    auto key = std::make_tuple(dev, p, m.K, m.G);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    auto P = make_plan(p, m, s);
    cache[key] = P;
    return P;
}

}  // namespace ebem
