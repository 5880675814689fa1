// Leaf-block Jacobi right preconditioner for the BEM GMRES (bem_gmres_solve, precond = 2).
//
// PAPER.md l. 369 names a preconditioner as future work; the paper's own solver is plain
// GMRES (precond = 0).  The 3x3 block-Jacobi of precond = 1 fixes the scaling of the mixed
// unknowns (tractions and displacements) but ignores the strong coupling of neighbouring
// panels.  Here the diagonal block of A over the panels whose collocation points share an
// octree leaf -- at most BMAX panels, consecutive in the sorted target order -- is formed
// exactly as the operator applies it and inverted:
//   A_ij = -sum_q w_q U(x_i, y_q)      (j Dirichlet: the unknown traction)
//   A_ij = +sum_q w_q P(x_i, y_q, n_j)  (j Neumann: the unknown displacement),   i != j,
//   A_ii = -U_self_i or 1/2 I + P_self_i (the local pass, bem.cu),
// with q over the nq quadrature points of panel j (Eq. num, l. 161-187; reading R1 for the
// sign of r).  Entries in fp64, Gauss-Jordan inversion with partial pivoting in fp64, one CTA
// per block; each GMRES iteration applies the inverses as a batched GEMV (a stream over the
// stored inverses, HBM-bound).  The preconditioner changes the Krylov space, not the solution
// (right preconditioning: the residual GMRES drives to tol is the true one).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bem_prec.cuh"
#include "elastic.cuh"

namespace ebem {

namespace {

constexpr int LB_THREADS = 256;
constexpr int LB_NSMEM = 156;              // largest block inverted in shared memory: 156^2 doubles = 190 KB

// A_ij (3x3, row-major into the block at (3 r, 3 c)) for every panel pair of the block
__global__ void lb_assemble(const int4* __restrict__ blocks, const int* __restrict__ trg_perm,
                            const float* __restrict__ cent, const float* __restrict__ qp,
                            const float* __restrict__ qn, const float* __restrict__ qw, int nq,
                            const int32_t* __restrict__ bc, const double* __restrict__ DU,
                            const double* __restrict__ DP, double cU, double a1, double cP, double a,
                            double* __restrict__ M) {
    const int4 bk = blocks[blockIdx.x];
    const int start = bk.x, sz = bk.y;
    const int64_t off = ((int64_t)bk.z << 32) | (uint32_t)bk.w;
    const int ld = 3 * sz;
    double* B = M + off;
    for (int e = threadIdx.x; e < sz * sz; e += blockDim.x) {
        const int r = e / sz, c = e % sz;
        const int i = trg_perm[start + r], j = trg_perm[start + c];
        double blk[3][3];
        const bool dir = bc[j] == 0;
        if (i == j) {
            for (int u = 0; u < 3; ++u)
                for (int v = 0; v < 3; ++v) blk[u][v] = dir ? -DU[9 * (int64_t)i + 3 * u + v] : DP[9 * (int64_t)i + 3 * u + v];
        } else {
            for (int u = 0; u < 3; ++u)
                for (int v = 0; v < 3; ++v) blk[u][v] = 0.0;
            const double x = cent[3 * (int64_t)i], y = cent[3 * (int64_t)i + 1], z = cent[3 * (int64_t)i + 2];
            for (int q = 0; q < nq; ++q) {
                const int64_t k = (int64_t)j * nq + q;
                const double dx = x - qp[3 * k], dy = y - qp[3 * k + 1], dz = z - qp[3 * k + 2];
                const double ri = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
                const double w = qw[k];
                for (int v = 0; v < 3; ++v) {           // column v: the kernel applied to e_v
                    double col[3] = {0.0, 0.0, 0.0};
                    const double ev[3] = {v == 0 ? 1.0 : 0.0, v == 1 ? 1.0 : 0.0, v == 2 ? 1.0 : 0.0};
                    if (dir) {
                        acc_U<double>(dx, dy, dz, ri, cU * w * ev[0], cU * w * ev[1], cU * w * ev[2], a1, col);
                        for (int u = 0; u < 3; ++u) blk[u][v] -= col[u];
                    } else {
                        const double gx = cP * w * ev[0], gy = cP * w * ev[1], gz = cP * w * ev[2];
                        const double nx = qn[3 * k], ny = qn[3 * k + 1], nz = qn[3 * k + 2];
                        const double qq = a * (nx * gx + ny * gy + nz * gz);
                        acc_P<double>(dx, dy, dz, ri, gx, gy, gz, 3.0 * nx, 3.0 * ny, 3.0 * nz, qq, a / 3.0, col);
                        for (int u = 0; u < 3; ++u) blk[u][v] += col[u];
                    }
                }
            }
        }
        for (int u = 0; u < 3; ++u)
            for (int v = 0; v < 3; ++v) B[(int64_t)(3 * r + u) * ld + 3 * c + v] = blk[u][v];
    }
}

// in-place Gauss-Jordan inversion with partial (row) pivoting, fp64, one CTA per block
__global__ void __launch_bounds__(LB_THREADS) lb_invert(const int4* __restrict__ blocks, double* __restrict__ M,
                                                        int* __restrict__ fail) {
    extern __shared__ double sh[];
    const int4 bk = blocks[blockIdx.x];
    const int n = 3 * bk.y;
    if (n <= LB_NSMEM) return;                           // done by lb_invert_smem
    const int64_t off = ((int64_t)bk.z << 32) | (uint32_t)bk.w;
    double* A = M + off;
    double* prow = sh;                                   // pivot row [n]
    double* pcol = sh + n;                               // pivot column [n]
    int* piv = (int*)(sh + 2 * n);                       // row swapped in at step k [n]
    __shared__ double red_v[LB_THREADS];
    __shared__ int red_i[LB_THREADS];
    for (int k = 0; k < n; ++k) {
        // pivot: the largest |A(i, k)|, i >= k
        double best = -1.0;
        int bi = k;
        for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
            const double v = fabs(A[(int64_t)i * n + k]);
            if (v > best) {
                best = v;
                bi = i;
            }
        }
        red_v[threadIdx.x] = best;
        red_i[threadIdx.x] = bi;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) {
                const double o = red_v[threadIdx.x + s];
                const int oi = red_i[threadIdx.x + s];
                if (o > red_v[threadIdx.x] || (o == red_v[threadIdx.x] && oi < red_i[threadIdx.x])) {
                    red_v[threadIdx.x] = o;
                    red_i[threadIdx.x] = oi;
                }
            }
            __syncthreads();
        }
        const int p = red_i[0];
        if (threadIdx.x == 0) {
            piv[k] = p;
            if (!(red_v[0] > 0.0)) atomicExch(fail, 1);
        }
        // swap rows k and p, keep the (new) pivot row and the pivot column
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const double a = A[(int64_t)k * n + j], b = A[(int64_t)p * n + j];
            A[(int64_t)k * n + j] = b;
            A[(int64_t)p * n + j] = a;
            prow[j] = b;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) pcol[i] = A[(int64_t)i * n + k];
        __syncthreads();
        const double d = 1.0 / prow[k];
        // row k := row k / pivot (column k := 1 / pivot); rows i != k: A(i, j) -= A(i, k) row k,
        // column k := -A(i, k) / pivot
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
            const int i = e / n, j = e % n;
            if (i == k) {
                A[(int64_t)i * n + j] = j == k ? d : prow[j] * d;
            } else {
                const double f = pcol[i];
                A[(int64_t)i * n + j] = j == k ? -f * d : A[(int64_t)i * n + j] - f * d * prow[j];
            }
        }
        __syncthreads();
    }
    // undo the row interchanges as column interchanges, last to first
    for (int k = n - 1; k >= 0; --k) {
        const int p = piv[k];
        if (p != k)
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const double a = A[(int64_t)i * n + k];
                A[(int64_t)i * n + k] = A[(int64_t)i * n + p];
                A[(int64_t)i * n + p] = a;
            }
        __syncthreads();
    }
}

// the same in shared memory, for the blocks of NLO < n <= NHI unknowns (a leaf averages ~30
// panels = 90 unknowns on configs[4]): the matrix is read and written once; 128 threads, the
// pivot search by warp shuffles; size classes keep the shared memory (and with it the CTAs
// per SM) proportional to the block
template <int NLO, int NHI, int NT>
__global__ void __launch_bounds__(NT) lb_invert_smem(const int4* __restrict__ blocks, double* __restrict__ M,
                                                     int* __restrict__ fail) {
    constexpr int NW = NT / 32;
    extern __shared__ double sh[];
    const int4 bk = blocks[blockIdx.x];
    const int n = 3 * bk.y;
    if (n <= NLO || n > NHI) return;
    const int64_t off = ((int64_t)bk.z << 32) | (uint32_t)bk.w;
    double* G = M + off;
    double* A = sh;                                      // [n][n + 1] (padded: column reads)
    const int ld = n + 1;
    __shared__ double prow[NHI], pcol[NHI];
    __shared__ int piv[NHI];
    __shared__ double wv[NW];
    __shared__ int wi[NW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) A[(e / n) * ld + e % n] = G[e];
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        double best = -1.0;
        int bi = k;
        for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
            const double v = fabs(A[i * ld + k]);
            if (v > best) {
                best = v;
                bi = i;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) {
                best = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            wv[warp] = best;
            wi[warp] = bi;
        }
        __syncthreads();
        int p = wi[0];
        double pv = wv[0];
        for (int w = 1; w < NW; ++w)
            if (wv[w] > pv || (wv[w] == pv && wi[w] < p)) {
                pv = wv[w];
                p = wi[w];
            }
        if (threadIdx.x == 0) {
            piv[k] = p;
            if (!(pv > 0.0)) atomicExch(fail, 1);
        }
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const double a = A[k * ld + j], b = A[p * ld + j];
            A[k * ld + j] = b;
            A[p * ld + j] = a;
            prow[j] = b;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) pcol[i] = A[i * ld + k];
        __syncthreads();
        const double d = 1.0 / prow[k];
        for (int i = warp; i < n; i += NW) {              // a warp per row
            const double f = pcol[i];
            for (int j = lane; j < n; j += 32) {
                if (i == k) A[i * ld + j] = j == k ? d : prow[j] * d;
                else A[i * ld + j] = j == k ? -f * d : A[i * ld + j] - f * d * prow[j];
            }
        }
        __syncthreads();
    }
    for (int k = n - 1; k >= 0; --k) {
        const int p = piv[k];
        if (p != k)
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const double a = A[i * ld + k];
                A[i * ld + k] = A[i * ld + p];
                A[i * ld + p] = a;
            }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) G[e] = A[(e / n) * ld + e % n];
}

// out[block panels] = Minv_block v[block panels]: a warp per row, lanes along the row
__global__ void __launch_bounds__(LB_THREADS) lb_apply(const int4* __restrict__ blocks, const int* __restrict__ trg_perm,
                                                       const double* __restrict__ M, const double* __restrict__ v,
                                                       double* __restrict__ out) {
    extern __shared__ double sv[];
    const int4 bk = blocks[blockIdx.x];
    const int start = bk.x, sz = bk.y, n = 3 * sz;
    const int64_t off = ((int64_t)bk.z << 32) | (uint32_t)bk.w;
    const double* A = M + off;
    for (int e = threadIdx.x; e < n; e += blockDim.x) sv[e] = v[3 * (int64_t)trg_perm[start + e / 3] + e % 3];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int r = warp; r < n; r += nw) {
        const double* row = A + (int64_t)r * n;
        double s = 0.0;
        for (int j = lane; j < n; j += 32) s = fma(__ldcs(row + j), sv[j], s);   // streamed once per iteration
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[3 * (int64_t)trg_perm[start + r / 3] + r % 3] = s;
    }
}

}  // namespace

bool leafblock_build(const Tree& t, int64_t npanels, int nq, const float* cent, const float* qp, const float* qn,
                     const float* qw, const int32_t* bc, const double* DU, const double* DP, const Material& m,
                     LeafBlockPrec& P, cudaStream_t s) {
    P.release();
    EB_REQUIRE(t.ntrg == npanels, "internal: the BEM tree's targets are the panel centroids");
    static const bool prof = std::getenv("EBEM_BEM_PROFILE") != nullptr;
    auto tick = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!prof) return;
        EB_CUDA(cudaStreamSynchronize(s));
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[bem leaf-block] %-10s %.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tick).count());
        tick = now;
    };
    // blocks: each leaf's sorted targets in runs of at most BMAX panels
    std::vector<int> eb(t.n_eval), tb(t.nboxes), te(t.nboxes);
    if (t.n_eval) d2h(eb.data(), t.eval_box.p, t.n_eval, s);
    d2h(tb.data(), t.tbeg.p, t.nboxes, s);
    d2h(te.data(), t.tend.p, t.nboxes, s);
    EB_CUDA(cudaStreamSynchronize(s));
    std::vector<int4> blk;
    int64_t total = 0;
    int maxn = 0;
    for (int b : eb)
        for (int s0 = tb[b]; s0 < te[b]; s0 += LeafBlockPrec::BMAX) {
            const int sz = std::min(LeafBlockPrec::BMAX, te[b] - s0);
            blk.push_back(make_int4(s0, sz, (int)(total >> 32), (int)(total & 0xffffffffLL)));
            total += (int64_t)(3 * sz) * (3 * sz);
            maxn = std::max(maxn, 3 * sz);
        }
    // memory budget: the inverses must fit beside the solve's other operators
    size_t fr = 0, tt = 0;
    cache_trim();
    EB_CUDA(cudaMemGetInfo(&fr, &tt));
    if ((double)total * 8.0 > 0.5 * (double)fr) return false;
    P.nblocks = (int)blk.size();
    P.maxn = maxn;
    P.entries = total;
    P.blocks.alloc(std::max<size_t>(blk.size(), 1));
    h2d(P.blocks.p, blk.data(), blk.size(), s);
    P.M.alloc(std::max<int64_t>(total, 1));
    if (prof) {
        int c1 = 0, c2 = 0, c3 = 0;
        for (const int4& b : blk) (3 * b.y <= 96 ? c1 : 3 * b.y <= LB_NSMEM ? c2 : c3)++;
        std::fprintf(stderr, "[bem leaf-block] blocks by unknowns: <= 96: %d, <= %d: %d, larger: %d (max %d)\n", c1,
                     LB_NSMEM, c2, c3, maxn);
    }
    lap("tables");
    if (P.nblocks == 0) return true;
    lb_assemble<<<P.nblocks, LB_THREADS, 0, s>>>(P.blocks.p, t.trg_perm.p, cent, qp, qn, qw, nq, bc, DU, DP, m.cU, m.a1,
                                                 m.cP, m.a, P.M.p);
    EB_CHECK_LAUNCH();
    lap("assemble");
    DBuf<int> fail(1);
    fail.zero(s);
    {   // small blocks in shared memory (two size classes), the rest in global memory
        // (the large class runs one CTA per SM: more warps hide the per-step latencies)
        auto run = [&](auto fn, int nhi, int nt) {
            const int ns = std::min(maxn, nhi);
            const size_t sm = (size_t)ns * (ns + 1) * sizeof(double);
            if (sm > 48 * 1024) EB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            fn<<<P.nblocks, nt, sm, s>>>(P.blocks.p, P.M.p, fail.p);
            EB_CHECK_LAUNCH();
        };
        run(lb_invert_smem<0, 96, 256>, 96, 256);
        lap("invert<=96");
        if (maxn > 96) run(lb_invert_smem<96, LB_NSMEM, 512>, LB_NSMEM, 512);
        lap("invert<=156");
    }
    if (maxn > LB_NSMEM) {
        const size_t sm = (size_t)maxn * (2 * sizeof(double) + sizeof(int));
        if (sm > 48 * 1024) EB_CUDA(cudaFuncSetAttribute(lb_invert, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        lb_invert<<<P.nblocks, LB_THREADS, sm, s>>>(P.blocks.p, P.M.p, fail.p);
        EB_CHECK_LAUNCH();
    }
    lap("invert");
    int hf = 0;
    d2h(&hf, fail.p, 1, s);
    EB_CUDA(cudaStreamSynchronize(s));
    if (hf) {                                   // a singular block: use the 3x3 blocks instead
        P.release();
        return false;
    }
    return true;
}

void leafblock_apply(const Tree& t, const LeafBlockPrec& P, const double* v, double* out, cudaStream_t s) {
    if (P.nblocks == 0) return;
    const size_t sm = (size_t)P.maxn * sizeof(double);
    lb_apply<<<P.nblocks, LB_THREADS, sm, s>>>(P.blocks.p, t.trg_perm.p, P.M.p, v, out);
    EB_CHECK_LAUNCH();
}

}  // namespace ebem
