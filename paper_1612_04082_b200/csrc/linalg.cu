// Device primitives: prefix scan, stable LSD radix sort, fp64 batched GEMM and the
// operator-grouped "pairs" GEMMs that apply the KIFMM translation operators.
#include <algorithm>

#include "fmm.cuh"

namespace ebem {

// ================================================================== scan
constexpr int SCAN_T = 256, SCAN_ITEMS = 8, SCAN_TILE = SCAN_T * SCAN_ITEMS;

__device__ __forceinline__ int block_exclusive_scan(int v, int* sh, int& total) {
    // sh: SCAN_T/32 ints
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int w = lane < SCAN_T / 32 ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < SCAN_T / 32) sh[lane] = w;
    }
    __syncthreads();
    int wprefix = wid ? sh[wid - 1] : 0;
    total = sh[SCAN_T / 32 - 1];
    __syncthreads();
    return wprefix + x - v;
}

__global__ void scan_tiles(const int* __restrict__ in, int* __restrict__ out, int64_t n,
                           int* __restrict__ tile_sums) {
    __shared__ int sh[SCAN_T / 32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int v[SCAN_ITEMS], s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        s += v[i];
    }
    int total;
    int ex = block_exclusive_scan(s, sh, total);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = ex;
        ex += v[i];
    }
    if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = total;
}

__global__ void scan_add(int* __restrict__ out, int64_t n, const int* __restrict__ offs) {
    int64_t i = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x;
    int add = offs[blockIdx.x];
    for (int k = 0; k < SCAN_ITEMS; ++k, i += SCAN_T)
        if (i < n) out[i] += add;
}

static void scan_rec(const int* in, int* out, int64_t n, cudaStream_t s) {
    const int nt = ceil_div(n, SCAN_TILE);
    if (nt == 1) {
        scan_tiles<<<1, SCAN_T, 0, s>>>(in, out, n, nullptr);
        EB_CHECK_LAUNCH();
        return;
    }
    int* sums = nullptr;
    EB_CUDA(cudaMallocAsync(&sums, sizeof(int) * nt, s));
    scan_tiles<<<nt, SCAN_T, 0, s>>>(in, out, n, sums);
    EB_CHECK_LAUNCH();
    scan_rec(sums, sums, nt, s);
    scan_add<<<nt, SCAN_T, 0, s>>>(out, n, sums);
    EB_CHECK_LAUNCH();
    EB_CUDA(cudaFreeAsync(sums, s));
}

int64_t exclusive_scan_i32(const int* in, int* out, int64_t n, cudaStream_t s) {
    if (n == 0) return 0;
    int last_in = 0, last_out = 0;
    EB_CUDA(cudaMemcpyAsync(&last_in, in + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    scan_rec(in, out, n, s);
    EB_CUDA(cudaMemcpyAsync(&last_out, out + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    EB_CUDA(cudaStreamSynchronize(s));
    return (int64_t)last_in + last_out;
}

// ================================================================== radix sort
// Stable LSD radix sort, 8-bit digits.  Per pass: (1) per-tile digit histograms,
// digit-major [256][ntiles]; (2) exclusive scan of that array -> global offsets;
// (3) stable scatter: tiles are processed 256 keys at a time in warp order, each key's
// rank among equal digits in its warp comes from __match_any_sync, and per-digit
// running counts are carried across warps and iterations in shared memory.
constexpr int RS_T = 256, RS_ITEMS = 8, RS_TILE = RS_T * RS_ITEMS, RS_WARPS = RS_T / 32;

__global__ void rs_hist(const long long* __restrict__ keys, int64_t n, int shift, int ntiles,
                        int* __restrict__ hist) {
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    for (int i = threadIdx.x; i < RS_TILE; i += RS_T) {
        int64_t k = base + i;
        if (k < n) atomicAdd(&h[(keys[k] >> shift) & 255], 1);
    }
    __syncthreads();
    hist[threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void rs_scatter(const long long* __restrict__ kin, const int* __restrict__ vin,
                           long long* __restrict__ kout, int* __restrict__ vout, int64_t n,
                           int shift, int ntiles, const int* __restrict__ offs) {
    __shared__ int base_d[256];
    __shared__ int running[256];
    __shared__ int wcount[RS_WARPS][256];
    __shared__ int woff[RS_WARPS][256];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    base_d[threadIdx.x] = offs[threadIdx.x * ntiles + blockIdx.x];
    running[threadIdx.x] = 0;
    for (int w = 0; w < RS_WARPS; ++w) wcount[w][threadIdx.x] = 0;
    __syncthreads();
    const int64_t tbase = (int64_t)blockIdx.x * RS_TILE;
    for (int it = 0; it < RS_ITEMS; ++it) {
        const int64_t i = tbase + (int64_t)it * RS_T + threadIdx.x;   // warp-contiguous, in order
        const bool valid = i < n;
        long long key = valid ? kin[i] : 0;
        int val = valid ? vin[i] : 0;
        int d = valid ? (int)((key >> shift) & 255) : 256 + lane;   // invalid lanes never match
        unsigned peers = __match_any_sync(0xffffffffu, d);
        int rank = __popc(peers & ((1u << lane) - 1u));
        if (valid && rank == 0) wcount[wid][d] = __popc(peers);
        __syncthreads();
        {
            int t = threadIdx.x, run = running[t];
            for (int w = 0; w < RS_WARPS; ++w) {
                woff[w][t] = run;
                run += wcount[w][t];
                wcount[w][t] = 0;
            }
            running[t] = run;
        }
        __syncthreads();
        if (valid) {
            int pos = base_d[d] + woff[wid][d] + rank;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
    }
}

void radix_sort_pairs(long long* keys, int* vals, int64_t n, int bits, cudaStream_t s) {
    if (n <= 1) return;
    const int ntiles = ceil_div(n, RS_TILE);
    long long* k2 = nullptr;
    int *v2 = nullptr, *hist = nullptr;
    EB_CUDA(cudaMallocAsync(&k2, sizeof(long long) * n, s));
    EB_CUDA(cudaMallocAsync(&v2, sizeof(int) * n, s));
    EB_CUDA(cudaMallocAsync(&hist, sizeof(int) * 256 * ntiles, s));
    long long *ka = keys, *kb = k2;
    int *va = vals, *vb = v2;
    int passes = 0;
    for (int shift = 0; shift < bits; shift += 8, ++passes) {
        rs_hist<<<ntiles, RS_T, 0, s>>>(ka, n, shift, ntiles, hist);
        EB_CHECK_LAUNCH();
        scan_rec(hist, hist, (int64_t)256 * ntiles, s);
        rs_scatter<<<ntiles, RS_T, 0, s>>>(ka, va, kb, vb, n, shift, ntiles, hist);
        EB_CHECK_LAUNCH();
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (passes & 1) {
        d2d(keys, ka, n, s);
        d2d(vals, va, n, s);
    }
    EB_CUDA(cudaFreeAsync(k2, s));
    EB_CUDA(cudaFreeAsync(v2, s));
    EB_CUDA(cudaFreeAsync(hist, s));
}

// ================================================================== fp64 GEMM
// 64x64 output tile per 256-thread CTA, 4x4 per thread, k-tile 16 (plan precompute only).
__global__ void __launch_bounds__(256)
gemm_f64_kernel(int m, int n, int k, double alpha, const double* __restrict__ A, int64_t sA, int lda,
                const double* __restrict__ B, int64_t sB, int ldb, double beta, double* __restrict__ C,
                int64_t sC, int ldc) {
    __shared__ double As[16][64 + 1];
    __shared__ double Bs[16][64 + 1];
    A += blockIdx.z * sA;
    B += blockIdx.z * sB;
    C += blockIdx.z * sC;
    const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < k; k0 += 16) {
        for (int e = threadIdx.x; e < 16 * 64; e += 256) {
            int r = e / 16, c = e % 16;          // A: row r (m), col c (k)
            int gm = m0 + r, gk = k0 + c;
            As[c][r] = (gm < m && gk < k) ? A[(int64_t)gm * lda + gk] : 0.0;
            int rb = e / 64, cb = e % 64;        // B: row rb (k), col cb (n)
            int gk2 = k0 + rb, gn = n0 + cb;
            Bs[rb][cb] = (gk2 < k && gn < n) ? B[(int64_t)gk2 * ldb + gn] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
            if (gm < m && gn < n) {
                double* c = C + (int64_t)gm * ldc + gn;
                *c = alpha * acc[i][j] + (beta != 0.0 ? beta * *c : 0.0);
            }
        }
}

void gemm_f64(int m, int n, int k, double alpha, const double* A, int64_t sA, int lda,
              const double* B, int64_t sB, int ldb, double beta, double* C, int64_t sC, int ldc,
              int batch, cudaStream_t s) {
    dim3 grid(ceil_div(n, 64), ceil_div(m, 64), batch);
    gemm_f64_kernel<<<grid, 256, 0, s>>>(m, n, k, alpha, A, sA, lda, B, sB, ldb, beta, C, sC, ldc);
    EB_CHECK_LAUNCH();
}

// ================================================================== pairs GEMM
// Tile table entry: (op, first pair, count <= 64).
void build_op_pairs(OpPairs& P, int nops, const std::vector<int>& op, const std::vector<int2>& pr,
                    cudaStream_t s) {
    P.nops = nops;
    P.npairs = (int64_t)pr.size();
    std::vector<int> cnt(nops + 1, 0);
    for (int o : op) cnt[o + 1]++;
    for (int i = 0; i < nops; ++i) cnt[i + 1] += cnt[i];
    std::vector<int2> sorted(pr.size());
    std::vector<int> cur(cnt.begin(), cnt.end() - 1);
    for (size_t i = 0; i < pr.size(); ++i) sorted[cur[op[i]]++] = pr[i];
    P.op_ptr_h = cnt;
    P.max_per_op = 0;
    for (int i = 0; i < nops; ++i) P.max_per_op = std::max(P.max_per_op, cnt[i + 1] - cnt[i]);
    P.op_ptr.alloc(nops + 1);
    h2d(P.op_ptr.p, cnt.data(), nops + 1, s);
    P.pairs.alloc(std::max<size_t>(sorted.size(), 1));
    h2d(P.pairs.p, sorted.data(), sorted.size(), s);
    EB_CUDA(cudaStreamSynchronize(s));
}

constexpr int PG_M = 64, PG_N = 64, PG_K = 16;

// Y[t] += Mat[op] X[src] for the 64 pairs of one tile: 64 rows of Mat x 64 pairs.
// Accumulates with atomicAdd (one pair per target per op, but different ops of the same
// target land on the same rows).
template <class XT>
__global__ void __launch_bounds__(256)
gemm_pairs_f32_kernel(const int* __restrict__ op_ptr, const int2* __restrict__ pairs, int nops,
                      const float* __restrict__ mats, int M, int K, int ldm, const XT* __restrict__ X,
                      int ldx, double* __restrict__ Y, int ldy) {
    const int op = blockIdx.z;
    const int p0 = op_ptr[op] + blockIdx.y * PG_N;
    const int p1 = op_ptr[op + 1];
    if (p0 >= p1) return;
    const int np = min(PG_N, p1 - p0);
    const int m0 = blockIdx.x * PG_M;
    const float* Mt = mats + (int64_t)op * M * ldm;
    __shared__ float As[PG_K][PG_M + 4];
    __shared__ float Bs[PG_K][PG_N + 4];
    __shared__ int2 pr[PG_N];
    if (threadIdx.x < PG_N) pr[threadIdx.x] = threadIdx.x < np ? pairs[p0 + threadIdx.x] : make_int2(-1, -1);
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += PG_K) {
        for (int e = threadIdx.x; e < PG_K * PG_M; e += 256) {
            int r = e / PG_K, c = e % PG_K;
            int gm = m0 + r, gk = k0 + c;
            As[c][r] = (gm < M && gk < K) ? Mt[(int64_t)gm * ldm + gk] : 0.f;
            int j = e / PG_K;                      // pair j, k offset c
            int src = pr[j].y;
            Bs[c][j] = (src >= 0 && gk < K) ? (float)X[(int64_t)src * ldx + gk] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < PG_K; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        int pj = tx + 16 * j;
        if (pj >= np) continue;
        double* y = Y + (int64_t)pr[pj].x * ldy;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int gm = m0 + ty + 16 * i;
            if (gm < M) atomicAdd(y + gm, (double)acc[i][j]);
        }
    }
}

template <class XT>
void gemm_pairs_f32(const OpPairs& P, const float* mats, int M, int K, int ldm, const XT* X, int ldx,
                    double* Y, int ldy, cudaStream_t s) {
    if (P.npairs == 0) return;
    dim3 grid(ceil_div(M, PG_M), ceil_div(P.max_per_op, PG_N), P.nops);
    gemm_pairs_f32_kernel<XT><<<grid, 256, 0, s>>>(P.op_ptr.p, P.pairs.p, P.nops, mats, M, K, ldm, X, ldx, Y, ldy);
    EB_CHECK_LAUNCH();
}
template void gemm_pairs_f32<float>(const OpPairs&, const float*, int, int, int, const float*, int, double*, int,
                                    cudaStream_t);
template void gemm_pairs_f32<double>(const OpPairs&, const float*, int, int, int, const double*, int, double*, int,
                                     cudaStream_t);

// fp64: Y[t] = scale[t] * Mat X[src] (one op; plain store; Mat upper triangular).
// OutT = double: Y row-major [t][ldy].  OutT = float4: the fp32 far-field layout, row t holds
// M/3 float4 (x, y, z, 0) = (float)(cf * scale[t] * (Mat X)[3k .. 3k+2]) (ldy in float4).
// Computed on the fp64 tensor cores (mma.sync m8n8k4 f64; measured 37 TFLOP/s on B200, the
// FP64 FMA peak): a SIMT version (4 x 4 register tiles) was bound by shared-memory loads (8 LDS per
// 16 DFMA) at ~41% of the FP64 pipe.  CTA tile 64 rows x 64 pairs, K step 16 double-buffered
// in smem (row stride 20 doubles: conflict-free fragment loads); 8 warps of 32 x 16 outputs
// (4 x 2 mma tiles, 6 fragment loads per 8 MMAs).
constexpr int DM_M = 64, DM_N = 64, DM_K = 16, DM_LD = 20;
template <class OutT>
__global__ void __launch_bounds__(256)
gemm_pairs_dmma_kernel(const int2* __restrict__ pairs, int npairs, const double* __restrict__ Mt, int M, int K,
                       const double* __restrict__ X, int ldx, const double* __restrict__ scale, double cf,
                       OutT* __restrict__ Y, int ldy) {
    const int p0 = blockIdx.y * DM_N;
    const int np = min(DM_N, npairs - p0);
    const int m0 = blockIdx.x * DM_M;
    __shared__ __align__(16) double As[2][DM_M * DM_LD];
    __shared__ __align__(16) double Bs[2][DM_N * DM_LD];
    __shared__ int2 pr[DM_N];
    if (threadIdx.x < DM_N) pr[threadIdx.x] = threadIdx.x < np ? pairs[p0 + threadIdx.x] : make_int2(-1, -1);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp >> 2, wn = warp & 3;                 // 2 x 4 warps: 32 rows x 16 pairs each
    // loader: row r = threadIdx / 4 (0..63), 4 consecutive doubles (2 x double2) at k = 4 (tid % 4)
    const int lr = threadIdx.x >> 2, lk = 4 * (threadIdx.x & 3);
    double2 la[2], lb[2];
    auto load = [&](int k0) {
        const int gm = m0 + lr, src = pr[lr].y;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gk = k0 + lk + 2 * h;
            la[h] = make_double2(gm < M && gk < K ? Mt[(int64_t)gm * K + gk] : 0.0,
                                 gm < M && gk + 1 < K ? Mt[(int64_t)gm * K + gk + 1] : 0.0);
            lb[h] = make_double2(src >= 0 && gk < K ? X[(int64_t)src * ldx + gk] : 0.0,
                                 src >= 0 && gk + 1 < K ? X[(int64_t)src * ldx + gk + 1] : 0.0);
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            *reinterpret_cast<double2*>(&As[buf][lr * DM_LD + lk + 2 * h]) = la[h];
            *reinterpret_cast<double2*>(&Bs[buf][lr * DM_LD + lk + 2 * h]) = lb[h];
        }
    };
    double c[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) c[i][j][0] = c[i][j][1] = 0.0;
    int k0 = (m0 / DM_K) * DM_K;                              // R^-1 is upper triangular
    load(k0);
    store(0);
    __syncthreads();
    int buf = 0;
    const int fr = lane >> 2, fk = lane & 3;                  // fragment row / k of this lane
    for (; k0 < K; k0 += DM_K) {
        const bool more = k0 + DM_K < K;
        if (more) load(k0 + DM_K);
#pragma unroll
        for (int kk = 0; kk < DM_K; kk += 4) {
            double a[4], b[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[buf][(wm * 32 + i * 8 + fr) * DM_LD + kk + fk];
#pragma unroll
            for (int j = 0; j < 2; ++j) b[j] = Bs[buf][(wn * 16 + j * 8 + fr) * DM_LD + kk + fk];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(c[i][j][0]), "+d"(c[i][j][1])
                                 : "d"(a[i]), "d"(b[j]));
        }
        if (more) {
            store(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
    // C fragment: row fr of the 8 x 8 tile, columns 2 (lane % 4) + {0, 1}
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int pj = wn * 16 + j * 8 + 2 * fk + e;
            if (pj >= np) continue;
            const int t = pr[pj].x;
            const double sc = scale[t];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int gm = m0 + wm * 32 + i * 8 + fr;
                if (gm >= M) continue;
                if constexpr (sizeof(OutT) == sizeof(double)) {
                    Y[(int64_t)t * ldy + gm] = sc * c[i][j][e];
                } else {
                    float* y = reinterpret_cast<float*>(Y + (int64_t)t * ldy);
                    y[4 * (gm / 3) + gm % 3] = (float)(cf * sc * c[i][j][e]);
                }
            }
        }
}

void gemm_pairs_f64(const OpPairs& P, const double* mat, int M, int K, const double* X, int ldx,
                    const double* scale, double* Y, int ldy, cudaStream_t s) {
    if (P.npairs == 0) return;
    dim3 grid(ceil_div(M, DM_M), ceil_div(P.npairs, DM_N), 1);
    gemm_pairs_dmma_kernel<double><<<grid, 256, 0, s>>>(P.pairs.p, (int)P.npairs, mat, M, K, X, ldx, scale, 1.0, Y,
                                                       ldy);
    EB_CHECK_LAUNCH();
}

void gemm_pairs_f64_to_f32(const OpPairs& P, const double* mat, int M, int K, const double* X, int ldx,
                           const double* scale, double cf, float4* Y, int ldy, cudaStream_t s) {
    if (P.npairs == 0) return;
    dim3 grid(ceil_div(M, DM_M), ceil_div(P.npairs, DM_N), 1);
    gemm_pairs_dmma_kernel<float4><<<grid, 256, 0, s>>>(P.pairs.p, (int)P.npairs, mat, M, K, X, ldx, scale, cf, Y,
                                                       ldy);
    EB_CHECK_LAUNCH();
}

}  // namespace ebem
