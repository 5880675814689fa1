// O(N^2) direct sum on the GPU: bem_kernel_direct.  PAPER.md Sec. 2.2 line 125 ("an
// iterative solution scheme would require O(N^2) operations") and Eq. fmm_summation.
//
// Layout: prepared source records (p2p.cuh) are streamed through shared memory in
// tiles of 128; each thread owns TPT targets in registers and does fp32 FFMA with one
// rsqrt per pair.  A one-wave persistent grid splits the (target block, source tile)
// units evenly over all resident CTA slots; partial sums of a target block from the CTAs
// that covered it are reduced in a fixed order (deterministic).
#include <cstdlib>

#include "p2p.cuh"

namespace ebem {

__global__ void prepare_kernel(int kernel, float cU, float cP, float cD, float cS, float a, float b4,
                               const float* __restrict__ y, const float* __restrict__ nrm,
                               const float* __restrict__ w, const float* __restrict__ f,
                               const float* __restrict__ g, const int* __restrict__ gperm,
                               const int* __restrict__ dperm, int64_t n, float4* __restrict__ rec) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t o = gperm ? gperm[i] : i;       // geometry index
    int64_t q = dperm ? dperm[i] : i;       // density index
    const bool sl = (kernel == K_U || kernel == K_UP || kernel == K_D || kernel == K_DS);
    const bool dl = (kernel == K_P || kernel == K_UP || kernel == K_S || kernel == K_DS);
    const bool st = kernel >= K_D;
    float ww = w ? w[o] : 1.0f;
    float px = y[3 * o], py = y[3 * o + 1], pz = y[3 * o + 2];
    float cf = st ? cD : cU, cg = st ? cS : cP;
    float fx = 0, fy = 0, fz = 0, gx = 0, gy = 0, gz = 0, nx = 0, ny = 0, nz = 0;
    if (sl) { fx = cf * ww * f[3 * q]; fy = cf * ww * f[3 * q + 1]; fz = cf * ww * f[3 * q + 2]; }
    if (dl) {
        gx = cg * ww * g[3 * q]; gy = cg * ww * g[3 * q + 1]; gz = cg * ww * g[3 * q + 2];
        nx = nrm[3 * o]; ny = nrm[3 * o + 1]; nz = nrm[3 * o + 2];
    }
    float ng = nx * gx + ny * gy + nz * gz;
    if (st && sl && dl) {    // acc_DS record (elastic.cuh): a-scaled f, the per-source constants
        float4* r = rec + i * REC_STRESS;
        r[0] = make_float4(px, py, pz, 1.5f * a * ng);
        r[1] = make_float4(a * fx, a * fy, a * fz, -0.5f * b4 * ng);
        r[2] = make_float4(gx, gy, gz, 0.f);
        r[3] = make_float4(nx, ny, nz, 0.f);
        r[4] = make_float4(a * nx * gx, a * ny * gy, a * nz * gz, a * (nx * gy + ny * gx));
        r[5] = make_float4(a * (ny * gz + nz * gy), a * (nx * gz + nz * gx), 0.f, 0.f);
        return;
    }
    if (!st) {
        float4* r = rec + i * REC_DISP;
        r[0] = make_float4(px, py, pz, a * ng);
        r[1] = make_float4(fx, fy, fz, 0.f);
        r[2] = make_float4(gx, gy, gz, 0.f);
        r[3] = make_float4(3.f * nx, 3.f * ny, 3.f * nz, 0.f);
    } else {
        float4* r = rec + i * REC_STRESS;
        r[0] = make_float4(px, py, pz, ng);
        r[1] = make_float4(fx, fy, fz, 0.f);
        r[2] = make_float4(gx, gy, gz, 0.f);
        r[3] = make_float4(nx, ny, nz, 0.f);
        r[4] = make_float4(2 * a * nx * gx, 2 * a * ny * gy, 2 * a * nz * gz, a * (nx * gy + ny * gx));
        r[5] = make_float4(a * (ny * gz + nz * gy), a * (nx * gz + nz * gx), 0.f, 0.f);
    }
}

void prepare_sources(int kernel, const Material& m, const float* y, const float* nrm,
                     const float* w, const int* gperm, const float* f, const float* g,
                     const int* dperm, int64_t n, float4* rec, cudaStream_t s) {
    if (n == 0) return;
    prepare_kernel<<<ceil_div(n, 256), 256, 0, s>>>(kernel, (float)m.cU, (float)m.cP, (float)m.cD,
                                                    (float)m.cS, (float)m.a, (float)m.b4, y, nrm, w, f, g, gperm,
                                                    dperm, n, rec);
    EB_CHECK_LAUNCH();
}

constexpr int DIRECT_THREADS = 128;
constexpr int DIRECT_TPT = 4;          // targets per thread (measured best of 3..8)
#ifndef EBEM_DIRECT_TILE
#define EBEM_DIRECT_TILE 64      // 64: configs[1] 50.3% of FP32 peak, 128: 49.9%, 256: 48.2%
#endif
constexpr int DIRECT_TILE = EBEM_DIRECT_TILE;   // sources per shared-memory tile
constexpr int DIRECT_TB = DIRECT_THREADS * DIRECT_TPT;   // targets per target block

// Work = (target block, source tile) units, target-block major.  The grid is exactly the
// resident CTA slots of one wave and CTA c takes the contiguous unit range
// [c U / G, (c+1) U / G): every SM gets the same number of pair interactions to within one
// tile (a 2-D grid of whole source chunks left 14% of the slots idle on configs[1]).
// A CTA flushes its accumulators whenever its range leaves a target block, into slot
// (c - first CTA of that block) of that block's partial sums; reduce_blocks adds the slots
// of each target in a fixed order (deterministic).
__device__ __forceinline__ int64_t first_cta(int64_t u, int64_t U, int64_t G) {
    return ((u + 1) * G + U - 1) / U - 1;          // CTA whose range contains unit u
}

#ifndef EBEM_PACKED
#define EBEM_PACKED 1        // packed FFMA2 pair loop (two targets per instruction)
#endif

template <bool SL, bool DL, bool STRESS>
__global__ void __launch_bounds__(DIRECT_THREADS)
direct_kernel(const float4* __restrict__ rec, int64_t nsrc, int64_t ntiles, const float* __restrict__ trg,
              int64_t ntrg, int64_t U, int kslots, KConst kc, float* __restrict__ partial) {
    constexpr int R = STRESS ? REC_STRESS : REC_DISP;
    constexpr int NC = STRESS ? 6 : 3;
    constexpr int NP = DIRECT_TPT / 2;
    __shared__ float4 srec[DIRECT_TILE * R];
    const int64_t G = gridDim.x, c = blockIdx.x;
    const int64_t u_beg = c * U / G, u_end = (c + 1) * U / G;
#if EBEM_PACKED
    const KConst2 kc2(kc);
#endif
    int64_t u = u_beg;
    while (u < u_end) {
        const int64_t tb = u / ntiles;
        const int64_t u_stop = min(u_end, (tb + 1) * ntiles);
        const int64_t t0 = tb * DIRECT_TB + threadIdx.x;
        float x[DIRECT_TPT], y[DIRECT_TPT], z[DIRECT_TPT], acc[DIRECT_TPT][NC];
#pragma unroll
        for (int k = 0; k < DIRECT_TPT; ++k) {
            const int64_t t = t0 + k * DIRECT_THREADS;
            const int64_t tc = t < ntrg ? t : ntrg - 1;
            x[k] = trg[3 * tc]; y[k] = trg[3 * tc + 1]; z[k] = trg[3 * tc + 2];
#pragma unroll
            for (int q = 0; q < NC; ++q) acc[k][q] = 0.f;
        }
#if EBEM_PACKED
        F2 x2[NP], y2[NP], z2[NP], acc2[NP][NC];
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            x2[k] = F2(x[2 * k], x[2 * k + 1]);
            y2[k] = F2(y[2 * k], y[2 * k + 1]);
            z2[k] = F2(z[2 * k], z[2 * k + 1]);
#pragma unroll
            for (int q = 0; q < NC; ++q) acc2[k][q] = F2(0.f);
        }
#endif
        for (; u < u_stop; ++u) {
            const int64_t s0 = (u - tb * ntiles) * DIRECT_TILE;
            const int cnt = (int)min((int64_t)DIRECT_TILE, nsrc - s0);
            __syncthreads();
            for (int i = threadIdx.x; i < cnt * R; i += DIRECT_THREADS) srec[i] = rec[s0 * R + i];
            __syncthreads();
#if EBEM_PACKED
            pair_loop_packed<SL, DL, STRESS, NP, R, true, PL_UNROLL>(srec, cnt, 0, 1, x2, y2, z2, kc2, acc2);
#else
            pair_loop_multi<SL, DL, STRESS, DIRECT_TPT>(srec, cnt, x, y, z, kc, acc);
#endif
        }
#if EBEM_PACKED
#pragma unroll
        for (int k = 0; k < NP; ++k)
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                acc[2 * k][q] = acc2[k][q].v.x;
                acc[2 * k + 1][q] = acc2[k][q].v.y;
            }
#endif
        const int slot = (int)(c - first_cta(tb * ntiles, U, G));
        float* o = partial + ((int64_t)tb * kslots + slot) * DIRECT_TB * NC;
        if (STRESS && SL && DL)   // acc_DS accumulates half of the diagonal
#pragma unroll
            for (int k = 0; k < DIRECT_TPT; ++k)
#pragma unroll
                for (int q = 0; q < 3; ++q) acc[k][q] *= 2.f;
#pragma unroll
        for (int k = 0; k < DIRECT_TPT; ++k)
#pragma unroll
            for (int q = 0; q < NC; ++q) o[(threadIdx.x + k * DIRECT_THREADS) * NC + q] = acc[k][q];
    }
}

// out[t] = sum over the CTAs that covered t's target block, in CTA order
__global__ void reduce_blocks(const float* __restrict__ partial, int64_t ntrg, int nc, int64_t ntiles, int64_t U,
                              int64_t G, int kslots, float* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ntrg * nc) return;
    const int64_t t = i / nc, q = i % nc, tb = t / DIRECT_TB, r = t % DIRECT_TB;
    const int64_t c0 = first_cta(tb * ntiles, U, G), c1 = first_cta((tb + 1) * ntiles - 1, U, G);
    const float* p = partial + (int64_t)tb * kslots * DIRECT_TB * nc + r * nc + q;
    float sum = 0.f;
    for (int64_t k = 0; k <= c1 - c0; ++k) sum += p[k * DIRECT_TB * nc];
    out[i] = sum;
}

template <bool SL, bool DL, bool STRESS>
static void launch_direct(const float4* rec, int64_t nsrc, const float* trg, int64_t ntrg,
                          const KConst& kc, float* out, cudaStream_t s) {
    constexpr int NC = STRESS ? 6 : 3;
    const int64_t tblocks = (ntrg + DIRECT_TB - 1) / DIRECT_TB;
    const int64_t ntiles = (nsrc + DIRECT_TILE - 1) / DIRECT_TILE;
    const int64_t U = tblocks * ntiles;
    int occ = 0;
    EB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, direct_kernel<SL, DL, STRESS>, DIRECT_THREADS, 0));
    int64_t G = std::min<int64_t>(U, (int64_t)num_sms() * std::max(occ, 1));
    if (const char* e = std::getenv("EBEM_DIRECT_GRID")) G = std::max<int64_t>(1, std::min<int64_t>(U, std::atoll(e)));
    // CTAs per target block: at most ceil(ntiles / floor(U / G)) + 1
    const int64_t per = std::max<int64_t>(1, U / G);
    const int kslots = (int)std::min<int64_t>(G, (ntiles + per - 1) / per + 1);
    float* partial = nullptr;
    EB_CUDA(cudaMallocAsync(&partial, sizeof(float) * tblocks * kslots * DIRECT_TB * NC, s));
    direct_kernel<SL, DL, STRESS><<<(unsigned)G, DIRECT_THREADS, 0, s>>>(rec, nsrc, ntiles, trg, ntrg, U, kslots, kc,
                                                                         partial);
    EB_CHECK_LAUNCH();
    reduce_blocks<<<(unsigned)ceil_div(ntrg * NC, 256), 256, 0, s>>>(partial, ntrg, NC, ntiles, U, G, kslots, out);
    EB_CHECK_LAUNCH();
    EB_CUDA(cudaFreeAsync(partial, s));
}

// device-pointer entry (all pointers on the device)
void direct_sum_device(int kernel, const Material& m, const float* trg, int64_t ntrg,
                       const float* src, const float* nrm, const float* w, const float* f,
                       const float* g, int64_t nsrc, float* out, cudaStream_t s) {
    const int nc = kernel_ncomp(kernel);
    if (ntrg == 0) return;
    if (nsrc == 0) {
        EB_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * ntrg * nc, s));
        return;
    }
    const int R = kernel_stress(kernel) ? REC_STRESS : REC_DISP;
    float4* rec = nullptr;
    EB_CUDA(cudaMallocAsync(&rec, sizeof(float4) * R * nsrc, s));
    prepare_sources(kernel, m, src, nrm, w, nullptr, f, g, nullptr, nsrc, rec, s);
    KConst kc = make_kconst(m);
    switch (kernel) {
        case K_U: launch_direct<true, false, false>(rec, nsrc, trg, ntrg, kc, out, s); break;
        case K_P: launch_direct<false, true, false>(rec, nsrc, trg, ntrg, kc, out, s); break;
        case K_UP: launch_direct<true, true, false>(rec, nsrc, trg, ntrg, kc, out, s); break;
        case K_D: launch_direct<true, false, true>(rec, nsrc, trg, ntrg, kc, out, s); break;
        case K_S: launch_direct<false, true, true>(rec, nsrc, trg, ntrg, kc, out, s); break;
        case K_DS: launch_direct<true, true, true>(rec, nsrc, trg, ntrg, kc, out, s); break;
        default: throw Error("bem_kernel_direct: unknown kernel id");
    }
    EB_CUDA(cudaFreeAsync(rec, s));
}

}  // namespace ebem
