// O(N^2) direct sum on the GPU: bem_kernel_direct.  PAPER.md Sec. 2.2 line 125 ("an
// iterative solution scheme would require O(N^2) operations") and Eq. fmm_summation.
//
// Layout: prepared source records (p2p.cuh) are streamed through shared memory in
// tiles of 128; each thread owns TPT targets in registers and does fp32 FFMA with one
// rsqrt per pair.  The source range is split across blockIdx.y so the grid covers all
// 148 SMs even for a few thousand targets; partial sums land in a [split][target][c]
// scratch and a second kernel reduces them in a fixed order (deterministic).
#include <cstdlib>

#include "p2p.cuh"

namespace ebem {

__global__ void prepare_kernel(int kernel, float cU, float cP, float cD, float cS, float a,
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
                                                    (float)m.cS, (float)m.a, y, nrm, w, f, g, gperm,
                                                    dperm, n, rec);
    EB_CHECK_LAUNCH();
}

constexpr int DIRECT_THREADS = 128;
constexpr int DIRECT_TPT = 4;          // targets per thread (one LDS.128 per pair)
constexpr int DIRECT_TILE = 128;       // sources per shared-memory tile

template <bool SL, bool DL, bool STRESS>
__global__ void __launch_bounds__(DIRECT_THREADS)
direct_kernel(const float4* __restrict__ rec, int64_t nsrc, int64_t chunk,
              const float* __restrict__ trg, int64_t ntrg, KConst kc, float* __restrict__ partial) {
    constexpr int R = STRESS ? REC_STRESS : REC_DISP;
    constexpr int NC = STRESS ? 6 : 3;
    __shared__ float4 srec[DIRECT_TILE * R];
    const int64_t t0 = (int64_t)blockIdx.x * DIRECT_THREADS * DIRECT_TPT + threadIdx.x;
    float x[DIRECT_TPT], y[DIRECT_TPT], z[DIRECT_TPT], acc[DIRECT_TPT][NC];
#pragma unroll
    for (int k = 0; k < DIRECT_TPT; ++k) {
        int64_t t = t0 + k * DIRECT_THREADS;
        int64_t tc = t < ntrg ? t : ntrg - 1;
        x[k] = trg[3 * tc]; y[k] = trg[3 * tc + 1]; z[k] = trg[3 * tc + 2];
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[k][c] = 0.f;
    }
    const int64_t s_begin = blockIdx.y * chunk;
    const int64_t s_end = min(nsrc, s_begin + chunk);
    for (int64_t s0 = s_begin; s0 < s_end; s0 += DIRECT_TILE) {
        const int cnt = (int)min((int64_t)DIRECT_TILE, s_end - s0);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt * R; i += DIRECT_THREADS) srec[i] = rec[s0 * R + i];
        __syncthreads();
        pair_loop_multi<SL, DL, STRESS, DIRECT_TPT>(srec, cnt, x, y, z, kc, acc);
    }
#pragma unroll
    for (int k = 0; k < DIRECT_TPT; ++k) {
        int64_t t = t0 + k * DIRECT_THREADS;
        if (t < ntrg) {
            float* o = partial + ((int64_t)blockIdx.y * ntrg + t) * NC;
#pragma unroll
            for (int c = 0; c < NC; ++c) o[c] = acc[k][c];
        }
    }
}

__global__ void reduce_splits(const float* __restrict__ partial, int nsplit, int64_t m,
                              float* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    float s = 0.f;
    for (int k = 0; k < nsplit; ++k) s += partial[k * m + i];
    out[i] = s;
}

template <bool SL, bool DL, bool STRESS>
static void launch_direct(const float4* rec, int64_t nsrc, const float* trg, int64_t ntrg,
                          const KConst& kc, float* out, cudaStream_t s) {
    constexpr int NC = STRESS ? 6 : 3;
    const int tblocks = ceil_div(ntrg, DIRECT_THREADS * DIRECT_TPT);
    // split the sources so the grid fills the resident CTA slots of one wave as closely
    // as possible (partial second waves cost more than an under-full first one)
    int occ = 0;
    EB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, direct_kernel<SL, DL, STRESS>, DIRECT_THREADS, 0));
    const int slots = num_sms() * std::max(occ, 1);
    int nsplit = std::max(1, std::min(slots / tblocks, ceil_div(nsrc, 4 * DIRECT_TILE)));
    if (const char* e = std::getenv("EBEM_DIRECT_SPLIT")) nsplit = std::max(1, std::atoi(e));
    nsplit = std::min(nsplit, 65535);
    // whole shared-memory tiles per CTA (measured: ragged chunks cost 15-100%)
    int64_t chunk = ((nsrc + nsplit - 1) / nsplit + DIRECT_TILE - 1) / DIRECT_TILE * DIRECT_TILE;
    nsplit = (int)((nsrc + chunk - 1) / chunk);
    if (nsplit <= 1) {
        dim3 grid(tblocks, 1);
        direct_kernel<SL, DL, STRESS><<<grid, DIRECT_THREADS, 0, s>>>(rec, nsrc, nsrc, trg, ntrg, kc, out);
        EB_CHECK_LAUNCH();
        return;
    }
    float* partial = nullptr;
    EB_CUDA(cudaMallocAsync(&partial, sizeof(float) * nsplit * ntrg * NC, s));
    dim3 grid(tblocks, nsplit);
    direct_kernel<SL, DL, STRESS><<<grid, DIRECT_THREADS, 0, s>>>(rec, nsrc, chunk, trg, ntrg, kc, partial);
    EB_CHECK_LAUNCH();
    reduce_splits<<<ceil_div(ntrg * NC, 256), 256, 0, s>>>(partial, nsplit, ntrg * NC, out);
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
