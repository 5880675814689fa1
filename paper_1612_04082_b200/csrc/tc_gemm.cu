// Tensor-core (tcgen05, sm_100a) operator-grouped pairs GEMM with three-product operand splits:
//     Y[t] += Mat[op] X[s]      for every pair (t, s) of every operator op
// used for the KIFMM translations ("M2M, L2L and M2L operators ...
// represented by matrices"): Q2Z, M2M, M2L, L2L.  Pairs are grouped by operator (for
// M2L: by translation vector), so a CTA tile is operator row slices times a block of pairs:
// a dense [rows x K] x [K x pairs] contraction with the B operand gathered row by row from
// the state array.
//
// Precision: A = A_b + A_s and B = B_b + B_s with round-to-nearest heads and remainders of 11
// significand bits (A_b = rn(A), A_s = rn(A - A_b), same for B); D += A_b B_b + A_b B_s +
// A_s B_b in fp32 TMEM accumulators: unbiased error ~3 * 2^-22 relative per product, the fp32
// level.  Two operand types: TF32 (kind::tf32, 8 K per MMA) and FP16 (kind::f16, 16 K per MMA,
// twice the rate; rows scaled by powers of two so that the fp16 exponent range never shows --
// split_rows_h_kernel, reading R14).
//
// Kernels: tc_pairs_kernel (one 128-row slice x 128 pairs, TF32, TMA gather4 rows, partial
// sums drained every two K chunks: the precise kernel); tc_pairs_fast_kernel (two slices x 128
// pairs) and tc_pairs_wide_kernel (one slice x 256 pairs), TF32 or FP16, rows gathered by
// cp.async, full-K TMEM accumulation or drained groups; tc_pairs_mc_kernel (cluster multicast of
// the operator tiles); tc_chain_kernel (a whole M2M / L2L chain in one persistent launch).
//
// CTA of the precise kernel = 8 warps.  warp 0: TMA producer (A_b, A_s 3-D tile loads; B_b, B_s
// gather4), warp 1 lane 0: tcgen05.mma issuer, warp 2: TMEM allocator, warps 4-7: drain TMEM
// partial sums into fp32 registers, then fp64 REDs into Y (coalesced along rows).
// 3-stage smem ring of 4 x 16 KB (SWIZZLE_128B, K-major), mbarrier full/empty pipeline.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>

#include "fmm.cuh"

namespace ebem {

namespace tc {

constexpr int BM = 128, BN = 128, BK = 32;     // tile: 128 rows x 128 pairs x 32 K (128 B)
constexpr int STAGES = 3;
constexpr int OPND_BYTES = BM * BK * 4;        // 16 KB per operand tile (BM == BN)
constexpr int STAGE_BYTES = 4 * OPND_BYTES;    // Ab, As, Bb, Bs
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int THREADS = 256;
constexpr int TMEM_COLS = 4 * BN;              // 2 main (ping-pong) + 2 correction accumulators

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
#ifdef MBAR_SPIN           // measurement build: non-blocking test_wait polling instead of try_wait
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
#else
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
#endif
    } while (!done);
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2,
                                            int r3, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(dst), "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
}

// K-major SWIZZLE_128B UMMA shared-memory descriptor (rows of 128 B, 8-row atoms 1024 B apart)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);          // start address
    d |= (uint64_t)1 << 16;                         // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;               // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                         // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                         // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// operand element type of the fast / wide kernels: TF32 (4 B, 8 per MMA) or FP16 (2 B, 16 per
// MMA).  A K chunk is 128 B of each operand row either way, so the shared-memory layout, the
// TMA boxes (in bytes) and the 16-B cp.async gathers are the same; an FP16 chunk carries twice
// the K extent for the same tensor-pipe time.
template <bool F16>
__device__ __forceinline__ void mma_op(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
#ifdef M2L_NO_MMA          // ablation build (timing only): loads, barriers and epilogue without the MMAs
    return;
#endif
    if (F16) mma_f16(tmem_d, a, b, idesc, acc);
    else mma_tf32(tmem_d, a, b, idesc, acc);
}
// instruction descriptor: D f32, A/B tf32 (format 2) or f16 (format 0), both K-major
template <bool F16>
__device__ __forceinline__ uint32_t make_idesc(uint32_t n, uint32_t m) {
    return (1u << 4) | ((F16 ? 0u : 2u) << 7) | ((F16 ? 0u : 2u) << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

struct Tile {
    int op, p0, np, m0;
    int kc0, kc1;        // K chunks [kc0, kc1) of this tile (split K on small launches)
};

// The tensor core's fp32 accumulation is not round-to-nearest: chaining all K/8 MMAs
// into one accumulator costs ~(chain length) x 2^-24 of bias (measured: FMM p=10 error
// 8e-6 with one chain vs 5.5e-7 with SIMT fp32).  The main products therefore go to two
// ping-pong TMEM accumulators that restart every GROUP K-chunks; epilogue warps drain
// each finished group into fp32 registers (round-to-nearest adds) while the MMA warp
// fills the other buffer.  The small correction products (A_b B_s + A_s B_b, ~2^-11 of
// the main) accumulate in a third buffer over the whole K.
constexpr int GROUP = 2;
constexpr int EPI_WARP0 = 4;                   // warps 4..7: epilogue / drain (TMEM lanes 0..127)

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
          "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// add the 128 columns of TMEM buffer `col` (this warp's 32 lanes) into acc[128]
__device__ __forceinline__ void drain_add(uint32_t tmem, int wq, int col, float* acc) {
#pragma unroll
    for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(32 * wq) << 16) + (uint32_t)(col + c0), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[c0 + j] += __uint_as_float(v[j]);
    }
}

// Epilogue of a translation tile: Y[target row][row] += v (fp64 atomic: exact, order
// independent).  Each lane owns one TMEM lane (operator row) and walks the tile's columns
// (pairs); the column's target row and scale are loaded once per 32 columns, one column per
// lane (coalesced, independent loads), and broadcast by shuffles.  FP16 operands are scaled by
// powers of two -- the operator set by 1 / ascale_inv, every source row by 1 / bscale[row]
// (split_rows_h_kernel) -- which the fp32 product undoes exactly.
//
// The column code is branch-free: every lane issues its RED, lanes and columns outside the
// tile add 0.0 to an element the tile owns anyway (a row 32 above for lanes past the
// operator's last row, the tile's last pair for columns past np; scale 0).  With a guarded
// `if (on) atomicAdd(...)` (also as a predicated inline-PTX RED) ptxas put a branch and a
// convergence barrier (BSSY / BSYNC) around every column, so each column's shuffle ->
// multiply -> convert -> RED chain (~90 cycles) ran after the previous one: the epilogue alone
// took 1.0 ms of the 1.37 ms FP16 M2L, with or without the REDs (ablation builds M2L_NO_*,
// DESIGN.md Sec. 6).
template <bool F16>
__device__ __forceinline__ void epi_cols_load(const int2* __restrict__ pp, int c0, int np, int lane,
                                              const float* __restrict__ bscale, float ascale_inv, int& trow,
                                              float& sc) {
    const bool in = c0 + lane < np;
    const int2 pr = __ldg(&pp[in ? c0 + lane : np - 1]);     // np >= 1 here
    trow = pr.x;
    sc = F16 ? ascale_inv * __ldg(&bscale[pr.y]) : 1.f;
    if (!in) sc = 0.f;
}
// rowc: the lane's row, or a valid row of the same slice for lanes past the last row (row_ok false)
__device__ __forceinline__ void epi_col_add(double* __restrict__ Y, int ldy, int rowc, bool row_ok, int trow, float sc,
                                            int j, float v) {
    const int tr = __shfl_sync(0xffffffffu, trow, j);
    const float scj = __shfl_sync(0xffffffffu, sc, j);
    v = row_ok ? v * scj : 0.f;
#ifdef M2L_NO_ATOMICS      // ablation build (timing only): everything but the RED
    if (v == 123456.789f)
#endif
#ifdef EPI_GUARD           // measurement build: the guarded (branchy) column code
    if (row_ok && scj != 0.f)
#endif
    atomicAdd(Y + (int64_t)tr * ldy + rowc, (double)v);
}

// Persistent: grid = #SMs, CTA b takes tiles b, b + grid, ... (op-major order, so the
// concurrently running tiles share operators in L2).  The smem ring, the ping-pong main
// accumulators and the two per-tile correction accumulators all continue across tiles,
// so the producers load tile i+1 while the MMA finishes tile i and the epilogue of tile
// i-1 does its atomics.
__global__ void __launch_bounds__(THREADS, 1)
tc_pairs_kernel(const __grid_constant__ CUtensorMap mapAb, const __grid_constant__ CUtensorMap mapAs,
                const __grid_constant__ CUtensorMap mapBb, const __grid_constant__ CUtensorMap mapBs,
                const Tile* __restrict__ tiles, int ntiles, const int2* __restrict__ pairs, int M, int K,
                double* __restrict__ Y, int ldy) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    // barriers: full[S], empty[S], acc_full[2], acc_empty[2], corr_full[2], corr_empty[2]
    uint64_t* bars = (uint64_t*)(smem + STAGES * STAGE_BYTES);
    uint64_t* full_b = bars;
    uint64_t* empty_b = bars + STAGES;
    uint64_t* accf_b = bars + 2 * STAGES;
    uint64_t* acce_b = bars + 2 * STAGES + 2;
    uint64_t* corf_b = bars + 2 * STAGES + 4;
    uint64_t* core_b = bars + 2 * STAGES + 6;
    uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    (void)K;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full_b[s]), 1);
            mbar_init(smem_u32(&empty_b[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&accf_b[b]), 1);
            mbar_init(smem_u32(&acce_b[b]), 4);
            mbar_init(smem_u32(&corf_b[b]), 1);
            mbar_init(smem_u32(&core_b[b]), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 || warp == 2 || warp == 3) {
        // ---------------- producers: warp 0 arms the stage barrier and loads A; the 32
        // four-row gathers of each B operand are spread over warps 0, 2, 3 (a TMA needs
        // uniform operands, so each warp issues its lanes' gathers one after another)
        const int pw = warp == 0 ? 0 : warp - 1;            // 0, 1, 2
        const int gi = pw * 11 + lane;
        const bool gact = lane < 11 && gi < 32;
        int c = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
            const Tile tl = tiles[ti];
            int r[4] = {0, 0, 0, 0};
            if (gact)
#pragma unroll
                for (int q = 0; q < 4; ++q) r[q] = pairs[tl.p0 + min(4 * gi + q, tl.np - 1)].y;
            for (int kc = tl.kc0; kc < tl.kc1; ++kc, ++c) {
                const int s = c % STAGES;
                mbar_wait(smem_u32(&empty_b[s]), ((c / STAGES) & 1) ^ 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                const uint32_t full = smem_u32(&full_b[s]);
                if (warp == 0 && lane == 0) {
                    mbar_expect_tx(full, STAGE_BYTES);
                    tma_load_3d(smem_u32(st), &mapAb, kc * BK, tl.m0, tl.op, full);
                    tma_load_3d(smem_u32(st + OPND_BYTES), &mapAs, kc * BK, tl.m0, tl.op, full);
                }
                __syncwarp();
                if (gact) {
                    tma_gather4(smem_u32(st + 2 * OPND_BYTES + 4 * gi * 128), &mapBb, kc * BK, r[0], r[1], r[2],
                                r[3], full);
                    tma_gather4(smem_u32(st + 3 * OPND_BYTES + 4 * gi * 128), &mapBs, kc * BK, r[0], r[1], r[2],
                                r[3], full);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread)
        // instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                               ((uint32_t)(BM >> 4) << 24);
        int c = 0, G = 0, it = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++it) {
            const int cb = it & 1;
            mbar_wait(smem_u32(&core_b[cb]), ((it >> 1) & 1) ^ 1);   // correction buffer drained
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t dcorr = tmem + (uint32_t)((2 + cb) * BN);
            const int kc0 = tiles[ti].kc0, kc1 = tiles[ti].kc1;
            for (int kc = kc0; kc < kc1; ++kc, ++c) {
                const int s = c % STAGES;
                const int b = G & 1;
                const bool gfirst = ((kc - kc0) % GROUP) == 0,
                           glast = ((kc - kc0) % GROUP) == GROUP - 1 || kc == kc1 - 1;
                if (gfirst) {   // the main buffer must have been drained
                    mbar_wait(smem_u32(&acce_b[b]), ((G >> 1) & 1) ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                mbar_wait(smem_u32(&full_b[s]), (c / STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (lane == 0) {
                    const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
                    const uint64_t ab = smem_desc(st), as = smem_desc(st + OPND_BYTES);
                    const uint64_t bb = smem_desc(st + 2 * OPND_BYTES), bs = smem_desc(st + 3 * OPND_BYTES);
                    const uint32_t dmain = tmem + (uint32_t)(b * BN);
                    const int ksteps = min(BK, K - kc * BK + 7) / 8;     // 8 tf32 (32 B) per MMA
                    for (int k = 0; k < ksteps; ++k) {
                        const uint64_t off = (uint64_t)(2 * k);          // +32 B in 16-B units
                        mma_tf32(dmain, ab + off, bb + off, idesc, (!gfirst) | (k != 0));
                        mma_tf32(dcorr, ab + off, bs + off, idesc, kc != kc0 || k != 0);
                        mma_tf32(dcorr, as + off, bb + off, idesc, 1);
                    }
                    mma_commit(smem_u32(&empty_b[s]));                   // frees the smem stage
                    if (glast) mma_commit(smem_u32(&accf_b[b]));          // group partial ready
                    if (kc == kc1 - 1) mma_commit(smem_u32(&corf_b[cb]));  // corrections ready
                }
                __syncwarp();
                if (glast) ++G;
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ---------------- drain + epilogue: fp32 register accumulation, then atomics into Y
        const int wq = warp - EPI_WARP0;            // TMEM lane quarter
        int G = 0, it = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++it) {
            const Tile tl = tiles[ti];
            const int cb = it & 1;
            float acc[BN];
#pragma unroll
            for (int j = 0; j < BN; ++j) acc[j] = 0.f;
            const int ngroups = (tl.kc1 - tl.kc0 + GROUP - 1) / GROUP;
            for (int g = 0; g < ngroups; ++g, ++G) {
                const int b = G & 1;
                mbar_wait(smem_u32(&accf_b[b]), (G >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                drain_add(tmem, wq, b * BN, acc);
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&acce_b[b]));
            }
            mbar_wait(smem_u32(&corf_b[cb]), (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            drain_add(tmem, wq, (2 + cb) * BN, acc);
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&core_b[cb]));
            const int row = tl.m0 + 32 * wq + lane;
            if (row - lane < M) {                            // (warp-uniform) some of this warp's rows exist
                const int2* pp = pairs + tl.p0;
                const int rowc = row < M ? row : row - 32;
#pragma unroll
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    if (c0 >= tl.np) break;
                    int trow;
                    float sc;
                    epi_cols_load<false>(pp, c0, tl.np, lane, nullptr, 1.f, trow, sc);
#pragma unroll
                    for (int j = 0; j < 32; ++j) epi_col_add(Y, ldy, rowc, row < M, trow, sc, j, acc[c0 + j]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// ------------------------------------------------------------------ fast variant (p <= 8)
// Same contraction, tuned for throughput where the full-K tensor-core accumulation chain
// (error ~1e-6 relative, see the precise kernel's note) is far below the FMM truncation
// error: each CTA tile is TWO 128-row operator slices x 128 pairs, so the gathered B rows
// (the expensive, L2-missing operand) are loaded once for 256 output rows, each K chunk
// carries 24 MMAs (half the per-stage pipeline overhead per MMA), and whole-K accumulators
// live in TMEM (2 tiles in flight = 4 x 128 columns) read straight into the atomics.
// B comes from the precomputed TF32 head/remainder copies by coalesced 16-B cp.async
// (8 lanes per 128-B row piece): a TMA gather4 issues only ~1 per 32 cycles per SM.
namespace fast {
constexpr int MT = 2;                                   // operator row slices per CTA tile
constexpr int STAGES = 2;
constexpr int STAGE_BYTES = (2 * MT + 2) * OPND_BYTES;  // A_b,A_s per slice + B_b,B_s = 96 KB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 512;                          // 2 tiles x MT slices x 128 columns
constexpr int NPROD = 3;                                // B-gather warps (0, 2, 3); 5 or 7 were no faster
constexpr int THREADS = 256;
constexpr int NG = (BN / 4 + NPROD - 1) / NPROD;        // 4-row groups per producer warp
}  // namespace fast

// DRAIN = true: the precise variant for p >= 9 and GMRES.  The MMAs of every GROUP K chunks go
// to one of two ping-pong TMEM buffers (2 slices x 128 columns each); eight epilogue warps
// (one per TMEM lane quarter and slice) add each finished group into fp32 registers (round
// to nearest) while the MMA fills the other buffer, so no tensor-core accumulation chain is
// longer than GROUP chunks.
template <bool DRAIN, bool F16>
__global__ void __launch_bounds__(DRAIN ? 384 : fast::THREADS, 1)
tc_pairs_fast_kernel(const __grid_constant__ CUtensorMap mapAb, const __grid_constant__ CUtensorMap mapAs,
                     const void* __restrict__ Bb_, const void* __restrict__ Bs_, int ldb,
                     const Tile* __restrict__ tiles, int ntiles, const int2* __restrict__ pairs, int M, int K,
                     double* __restrict__ Y, int ldy, const float* __restrict__ bscale, float ascale_inv) {
    // element size / K elements per 128-B chunk / K elements per MMA of the operand type
    constexpr int ES = F16 ? 2 : 4, BKE = 128 / ES, KS = 32 / ES;
    const char* Bb = reinterpret_cast<const char*>(Bb_);
    const char* Bs = reinterpret_cast<const char*>(Bs_);
    constexpr int MT = fast::MT, STAGES = fast::STAGES, STAGE_BYTES = fast::STAGE_BYTES, TMEM_COLS = fast::TMEM_COLS;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(smem + STAGES * STAGE_BYTES);
    uint64_t* full_b = bars;                     // [STAGES]
    uint64_t* empty_b = bars + STAGES;           // [STAGES]
    uint64_t* accf_b = bars + 2 * STAGES;        // [2]
    uint64_t* acce_b = bars + 2 * STAGES + 2;    // [2]
    uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full_b[s]), 1 + 32 * fast::NPROD);   // A expect_tx + cp.async arrivals
            mbar_init(smem_u32(&empty_b[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&accf_b[b]), 1);
            mbar_init(smem_u32(&acce_b[b]), DRAIN ? 8 : 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 || warp == 2 || warp == 3) {
        // ---------------- producers: warp 0 lane 0 issues the A tiles (TMA); warps 0, 2, 3
        // gather the B rows with 16-B cp.async (one warp could not issue them fast enough:
        // the loads are latency bound per instruction, the MMA warp waited on full barriers)
        const int pi = warp == 0 ? 0 : warp - 1;
        const int piece = lane & 7, rsub = lane >> 3;
        int c = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
            const Tile tl = tiles[ti];
            int64_t srow[fast::NG];                      // this lane's source rows x ldb
#pragma unroll
            for (int g = 0; g < fast::NG; ++g) {
                const int r = rsub + 4 * (pi + fast::NPROD * g);
                srow[g] = (int64_t)__ldg(&pairs[tl.p0 + min(r, tl.np - 1)].y) * ldb;
            }
            for (int kc = tl.kc0; kc < tl.kc1; ++kc, ++c) {
                const int s = c % STAGES;
                mbar_wait(smem_u32(&empty_b[s]), ((c / STAGES) & 1) ^ 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                const uint32_t full = smem_u32(&full_b[s]);
                // a second row slice entirely past the operator's M rows is neither loaded nor
                // multiplied (p = 8: 888 rows = 3.5 tile pairs, 12% of the MMAs saved)
                const int nmt = tl.m0 + BM < M ? MT : 1;
                if (pi == 0 && lane == 0) {
#ifdef M2L_NO_A            // ablation build (timing only): no operator tiles
                    mbar_arrive(full);
#else
                    mbar_expect_tx(full, 2 * nmt * OPND_BYTES);
                    for (int mt = 0; mt < nmt; ++mt) {
                        tma_load_3d(smem_u32(st + (2 * mt) * OPND_BYTES), &mapAb, kc * BKE, tl.m0 + mt * BM, tl.op, full);
                        tma_load_3d(smem_u32(st + (2 * mt + 1) * OPND_BYTES), &mapAs, kc * BKE, tl.m0 + mt * BM, tl.op,
                                    full);
                    }
#endif
                }
                const int col = kc * BKE + (16 / ES) * piece;
                const uint32_t nb = col < ldb ? 16u : 0u;      // zero-fill past the row
                const int ngrp = ((tl.np + 15) & ~15) / 4;     // row groups the MMA reads (N)
                const uint32_t b0 = smem_u32(st + 2 * MT * OPND_BYTES);
                const uint32_t b1 = b0 + OPND_BYTES;
#pragma unroll
                for (int g = 0; g < fast::NG; ++g) {
                    const int grp = pi + fast::NPROD * g;
#ifdef M2L_NO_B            // ablation build (timing only): no gathered rows
                    if (false) {
#else
                    if (grp < ngrp) {
#endif
                        const int r = rsub + 4 * grp;
                        const int64_t off = (srow[g] + col) * ES;
                        const uint32_t so = (uint32_t)(r * 128 + ((piece ^ (r & 7)) * 16));
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(b0 + so),
                                     "l"(nb ? Bb + off : Bb), "r"(nb)
                                     : "memory");
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(b1 + so),
                                     "l"(nb ? Bs + off : Bs), "r"(nb)
                                     : "memory");
                    }
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full) : "memory");
            }
        }
    } else if (warp == 1 && DRAIN) {
        // ---------------- MMA issuer, drained groups
        int c = 0, G = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
            const uint32_t nmma = (uint32_t)((tiles[ti].np + 15) & ~15);
            const uint32_t idesc = make_idesc<F16>(nmma, BM);
            const int kc0 = tiles[ti].kc0, kc1 = tiles[ti].kc1;
            for (int kc = kc0; kc < kc1; ++kc, ++c) {
                const int s = c % STAGES;
                const int b = G & 1;
                const bool gfirst = ((kc - kc0) % GROUP) == 0,
                           glast = ((kc - kc0) % GROUP) == GROUP - 1 || kc == kc1 - 1;
                if (gfirst) {   // the buffer's previous group has been drained
                    mbar_wait(smem_u32(&acce_b[b]), ((G >> 1) & 1) ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                mbar_wait(smem_u32(&full_b[s]), (c / STAGES) & 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (lane == 0) {
                    const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
                    const uint64_t bb = smem_desc(st + 2 * MT * OPND_BYTES), bs = smem_desc(st + (2 * MT + 1) * OPND_BYTES);
                    const int ksteps = min(BKE, K - kc * BKE + KS - 1) / KS;
                    for (int k = 0; k < ksteps; ++k) {
                        const uint64_t off = (uint64_t)(2 * k);
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            if (tiles[ti].m0 + mt * BM >= M) continue;
                            const uint64_t a_b = smem_desc(st + (2 * mt) * OPND_BYTES) + off;
                            const uint64_t a_s = smem_desc(st + (2 * mt + 1) * OPND_BYTES) + off;
                            const uint32_t d = tmem + (uint32_t)((b * MT + mt) * BN);
                            mma_op<F16>(d, a_b, bb + off, idesc, !gfirst || k != 0);
                            mma_op<F16>(d, a_b, bs + off, idesc, 1);
                            mma_op<F16>(d, a_s, bb + off, idesc, 1);
                        }
                    }
                    mma_commit(smem_u32(&empty_b[s]));
                    if (glast) mma_commit(smem_u32(&accf_b[b]));
                }
                __syncwarp();
                if (glast) ++G;
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        int c = 0, it = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++it) {
            const int ab = it & 1;
            // N = the tile's pairs rounded up to 16: partial tiles cost in proportion
            const uint32_t nmma = (uint32_t)((tiles[ti].np + 15) & ~15);
            const uint32_t idesc = make_idesc<F16>(nmma, BM);
            mbar_wait(smem_u32(&acce_b[ab]), ((it >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int kc0 = tiles[ti].kc0, kc1 = tiles[ti].kc1;
            for (int kc = kc0; kc < kc1; ++kc, ++c) {
                const int s = c % STAGES;
                mbar_wait(smem_u32(&full_b[s]), (c / STAGES) & 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // cp.async data -> tensor core
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (lane == 0) {
                    const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
                    const uint64_t bb = smem_desc(st + 2 * MT * OPND_BYTES), bs = smem_desc(st + (2 * MT + 1) * OPND_BYTES);
                    const int ksteps = min(BKE, K - kc * BKE + KS - 1) / KS;
                    for (int k = 0; k < ksteps; ++k) {
                        const uint64_t off = (uint64_t)(2 * k);
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            if (tiles[ti].m0 + mt * BM >= M) continue;
                            const uint64_t a_b = smem_desc(st + (2 * mt) * OPND_BYTES) + off;
                            const uint64_t a_s = smem_desc(st + (2 * mt + 1) * OPND_BYTES) + off;
                            const uint32_t d = tmem + (uint32_t)((ab * MT + mt) * BN);
                            mma_op<F16>(d, a_b, bb + off, idesc, kc != kc0 || k != 0);
                            mma_op<F16>(d, a_b, bs + off, idesc, 1);
                            mma_op<F16>(d, a_s, bb + off, idesc, 1);
                        }
                    }
                    mma_commit(smem_u32(&empty_b[s]));
                    if (kc == kc1 - 1) mma_commit(smem_u32(&accf_b[ab]));
                }
                __syncwarp();
            }
        }
    } else if (warp >= EPI_WARP0 && DRAIN) {
        // ---------------- drains: warp -> (lane quarter, slice); fp32 register sums, then atomics
        const int wq = warp & 3, mt = (warp - EPI_WARP0) >> 2;
        int G = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
            const Tile tl = tiles[ti];
            float acc[BN];
#pragma unroll
            for (int j = 0; j < BN; ++j) acc[j] = 0.f;
            const int ngroups = (tl.kc1 - tl.kc0 + GROUP - 1) / GROUP;
            for (int g = 0; g < ngroups; ++g, ++G) {
                const int b = G & 1;
                mbar_wait(smem_u32(&accf_b[b]), (G >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                drain_add(tmem, wq, (b * MT + mt) * BN, acc);
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&acce_b[b]));
            }
            const int row = tl.m0 + mt * BM + 32 * wq + lane;
            const int2* pp = pairs + tl.p0;
            if (row - lane < M) {                            // (warp-uniform) some of this warp's rows exist
                const int rowc = row < M ? row : row - 32;
#pragma unroll
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    if (c0 >= tl.np) break;
                    int trow;
                    float sc;
                    epi_cols_load<F16>(pp, c0, tl.np, lane, bscale, ascale_inv, trow, sc);
#pragma unroll
                    for (int j = 0; j < 32; ++j) epi_col_add(Y, ldy, rowc, row < M, trow, sc, j, acc[c0 + j]);
                }
            }
        }
    } else if (warp >= EPI_WARP0 && warp < EPI_WARP0 + 4) {
        // ---------------- epilogue: TMEM -> fp64 atomics, 32 columns at a time
        const int wq = warp - EPI_WARP0;
        int it = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++it) {
            const Tile tl = tiles[ti];
            const int ab = it & 1;
            mbar_wait(smem_u32(&accf_b[ab]), (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int2* pp = pairs + tl.p0;
#ifdef M2L_NO_EPI          // ablation build (timing only): accumulators released unread
            const int np_epi = 0;
#else
            const int np_epi = tl.np;
#endif
#pragma unroll 1
            for (int c0 = 0; c0 < np_epi; c0 += 32) {
                int trow;
                float sc;
                epi_cols_load<F16>(pp, c0, tl.np, lane, bscale, ascale_inv, trow, sc);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const int row = tl.m0 + mt * BM + 32 * wq + lane;
                    if (row - lane >= M) continue;           // none of this warp's rows exist (warp-uniform)
                    const int rowc = row < M ? row : row - 32;
                    uint32_t v[32];
                    tmem_ld32(tmem + ((uint32_t)(32 * wq) << 16) + (uint32_t)((ab * MT + mt) * BN + c0), v);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 32; ++j) epi_col_add(Y, ldy, rowc, row < M, trow, sc, j, __uint_as_float(v[j]));
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&acce_b[ab]));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// ------------------------------------------------------------------ cluster-multicast variant
// The full-chain two-slice contraction on thread-block clusters of CS = 2 or 4 CTAs: the CTAs
// of a cluster take pair blocks of the SAME operator and row slices, so the operator tiles
// (A: 64 of the 96 KB a stage moves) are loaded once per cluster -- each CTA issues its share
// of the four A tiles by TMA multicast into every CTA's shared memory -- and only the gathered
// B rows are per CTA.  With FP16 operands the MMAs of the M2L take ~0.6 ms and its operand
// loads alone ~1.0 ms (8 GB through the L2 at p = 6; ablation builds M2L_NO_MMA /
// M2L_NO_ATOMICS): the kernel is bound by L2 -> SM bandwidth, which multicast cuts by a third
// (CS = 2) or a half (CS = 4).  A stage may be refilled only when EVERY CTA's MMAs are done
// with it: each MMA commit arrives on the empty barrier of all CTAs (tcgen05.commit multicast;
// count CS).
__device__ __forceinline__ void tma_load_3d_mc(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                               uint32_t bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%2, %3, %4}], [%5], %6;"
        ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
        ::"r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// tiles[CS c + r] is the work of cluster rank r in cluster tile c (same op, m0 and K range;
// np = 0 pads an operator's last cluster tile)
template <bool F16, int CS>
__global__ void __launch_bounds__(fast::THREADS, 1)
tc_pairs_mc_kernel(const __grid_constant__ CUtensorMap mapAb, const __grid_constant__ CUtensorMap mapAs,
                   const void* __restrict__ Bb_, const void* __restrict__ Bs_, int ldb,
                   const Tile* __restrict__ tiles, int nctiles, const int2* __restrict__ pairs, int M, int K,
                   double* __restrict__ Y, int ldy, const float* __restrict__ bscale, float ascale_inv) {
    constexpr int MT = fast::MT, STAGES = fast::STAGES, STAGE_BYTES = fast::STAGE_BYTES, TMEM_COLS = fast::TMEM_COLS;
    constexpr int ES = F16 ? 2 : 4, BKE = 128 / ES, KS = 32 / ES;
    static_assert(CS == 2 || CS == 4, "cluster of 2 or 4");
    const char* Bb = reinterpret_cast<const char*>(Bb_);
    const char* Bs = reinterpret_cast<const char*>(Bs_);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(smem + STAGES * STAGE_BYTES);
    uint64_t* full_b = bars;                     // [STAGES]
    uint64_t* empty_b = bars + STAGES;           // [STAGES]
    uint64_t* accf_b = bars + 2 * STAGES;        // [2]
    uint64_t* acce_b = bars + 2 * STAGES + 2;    // [2]
    uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;
    const uint16_t all = (uint16_t)((1u << CS) - 1);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full_b[s]), 1 + 32 * fast::NPROD);   // A expect_tx + cp.async arrivals
            mbar_init(smem_u32(&empty_b[s]), CS);                    // every CTA's MMA commit
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&accf_b[b]), 1);
            mbar_init(smem_u32(&acce_b[b]), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();                              // every CTA's barriers initialised before any multicast
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 || warp == 2 || warp == 3) {
        // ---------------- producers: this CTA's share of the A tiles (multicast), its own B rows
        const int pi = warp == 0 ? 0 : warp - 1;
        const int piece = lane & 7, rsub = lane >> 3;
        int c = 0;
        for (int ci = cid; ci < nctiles; ci += ncl) {
            const Tile tl = tiles[CS * ci + rank];
            int64_t srow[fast::NG];
#pragma unroll
            for (int g = 0; g < fast::NG; ++g) {
                const int r = rsub + 4 * (pi + fast::NPROD * g);
                srow[g] = (int64_t)__ldg(&pairs[tl.p0 + max(min(r, tl.np - 1), 0)].y) * ldb;
            }
            const int ngrp = ((tl.np + 15) & ~15) / 4;
            for (int kc = tl.kc0; kc < tl.kc1; ++kc, ++c) {
                const int s = c % STAGES;
                mbar_wait(smem_u32(&empty_b[s]), ((c / STAGES) & 1) ^ 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                const uint32_t full = smem_u32(&full_b[s]);
                if (pi == 0 && lane == 0) {
                    mbar_expect_tx(full, 2 * MT * OPND_BYTES);          // all four A tiles land here
                    if (CS == 2) {   // rank 0 multicasts the head tiles, rank 1 the remainder tiles
                        const CUtensorMap* map = rank == 0 ? &mapAb : &mapAs;
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt)
                            tma_load_3d_mc(smem_u32(st + (2 * mt + rank) * OPND_BYTES), map, kc * BKE, tl.m0 + mt * BM,
                                           tl.op, full, all);
                    } else {         // rank = 2 slice + (head 0 / remainder 1): one tile each
                        const CUtensorMap* map = (rank & 1) == 0 ? &mapAb : &mapAs;
                        tma_load_3d_mc(smem_u32(st + rank * OPND_BYTES), map, kc * BKE, tl.m0 + (int)(rank >> 1) * BM,
                                       tl.op, full, all);
                    }
                }
                const int col = kc * BKE + (16 / ES) * piece;
                const uint32_t nb = col < ldb ? 16u : 0u;
                const uint32_t b0 = smem_u32(st + 2 * MT * OPND_BYTES);
                const uint32_t b1 = b0 + OPND_BYTES;
#pragma unroll
                for (int g = 0; g < fast::NG; ++g) {
                    const int grp = pi + fast::NPROD * g;
                    if (grp < ngrp) {
                        const int r = rsub + 4 * grp;
                        const int64_t off = (srow[g] + col) * ES;
                        const uint32_t so = (uint32_t)(r * 128 + ((piece ^ (r & 7)) * 16));
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(b0 + so),
                                     "l"(nb ? Bb + off : Bb), "r"(nb)
                                     : "memory");
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(b1 + so),
                                     "l"(nb ? Bs + off : Bs), "r"(nb)
                                     : "memory");
                    }
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full) : "memory");
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer; the stage release goes to every CTA of the cluster
        int c = 0, it = 0;
        for (int ci = cid; ci < nctiles; ci += ncl, ++it) {
            const Tile tl = tiles[CS * ci + rank];
            const int ab = it & 1;
            const uint32_t nmma = (uint32_t)max(16, (tl.np + 15) & ~15);
            const uint32_t idesc = make_idesc<F16>(nmma, BM);
            mbar_wait(smem_u32(&acce_b[ab]), ((it >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int kc = tl.kc0; kc < tl.kc1; ++kc, ++c) {
                const int s = c % STAGES;
                mbar_wait(smem_u32(&full_b[s]), (c / STAGES) & 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (lane == 0) {
                    const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
                    const uint64_t bb = smem_desc(st + 2 * MT * OPND_BYTES), bs = smem_desc(st + (2 * MT + 1) * OPND_BYTES);
                    const int ksteps = min(BKE, K - kc * BKE + KS - 1) / KS;
                    if (tl.np > 0)
                        for (int k = 0; k < ksteps; ++k) {
                            const uint64_t off = (uint64_t)(2 * k);
#pragma unroll
                            for (int mt = 0; mt < MT; ++mt) {
                                if (tl.m0 + mt * BM >= M) continue;
                                const uint64_t a_b = smem_desc(st + (2 * mt) * OPND_BYTES) + off;
                                const uint64_t a_s = smem_desc(st + (2 * mt + 1) * OPND_BYTES) + off;
                                const uint32_t d = tmem + (uint32_t)((ab * MT + mt) * BN);
                                mma_op<F16>(d, a_b, bb + off, idesc, kc != tl.kc0 || k != 0);
                                mma_op<F16>(d, a_b, bs + off, idesc, 1);
                                mma_op<F16>(d, a_s, bb + off, idesc, 1);
                            }
                        }
                    mma_commit_mc(smem_u32(&empty_b[s]), all);
                    if (kc == tl.kc1 - 1) mma_commit(smem_u32(&accf_b[ab]));
                }
                __syncwarp();
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ---------------- epilogue: TMEM -> fp64 atomics, 32 columns at a time
        const int wq = warp - EPI_WARP0;
        int it = 0;
        for (int ci = cid; ci < nctiles; ci += ncl, ++it) {
            const Tile tl = tiles[CS * ci + rank];
            const int ab = it & 1;
            mbar_wait(smem_u32(&accf_b[ab]), (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int2* pp = pairs + tl.p0;
            const int np_epi = tl.np;
#pragma unroll 1
            for (int c0 = 0; c0 < np_epi; c0 += 32) {
                int trow;
                float sc;
                epi_cols_load<F16>(pp, c0, tl.np, lane, bscale, ascale_inv, trow, sc);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const int row = tl.m0 + mt * BM + 32 * wq + lane;
                    if (row - lane >= M) continue;           // none of this warp's rows exist (warp-uniform)
                    const int rowc = row < M ? row : row - 32;
                    uint32_t v[32];
                    tmem_ld32(tmem + ((uint32_t)(32 * wq) << 16) + (uint32_t)((ab * MT + mt) * BN + c0), v);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 32; ++j) epi_col_add(Y, ldy, rowc, row < M, trow, sc, j, __uint_as_float(v[j]));
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&acce_b[ab]));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();                              // no CTA leaves while a peer may still signal it
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// ------------------------------------------------------------------ wide variant (full chain)
// The same contraction with one 128-row operator slice x 256 pairs per tile (MMA N = 256).
// A tf32 M128 x N x K8 MMA takes 128 N / 256 cycles and reads (128 + N) x 32 B of shared
// memory (both operands from smem): at N = 128 that is 128 B / cycle, the whole shared-memory
// bandwidth, before the TMA / cp.async fills of the next stage (another ~62 B / cycle) -- the
// two-slice kernel's tensor pipe could not exceed ~2/3.  At N = 256 the operand reads are
// 96 B / cycle for the same bytes filled per MMA cycle.  TMEM: 2 tiles x 256 columns.
namespace wide {
constexpr int BNW = 256;
constexpr int STAGES = 2;
constexpr int A_BYTES = BM * BK * 4;                    // 16 KB (128 rows x 32 K)
constexpr int B_BYTES = BNW * BK * 4;                   // 32 KB (256 rows x 32 K)
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // A_b, A_s, B_b, B_s = 96 KB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 512;
constexpr int NPROD = 3;
constexpr int THREADS = 256;
constexpr int NG = (BNW / 4 + NPROD - 1) / NPROD;       // four-row groups per producer warp
}  // namespace wide

// DRAIN = true: drained groups as in tc_pairs_fast_kernel<true> (GROUP K chunks per ping-pong
// buffer of 256 columns, eight drain warps: lane quarter x column half, fp32 register sums)
template <bool DRAIN, bool F16>
__global__ void __launch_bounds__(DRAIN ? 384 : wide::THREADS, 1)
tc_pairs_wide_kernel(const __grid_constant__ CUtensorMap mapAb, const __grid_constant__ CUtensorMap mapAs,
                     const void* __restrict__ Bb_, const void* __restrict__ Bs_, int ldb,
                     const Tile* __restrict__ tiles, int ntiles, const int2* __restrict__ pairs, int M, int K,
                     double* __restrict__ Y, int ldy, const float* __restrict__ bscale, float ascale_inv) {
    // element size / K elements per 128-B chunk / K elements per MMA of the operand type
    constexpr int ES = F16 ? 2 : 4, BKE = 128 / ES, KS = 32 / ES;
    const char* Bb = reinterpret_cast<const char*>(Bb_);
    const char* Bs = reinterpret_cast<const char*>(Bs_);
    constexpr int STAGES = wide::STAGES, STAGE_BYTES = wide::STAGE_BYTES, A_BYTES = wide::A_BYTES,
                  B_BYTES = wide::B_BYTES, TMEM_COLS = wide::TMEM_COLS, NPROD = wide::NPROD, NG = wide::NG,
                  BNW = wide::BNW;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(smem + STAGES * STAGE_BYTES);
    uint64_t* full_b = bars;                     // [STAGES]
    uint64_t* empty_b = bars + STAGES;           // [STAGES]
    uint64_t* accf_b = bars + 2 * STAGES;        // [2]
    uint64_t* acce_b = bars + 2 * STAGES + 2;    // [2]
    uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full_b[s]), 1 + 32 * NPROD);   // A expect_tx + cp.async arrivals
            mbar_init(smem_u32(&empty_b[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&accf_b[b]), 1);
            mbar_init(smem_u32(&acce_b[b]), DRAIN ? 8 : 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 || warp == 2 || warp == 3) {
        // ---------------- producers: warp 0 lane 0 the A tiles (TMA); warps 0, 2, 3 the B rows
        const int pi = warp == 0 ? 0 : warp - 1;
        const int piece = lane & 7, rsub = lane >> 3;
        int c = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
            const Tile tl = tiles[ti];
            int64_t srow[NG];
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const int r = rsub + 4 * (pi + NPROD * g);
                srow[g] = (int64_t)__ldg(&pairs[tl.p0 + min(r, tl.np - 1)].y) * ldb;
            }
            const int ngrp = ((tl.np + 15) & ~15) / 4;     // row groups the MMA reads (N)
            for (int kc = tl.kc0; kc < tl.kc1; ++kc, ++c) {
                const int s = c % STAGES;
                mbar_wait(smem_u32(&empty_b[s]), ((c / STAGES) & 1) ^ 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                const uint32_t full = smem_u32(&full_b[s]);
                if (pi == 0 && lane == 0) {
                    mbar_expect_tx(full, 2 * A_BYTES);
                    tma_load_3d(smem_u32(st), &mapAb, kc * BKE, tl.m0, tl.op, full);
                    tma_load_3d(smem_u32(st + A_BYTES), &mapAs, kc * BKE, tl.m0, tl.op, full);
                }
                const int col = kc * BKE + (16 / ES) * piece;
                const uint32_t nb = col < ldb ? 16u : 0u;      // zero-fill past the row
                const uint32_t b0 = smem_u32(st + 2 * A_BYTES);
                const uint32_t b1 = b0 + B_BYTES;
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    const int grp = pi + NPROD * g;
                    if (grp < ngrp) {
                        const int r = rsub + 4 * grp;
                        const int64_t off = (srow[g] + col) * ES;
                        const uint32_t so = (uint32_t)(r * 128 + ((piece ^ (r & 7)) * 16));
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(b0 + so),
                                     "l"(nb ? Bb + off : Bb), "r"(nb)
                                     : "memory");
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(b1 + so),
                                     "l"(nb ? Bs + off : Bs), "r"(nb)
                                     : "memory");
                    }
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full) : "memory");
            }
        }
    } else if (warp == 1 && DRAIN) {
        // ---------------- MMA issuer, drained groups
        int c = 0, G = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
            const uint32_t nmma = (uint32_t)((tiles[ti].np + 15) & ~15);
            const uint32_t idesc = make_idesc<F16>(nmma, BM);
            const int kc0 = tiles[ti].kc0, kc1 = tiles[ti].kc1;
            for (int kc = kc0; kc < kc1; ++kc, ++c) {
                const int s = c % STAGES;
                const int b = G & 1;
                const bool gfirst = ((kc - kc0) % GROUP) == 0,
                           glast = ((kc - kc0) % GROUP) == GROUP - 1 || kc == kc1 - 1;
                if (gfirst) {
                    mbar_wait(smem_u32(&acce_b[b]), ((G >> 1) & 1) ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                mbar_wait(smem_u32(&full_b[s]), (c / STAGES) & 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (lane == 0) {
                    const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
                    const uint64_t a_b = smem_desc(st), a_s = smem_desc(st + A_BYTES);
                    const uint64_t bb = smem_desc(st + 2 * A_BYTES), bs = smem_desc(st + 2 * A_BYTES + B_BYTES);
                    const uint32_t d = tmem + (uint32_t)(b * BNW);
                    const int ksteps = min(BKE, K - kc * BKE + KS - 1) / KS;
                    for (int k = 0; k < ksteps; ++k) {
                        const uint64_t off = (uint64_t)(2 * k);
                        mma_op<F16>(d, a_b + off, bb + off, idesc, !gfirst || k != 0);
                        mma_op<F16>(d, a_b + off, bs + off, idesc, 1);
                        mma_op<F16>(d, a_s + off, bb + off, idesc, 1);
                    }
                    mma_commit(smem_u32(&empty_b[s]));
                    if (glast) mma_commit(smem_u32(&accf_b[b]));
                }
                __syncwarp();
                if (glast) ++G;
            }
        }
    } else if (warp >= EPI_WARP0 && DRAIN) {
        // ---------------- drains: warp -> (lane quarter, column half); fp32 register sums, then atomics
        const int wq = warp & 3, half = (warp - EPI_WARP0) >> 2;
        int G = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
            const Tile tl = tiles[ti];
            float acc[BN];
#pragma unroll
            for (int j = 0; j < BN; ++j) acc[j] = 0.f;
            const int ngroups = (tl.kc1 - tl.kc0 + GROUP - 1) / GROUP;
            for (int g = 0; g < ngroups; ++g, ++G) {
                const int b = G & 1;
                mbar_wait(smem_u32(&accf_b[b]), (G >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (half * BN < tl.np) drain_add(tmem, wq, b * BNW + half * BN, acc);
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&acce_b[b]));
            }
            const int row = tl.m0 + 32 * wq + lane;
            const int2* pp = pairs + tl.p0 + half * BN;
            const int npl = tl.np - half * BN;           // this warp's columns
            if (row - lane < M) {
                const int rowc = row < M ? row : row - 32;
#pragma unroll
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    if (c0 >= npl) break;
                    int trow;
                    float sc;
                    epi_cols_load<F16>(pp, c0, npl, lane, bscale, ascale_inv, trow, sc);
#pragma unroll
                    for (int j = 0; j < 32; ++j) epi_col_add(Y, ldy, rowc, row < M, trow, sc, j, acc[c0 + j]);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        int c = 0, it = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++it) {
            const int ab = it & 1;
            const uint32_t nmma = (uint32_t)((tiles[ti].np + 15) & ~15);
            const uint32_t idesc = make_idesc<F16>(nmma, BM);
            mbar_wait(smem_u32(&acce_b[ab]), ((it >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int kc0 = tiles[ti].kc0, kc1 = tiles[ti].kc1;
            for (int kc = kc0; kc < kc1; ++kc, ++c) {
                const int s = c % STAGES;
                mbar_wait(smem_u32(&full_b[s]), (c / STAGES) & 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // cp.async data -> tensor core
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (lane == 0) {
                    const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
                    const uint64_t a_b = smem_desc(st), a_s = smem_desc(st + A_BYTES);
                    const uint64_t bb = smem_desc(st + 2 * A_BYTES), bs = smem_desc(st + 2 * A_BYTES + B_BYTES);
                    const uint32_t d = tmem + (uint32_t)(ab * BNW);
                    const int ksteps = min(BKE, K - kc * BKE + KS - 1) / KS;
                    for (int k = 0; k < ksteps; ++k) {
                        const uint64_t off = (uint64_t)(2 * k);
                        mma_op<F16>(d, a_b + off, bb + off, idesc, kc != kc0 || k != 0);
                        mma_op<F16>(d, a_b + off, bs + off, idesc, 1);
                        mma_op<F16>(d, a_s + off, bb + off, idesc, 1);
                    }
                    mma_commit(smem_u32(&empty_b[s]));
                    if (kc == kc1 - 1) mma_commit(smem_u32(&accf_b[ab]));
                }
                __syncwarp();
            }
        }
    } else if (warp >= EPI_WARP0 && warp < EPI_WARP0 + 4) {
        // ---------------- epilogue: TMEM -> fp64 atomics, 32 columns at a time
        const int wq = warp - EPI_WARP0;
        int it = 0;
        for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++it) {
            const Tile tl = tiles[ti];
            const int ab = it & 1;
            mbar_wait(smem_u32(&accf_b[ab]), (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int2* pp = pairs + tl.p0;
            const int row = tl.m0 + 32 * wq + lane;
            const int rowc = row < M ? row : row - 32;
            const int np_epi = row - lane < M ? tl.np : 0;       // (warp-uniform) some of this warp's rows exist
#pragma unroll 1
            for (int c0 = 0; c0 < np_epi; c0 += 32) {
                int trow;
                float sc;
                epi_cols_load<F16>(pp, c0, tl.np, lane, bscale, ascale_inv, trow, sc);
                uint32_t v[32];
                tmem_ld32(tmem + ((uint32_t)(32 * wq) << 16) + (uint32_t)(ab * BNW + c0), v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < 32; ++j) epi_col_add(Y, ldy, rowc, row < M, trow, sc, j, __uint_as_float(v[j]));
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&acce_b[ab]));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// round-to-nearest TF32 (low 13 mantissa bits zero): both halves of the split are exact TF32
// values, so the tensor core's own fp32->tf32 handling (truncation) never applies, and the
// two rounding errors are unbiased (truncated remainders are one-signed and their dropped
// product A_s B_s biases long dot products; measured 7e-6 -> see DESIGN.md Sec. 6).
__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ float to_tf32(double x) { return to_tf32((float)x); }

// split fp32 rows into a TF32 head and a TF32 remainder (columns >= K untouched)
template <class XT>
__global__ void split_rows_kernel(const XT* __restrict__ X, int ld, int64_t row0, int64_t nrows, int K,
                                  float* __restrict__ Xb, float* __restrict__ Xs) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nrows * K) return;
    const int64_t r = row0 + i / K;
    const int c = (int)(i % K);
    const XT x = X[r * ld + c];
    const float b = to_tf32(x);
    Xb[r * ld + c] = b;
    Xs[r * ld + c] = to_tf32(x - (XT)b);
}

// ---- FP16 head / remainder split (3xFP16 translations) ----
// An fp16 value carries the same 11 significand bits as a TF32 one, and the tensor core
// multiplies fp16 operands at twice the TF32 rate (kind::f16, K = 16 per MMA).  The 5-bit
// exponent is handled by scaling with powers of two (exact): each row is scaled so that its
// largest magnitude lies in [2^12, 2^13); head = rn_fp16(s x), remainder = rn_fp16(s x - head).
// Entries more than 2^-15 below the row maximum have a subnormal remainder (absolute spacing
// 2^-24, i.e. 2^-37 of the row maximum): the split keeps min(22 bits relative, 2^-37 of the
// largest entry) -- for a dot product the same error level as the TF32 split.

// rows [row0, row0 + nrows) of the fp64 state X (row stride ldx) -> Xh / Xr (row stride ldh
// halves) and the factor that undoes the row's scaling; a warp per row
__global__ void split_rows_h_kernel(const double* __restrict__ X, int ldx, int64_t row0, int64_t nrows, int K,
                                    __half* __restrict__ Xh, __half* __restrict__ Xr, int ldh,
                                    float* __restrict__ inv_scale) {
    const int lane = threadIdx.x & 31;
    const int64_t r = row0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (r >= row0 + nrows) return;
    const double2* src = reinterpret_cast<const double2*>(X + r * ldx);
    const int K2 = K >> 1;                       // K even (3 n_e, n_e even)
    constexpr int NV = 16;                       // up to 1024 columns per row held in registers
    double2 v[NV];
    float amax = 0.f;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const int j = q * 32 + lane;
        v[q] = j < K2 ? src[j] : make_double2(0.0, 0.0);
        amax = fmaxf(amax, fmaxf(fabsf((float)v[q].x), fabsf((float)v[q].y)));
    }
    for (int j = NV * 32 + lane; j < K2; j += 32) {   // longer rows: second pass re-reads them
        const double2 w = src[j];
        amax = fmaxf(amax, fmaxf(fabsf((float)w.x), fabsf((float)w.y)));
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    const float sc = pow2_scale(amax);
    if (lane == 0) inv_scale[r] = 1.f / sc;
    __half2* dh = reinterpret_cast<__half2*>(Xh + r * ldh);
    __half2* dr = reinterpret_cast<__half2*>(Xr + r * ldh);
    auto put = [&](int j, double2 w) {
        const float a = (float)(w.x * (double)sc), b = (float)(w.y * (double)sc);   // exact scaling, one rounding
        const __half ha = __float2half_rn(a), hb = __float2half_rn(b);
        dh[j] = __halves2half2(ha, hb);
        dr[j] = __halves2half2(__float2half_rn(a - __half2float(ha)), __float2half_rn(b - __half2float(hb)));
    };
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const int j = q * 32 + lane;
        if (j < K2) put(j, v[q]);
    }
    for (int j = NV * 32 + lane; j < K2; j += 32) put(j, src[j]);
}

// largest magnitude of a float array (bit pattern of |x| is monotone as an unsigned integer)
__global__ void absmax_kernel(const float* __restrict__ X, int64_t n, unsigned* __restrict__ out) {
    unsigned m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, __float_as_uint(fabsf(X[i])));
#pragma unroll
    for (int off = 16; off; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// operator rows [nrows][ld] fp32 -> scaled fp16 head / remainder [nrows][ldh] (one scale for the set)
__global__ void split_ops_h_kernel(const float* __restrict__ X, int ld, int64_t nrows, int K, float sc,
                                   __half* __restrict__ Xh, __half* __restrict__ Xr, int ldh) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nrows * K) return;
    const int64_t r = i / K;
    const int c = (int)(i % K);
    const float a = X[r * ld + c] * sc;
    const __half h = __float2half_rn(a);
    Xh[r * ldh + c] = h;
    Xr[r * ldh + c] = __float2half_rn(a - __half2float(h));
}

// ------------------------------------------------------------------ level chain (M2M, L2L)
// The upward (M2M, fine to coarse) and downward (L2L, coarse to fine) passes are chains of
// small dependent contractions, one per tree level.  Launched level by
// level they cost a split launch (fp64 state -> TF32 head / remainder) plus a translation
// launch per level, and the coarse levels are all latency (kernel prologue, pipeline fill,
// epilogue, teardown).  This persistent kernel runs a whole chain in one cooperative launch:
// per level, all threads of the grid split that level's source rows (grid-stride sweep), a
// grid-wide barrier, the level's translation tiles (data flow of tc_pairs_fast_kernel<false>:
// two 128-row operator slices x up to 128 pairs, TMA A, cp.async B, full-K TMEM accumulation,
// fp64 atomic epilogue), another grid barrier.  The upward chain's last sweep also splits the
// coarsest rows, which the M2L reads.
// (A variant whose producers read the fp64 rows and split them while staging was measured 4x
// slower per level: register-staged loads cannot run ahead of the ring like cp.async.)
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// grid-wide barrier number `k` (0, 1, ...): the CTA's prior writes are released, every CTA's
// writes before its arrival are acquired (the acquire also invalidates this SM's L1)
__device__ __forceinline__ void grid_barrier(unsigned* gbar, unsigned k) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gbar) : "memory");
        const unsigned target = (k + 1) * gridDim.x;
        while (ld_acquire_u32(gbar) < target) __nanosleep(32);
    }
    __syncthreads();
}

// rows [row0, row0 + nrows) of X split into Xb / Xs: a warp per row, each lane up to 8
// independent 16-B loads in flight (a grid-stride element loop was latency bound: ~0.3 TB/s)
__device__ __forceinline__ void split_sweep(const double* X, int ldx, int64_t row0, int64_t nrows, int K,
                                            float* __restrict__ Xb, float* __restrict__ Xs) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int K2 = K >> 1;                       // K is even (3 n_e, n_e even)
    for (int64_t r = row0 + gw; r < row0 + nrows; r += nw) {
        const double2* src = reinterpret_cast<const double2*>(X + r * ldx);
        float2* db = reinterpret_cast<float2*>(Xb + r * ldx);
        float2* ds = reinterpret_cast<float2*>(Xs + r * ldx);
        for (int j0 = 0; j0 < K2; j0 += 8 * 32) {
            double2 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int j = j0 + q * 32 + lane;
                v[q] = j < K2 ? src[j] : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int j = j0 + q * 32 + lane;
                if (j < K2) {
                    const float h0 = to_tf32(v[q].x), h1 = to_tf32(v[q].y);
                    db[j] = make_float2(h0, h1);
                    ds[j] = make_float2(to_tf32(v[q].x - (double)h0), to_tf32(v[q].y - (double)h1));
                }
            }
        }
    }
}

__global__ void __launch_bounds__(fast::THREADS, 1)
tc_chain_kernel(const __grid_constant__ CUtensorMap mapAb, const __grid_constant__ CUtensorMap mapAs,
                const double* X, int ldx, float* Xb, float* Xs, const Tile* __restrict__ tiles,
                const int2* __restrict__ pairs, int M, int K, double* Y, int ldy, const __grid_constant__ ChainArgs ca,
                unsigned* __restrict__ gbar) {
    constexpr int MT = fast::MT, STAGES = fast::STAGES, STAGE_BYTES = fast::STAGE_BYTES, TMEM_COLS = fast::TMEM_COLS;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(smem + STAGES * STAGE_BYTES);
    uint64_t* full_b = bars;                     // [STAGES]
    uint64_t* empty_b = bars + STAGES;           // [STAGES]
    uint64_t* accf_b = bars + 2 * STAGES;        // [2]
    uint64_t* acce_b = bars + 2 * STAGES + 2;    // [2]
    uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 4);
    unsigned long long* trace = reinterpret_cast<unsigned long long*>(gbar + 2);
    auto stamp = [&](int i) {                    // diagnostics (EBEM_CHAIN_TRACE): level end times
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[i] = t;
        }
    };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full_b[s]), 1 + 32 * fast::NPROD);   // A expect_tx + cp.async arrivals
            mbar_init(smem_u32(&empty_b[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&accf_b[b]), 1);
            mbar_init(smem_u32(&acce_b[b]), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    stamp(0);

    int c = 0, it = 0;                           // stage uses / accumulator uses (per role)
    unsigned nb = 0;                             // grid barriers passed
    for (int lv = 0; lv < ca.nlev; ++lv) {
        split_sweep(X, ldx, ca.row0[lv], ca.nrows[lv], K, Xb, Xs);   // this level's source rows
        grid_barrier(gbar, nb++);
        const int tb = ca.lvl_tile[lv], te = ca.lvl_tile[lv + 1];
        if (warp == 0 || warp == 2 || warp == 3) {
            // ---------------- producers (as tc_pairs_fast_kernel)
            const int pi = warp == 0 ? 0 : warp - 1;
            const int piece = lane & 7, rsub = lane >> 3;
            for (int ti = tb + blockIdx.x; ti < te; ti += gridDim.x) {
                const Tile tl = tiles[ti];
                int64_t srow[fast::NG];
#pragma unroll
                for (int g = 0; g < fast::NG; ++g) {
                    const int r = rsub + 4 * (pi + fast::NPROD * g);
                    srow[g] = (int64_t)__ldg(&pairs[tl.p0 + min(r, tl.np - 1)].y) * ldx;
                }
                const int ngrp = ((tl.np + 15) & ~15) / 4;
                for (int kc = tl.kc0; kc < tl.kc1; ++kc, ++c) {
                    const int s = c % STAGES;
                    mbar_wait(smem_u32(&empty_b[s]), ((c / STAGES) & 1) ^ 1);
                    uint8_t* st = smem + s * STAGE_BYTES;
                    const uint32_t full = smem_u32(&full_b[s]);
                    if (pi == 0 && lane == 0) {
                        mbar_expect_tx(full, 2 * MT * OPND_BYTES);
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            tma_load_3d(smem_u32(st + (2 * mt) * OPND_BYTES), &mapAb, kc * BK, tl.m0 + mt * BM, tl.op,
                                        full);
                            tma_load_3d(smem_u32(st + (2 * mt + 1) * OPND_BYTES), &mapAs, kc * BK, tl.m0 + mt * BM,
                                        tl.op, full);
                        }
                    }
                    const int col = kc * BK + 4 * piece;
                    const uint32_t nbytes = col < ldx ? 16u : 0u;
                    const uint32_t b0 = smem_u32(st + 2 * MT * OPND_BYTES);
                    const uint32_t b1 = b0 + OPND_BYTES;
#pragma unroll
                    for (int g = 0; g < fast::NG; ++g) {
                        const int grp = pi + fast::NPROD * g;
                        if (grp < ngrp) {
                            const int r = rsub + 4 * grp;
                            const int64_t off = srow[g] + col;
                            const uint32_t so = (uint32_t)(r * 128 + ((piece ^ (r & 7)) * 16));
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(b0 + so),
                                         "l"(nbytes ? Xb + off : Xb), "r"(nbytes)
                                         : "memory");
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(b1 + so),
                                         "l"(nbytes ? Xs + off : Xs), "r"(nbytes)
                                         : "memory");
                        }
                    }
                    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full) : "memory");
                }
            }
        } else if (warp == 1) {
            // ---------------- MMA issuer (as tc_pairs_fast_kernel<false>)
            for (int ti = tb + blockIdx.x; ti < te; ti += gridDim.x, ++it) {
                const int ab = it & 1;
                const uint32_t nmma = (uint32_t)((tiles[ti].np + 15) & ~15);
                const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((nmma >> 3) << 17) |
                                       ((uint32_t)(BM >> 4) << 24);
                mbar_wait(smem_u32(&acce_b[ab]), ((it >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const int kc0 = tiles[ti].kc0, kc1 = tiles[ti].kc1;
                for (int kc = kc0; kc < kc1; ++kc, ++c) {
                    const int s = c % STAGES;
                    mbar_wait(smem_u32(&full_b[s]), (c / STAGES) & 1);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    if (lane == 0) {
                        const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
                        const uint64_t bb = smem_desc(st + 2 * MT * OPND_BYTES),
                                       bs = smem_desc(st + (2 * MT + 1) * OPND_BYTES);
                        const int ksteps = min(BK, K - kc * BK + 7) / 8;
                        for (int k = 0; k < ksteps; ++k) {
                            const uint64_t off = (uint64_t)(2 * k);
#pragma unroll
                            for (int mt = 0; mt < MT; ++mt) {
                                const uint64_t a_b = smem_desc(st + (2 * mt) * OPND_BYTES) + off;
                                const uint64_t a_s = smem_desc(st + (2 * mt + 1) * OPND_BYTES) + off;
                                const uint32_t d = tmem + (uint32_t)((ab * MT + mt) * BN);
                                mma_tf32(d, a_b, bb + off, idesc, kc != kc0 || k != 0);
                                mma_tf32(d, a_b, bs + off, idesc, 1);
                                mma_tf32(d, a_s, bb + off, idesc, 1);
                            }
                        }
                        mma_commit(smem_u32(&empty_b[s]));
                        if (kc == kc1 - 1) mma_commit(smem_u32(&accf_b[ab]));
                    }
                    __syncwarp();
                }
            }
        } else if (warp >= EPI_WARP0) {
            // ---------------- epilogue: TMEM -> fp64 atomics (REDs; no per-thread fence, which
            // would make them returning ATOMs: thread 0's release after the CTA barrier covers them)
            const int wq = warp - EPI_WARP0;
            for (int ti = tb + blockIdx.x; ti < te; ti += gridDim.x, ++it) {
                const Tile tl = tiles[ti];
                const int ab = it & 1;
                mbar_wait(smem_u32(&accf_b[ab]), (it >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const int2* pp = pairs + tl.p0;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const int row = tl.m0 + mt * BM + 32 * wq + lane;
#pragma unroll 1
                    for (int c0 = 0; c0 < tl.np; c0 += 32) {
                        uint32_t v[32];
                        tmem_ld32(tmem + ((uint32_t)(32 * wq) << 16) + (uint32_t)((ab * MT + mt) * BN + c0), v);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (row < M) {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (c0 + j < tl.np)
                                    atomicAdd(Y + (int64_t)__ldg(&pp[c0 + j].x) * ldy + row,
                                              (double)__uint_as_float(v[j]));
                        }
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&acce_b[ab]));
            }
        }
        grid_barrier(gbar, nb++);                // this level's results complete and visible
        stamp(lv + 1);
    }
    // the coarsest rows (upward chain: read by the M2L)
    if (ca.tail_rows > 0) split_sweep(X, ldx, ca.tail_row0, ca.tail_rows, K, Xb, Xs);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encoder() {
    static EncodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        EB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        EB_REQUIRE(p && q == cudaDriverEntryPointSuccess, "cuTensorMapEncodeTiled not available");
        fn = (EncodeTiled)p;
    }
    return fn;
}

}  // namespace tc

// A maps: [nops][M][ld] fp32, box {32, 128, 1}
void tc_make_map_a(CUtensorMap* m, const float* base, int nops, int M, int K, int ld) {
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)M, (cuuint64_t)nops};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)M * ld * 4};
    cuuint32_t box[3] = {tc::BK, tc::BM, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = tc::encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    EB_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (A) failed: " + std::to_string((int)r));
}

// B maps: [rows][ld] fp32, gathered 4 rows at a time, box {32, 1}
void tc_make_map_b(CUtensorMap* m, const float* base, int64_t rows, int K, int ld) {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)std::max<int64_t>(rows, 1)};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {tc::BK, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = tc::encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    EB_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (B) failed: " + std::to_string((int)r));
}

// A maps of the FP16 operator copies: [nops][M][ldh] halves, box {64, 128, 1} (128-B rows)
void tc_make_map_a_h(CUtensorMap* m, const __half* base, int nops, int M, int K, int ldh) {
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)M, (cuuint64_t)nops};
    cuuint64_t strides[2] = {(cuuint64_t)ldh * 2, (cuuint64_t)M * ldh * 2};
    cuuint32_t box[3] = {64, tc::BM, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = tc::encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, (void*)base, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    EB_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (A, fp16) failed: " + std::to_string((int)r));
}

// scaled FP16 head / remainder copies of an operator set; returns the factor undoing the scale
float tc_split_ops_h(const float* X, int ld, int64_t nrows, int K, __half* Xh, __half* Xr, int ldh, cudaStream_t s) {
    DBuf<unsigned> m;
    m.alloc(1);
    m.zero(s);
    tc::absmax_kernel<<<1024, 256, 0, s>>>(X, nrows * ld, m.p);
    EB_CHECK_LAUNCH();
    unsigned bits = 0;
    EB_CUDA(cudaMemcpyAsync(&bits, m.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    EB_CUDA(cudaStreamSynchronize(s));
    float amax;
    std::memcpy(&amax, &bits, sizeof(float));
    const float sc = (amax > 0.f && std::isfinite(amax)) ? std::scalbn(1.f, 12 - std::ilogb(amax)) : 1.f;
    tc::split_ops_h_kernel<<<ceil_div(nrows * K, 256), 256, 0, s>>>(X, ld, nrows, K, sc, Xh, Xr, ldh);
    EB_CHECK_LAUNCH();
    return 1.f / sc;
}

void tc_split_rows_h(const double* X, int ldx, int64_t row0, int64_t nrows, int K, __half* Xh, __half* Xr, int ldh,
                     float* inv_scale, cudaStream_t s) {
    if (nrows <= 0) return;
    tc::split_rows_h_kernel<<<ceil_div(nrows * 32, 256), 256, 0, s>>>(X, ldx, row0, nrows, K, Xh, Xr, ldh, inv_scale);
    EB_CHECK_LAUNCH();
}

template <class XT>
void tc_split_rows(const XT* X, int ld, int64_t row0, int64_t nrows, int K, float* Xb, float* Xs, cudaStream_t s) {
    if (nrows <= 0) return;
    tc::split_rows_kernel<XT><<<ceil_div(nrows * K, 256), 256, 0, s>>>(X, ld, row0, nrows, K, Xb, Xs);
    EB_CHECK_LAUNCH();
}
template void tc_split_rows<float>(const float*, int, int64_t, int64_t, int, float*, float*, cudaStream_t);
template void tc_split_rows<double>(const double*, int, int64_t, int64_t, int, float*, float*, cudaStream_t);

// Tiles in operator-major order (ordering the M2L tiles by target-row chunks first kept W
// and Z rows in L2 across operators but re-read the operators per chunk: no faster).  Launches with fewer tiles than SMs (the coarse M2M/L2L
// levels) split K over several CTAs: a lone tile streams its 15 K chunks through one SM in
// ~20 us, while its partial sums are added by the fp64 atomics of the epilogue anyway.
int tc_fast_tile_mode(int M) {
    // Tile shape of the full-chain translations by the operator's row count M = 3 n_e: the
    // two-slice tiles (256 rows x 128 pairs: every gathered row feeds 256 outputs) unless they
    // pad M more than the wide tiles (128 rows x 256 pairs) do.  p = 6 (456 rows): both pad to
    // 512, two-slice (matvec 4.46 vs 4.61 ms); p = 8 (888 rows): 1024 vs 896 rows, wide (BEM
    // operator M2L 24.6 vs 28.4 ms; configs[3] 8.76 vs 8.73 ms).  EBEM_M2L_WIDE=0 / 1 forces
    // one of them.
    if (const char* e = std::getenv("EBEM_M2L_WIDE")) return std::atoi(e) == 1 ? 2 : 1;
    const int two = (M + 2 * tc::BM - 1) / (2 * tc::BM) * 2 * tc::BM, wide = (M + tc::BM - 1) / tc::BM * tc::BM;
    return two > wide ? 2 : 1;
}

void tc_build_tiles(OpPairs& P, int M, int K, int mode, int bke, int cs) {
    std::vector<tc::Tile> t;
    const int mstep = mode == 1 ? tc::fast::MT * tc::BM : tc::BM;
    const int bn = mode == 2 ? tc::wide::BNW : tc::BN;
    const int nk = (K + bke - 1) / bke;          // K chunks of 128 B: 32 TF32 or 64 FP16 elements
    P.tile_mode = mode;
    P.tile_bke = bke;
    P.tile_cs = 1;
    if (mode == 1 && cs > 1) {
        // cluster tiles (tc_pairs_mc_kernel): cs consecutive pair blocks of one operator and row
        // slice pair go to the cs CTAs of a cluster (an operator's last cluster tile is padded
        // with empty blocks)
        EB_REQUIRE(cs == 2 || cs == 4, "internal: cluster size");
        P.tile_mode = 3;
        P.tile_cs = cs;
        for (int o = 0; o < P.nops; ++o) {
            const int a = P.op_ptr_h[o], e = P.op_ptr_h[o + 1];
            for (int p0 = a; p0 < e; p0 += cs * bn)
                for (int m0 = 0; m0 < M; m0 += mstep)
                    for (int r = 0; r < cs; ++r) {
                        const int q = p0 + r * bn;
                        t.push_back({o, q < e ? q : a, q < e ? std::min(bn, e - q) : 0, m0, 0, nk});
                    }
        }
        P.ntiles = (int)t.size() / cs;
        P.tiles.alloc(std::max<size_t>(t.size(), 1) * sizeof(tc::Tile) / sizeof(int));
        if (!t.empty()) EB_CUDA(cudaMemcpy(P.tiles.p, t.data(), t.size() * sizeof(tc::Tile), cudaMemcpyHostToDevice));
        return;
    }
    // op-major; the row blocks of one pair group are consecutive (run side by side on
    // neighbouring CTAs, so the second load of the same gathered B rows hits L2)
    for (int o = 0; o < P.nops; ++o)
        for (int p0 = P.op_ptr_h[o]; p0 < P.op_ptr_h[o + 1]; p0 += bn)
            for (int m0 = 0; m0 < M; m0 += mstep)
                t.push_back({o, p0, std::min(bn, P.op_ptr_h[o + 1] - p0), m0, 0, nk});
    const int nsplit = t.empty() ? 1 : std::max(1, std::min(nk / 3, num_sms() / (int)t.size()));
    if (nsplit > 1) {
        std::vector<tc::Tile> u;
        for (const tc::Tile& x : t)
            for (int q = 0; q < nsplit; ++q) {
                tc::Tile y = x;
                y.kc0 = nk * q / nsplit;
                y.kc1 = nk * (q + 1) / nsplit;
                u.push_back(y);
            }
        t.swap(u);
    }
    P.ntiles = (int)t.size();
    P.tiles.alloc(std::max<size_t>(t.size(), 1) * sizeof(tc::Tile) / sizeof(int));
    if (!t.empty()) EB_CUDA(cudaMemcpy(P.tiles.p, t.data(), t.size() * sizeof(tc::Tile), cudaMemcpyHostToDevice));
}

int tc_fast_smem_bytes() { return tc::fast::SMEM_BYTES; }

template <class KernelT>
static void launch_fast(KernelT fn, bool& attr, int smem, int threads, const OpPairs& P, const CUtensorMap& Ab,
                        const CUtensorMap& As, const void* Bb, const void* Bs, int ldb, int M, int K, double* Y,
                        int ldy, const float* bscale, float ascale_inv, cudaStream_t s) {
    if (!attr) {
        EB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    const int grid = std::min(P.ntiles, num_sms());
    fn<<<grid, threads, smem, s>>>(Ab, As, Bb, Bs, ldb, reinterpret_cast<const tc::Tile*>(P.tiles.p), P.ntiles,
                                   P.pairs.p, M, K, Y, ldy, bscale, ascale_inv);
    EB_CHECK_LAUNCH();
}

// f16: Ab / As are FP16 operator maps (tc_make_map_a_h), Bb / Bs fp16 rows of ldb halves with
// the per-row factors bscale (tc_split_rows_h) and the operator set's factor ascale_inv; the
// tiles must have been built with 64-element chunks.  Otherwise TF32 operands in fp32 words.
void tc_pairs_gemm_fast(const OpPairs& P, const CUtensorMap& Ab, const CUtensorMap& As, const void* Bb,
                        const void* Bs, int ldb, int M, int K, double* Y, int ldy, bool drain, cudaStream_t s,
                        bool f16, const float* bscale, float ascale_inv) {
    if (P.ntiles == 0) return;
    EB_REQUIRE(P.tile_bke == (f16 ? 64 : 32), "internal: translation tiles built for the other operand type");
    if (P.tile_mode == 3) {
        EB_REQUIRE(!drain, "internal: cluster tiles with the drained kernel");
        const int cs = P.tile_cs;
        void (*fn)(const CUtensorMap, const CUtensorMap, const void*, const void*, int, const tc::Tile*, int, const int2*,
                   int, int, double*, int, const float*, float) =
            cs == 2 ? (f16 ? tc::tc_pairs_mc_kernel<true, 2> : tc::tc_pairs_mc_kernel<false, 2>)
                    : (f16 ? tc::tc_pairs_mc_kernel<true, 4> : tc::tc_pairs_mc_kernel<false, 4>);
        static bool mattr[2][2] = {};
        if (!mattr[cs == 4][f16]) {
            EB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::fast::SMEM_BYTES));
            mattr[cs == 4][f16] = true;
        }
        const int ncl = std::min(P.ntiles, num_sms() / cs);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ncl * cs);
        cfg.blockDim = dim3(tc::fast::THREADS);
        cfg.dynamicSmemBytes = tc::fast::SMEM_BYTES;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        EB_CUDA(cudaLaunchKernelEx(&cfg, fn, Ab, As, Bb, Bs, ldb, reinterpret_cast<const tc::Tile*>(P.tiles.p), P.ntiles,
                                   (const int2*)P.pairs.p, M, K, Y, ldy, bscale, ascale_inv));
        EB_CHECK_LAUNCH();
        return;
    }
    EB_REQUIRE(P.tile_mode == 1 || P.tile_mode == 2, "internal: fast kernel needs two-slice or wide tiles");
    static bool attr[2][2][2] = {};
    const bool w = P.tile_mode == 2;
    const int smem = w ? tc::wide::SMEM_BYTES : tc::fast::SMEM_BYTES;
    const int threads = drain ? 384 : (w ? tc::wide::THREADS : tc::fast::THREADS);
#define EB_TC_LAUNCH(KERNEL) \
    launch_fast(KERNEL, attr[w][drain][f16], smem, threads, P, Ab, As, Bb, Bs, ldb, M, K, Y, ldy, bscale, ascale_inv, s)
    if (w) {
        if (drain) { if (f16) EB_TC_LAUNCH((tc::tc_pairs_wide_kernel<true, true>)); else EB_TC_LAUNCH((tc::tc_pairs_wide_kernel<true, false>)); }
        else { if (f16) EB_TC_LAUNCH((tc::tc_pairs_wide_kernel<false, true>)); else EB_TC_LAUNCH((tc::tc_pairs_wide_kernel<false, false>)); }
    } else {
        if (drain) { if (f16) EB_TC_LAUNCH((tc::tc_pairs_fast_kernel<true, true>)); else EB_TC_LAUNCH((tc::tc_pairs_fast_kernel<true, false>)); }
        else { if (f16) EB_TC_LAUNCH((tc::tc_pairs_fast_kernel<false, true>)); else EB_TC_LAUNCH((tc::tc_pairs_fast_kernel<false, false>)); }
    }
#undef EB_TC_LAUNCH
}

void tc_pairs_gemm(const OpPairs& P, const CUtensorMap& Ab, const CUtensorMap& As, const CUtensorMap& Bb,
                   const CUtensorMap& Bs, int M, int K, double* Y, int ldy, cudaStream_t s) {
    if (P.ntiles == 0) return;
    static bool attr = false;
    if (!attr) {
        EB_CUDA(cudaFuncSetAttribute(tc::tc_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     tc::SMEM_BYTES));
        attr = true;
    }
    const int grid = std::min(P.ntiles, num_sms());
    tc::tc_pairs_kernel<<<grid, tc::THREADS, tc::SMEM_BYTES, s>>>(
        Ab, As, Bb, Bs, reinterpret_cast<const tc::Tile*>(P.tiles.p), P.ntiles, P.pairs.p, M, K, Y, ldy);
    EB_CHECK_LAUNCH();
}


// ------------------------------------------------------------------ level chain (host)
// Tiles of every level of a chain in execution order (two-slice tiles as tc_build_tiles
// mode 1, split K on levels with fewer tiles than SMs), over one concatenated pair array.
void tc_build_chain(Chain& ch, const std::vector<const OpPairs*>& levels, const std::vector<int64_t>& row0,
                    const std::vector<int64_t>& nrows, int M, int K, cudaStream_t s) {
    std::vector<tc::Tile> t;
    std::vector<int> lt(1, 0);
    int64_t np = 0;
    for (const OpPairs* P : levels) np += P->npairs;
    ch.pairs.alloc(std::max<int64_t>(np, 1));
    int64_t base = 0;
    const int mstep = tc::fast::MT * tc::BM;
    const int nk = (K + tc::BK - 1) / tc::BK;
    for (const OpPairs* P : levels) {
        if (P->npairs) d2d(ch.pairs.p + base, P->pairs.p, (size_t)P->npairs, s);
        std::vector<tc::Tile> u;
        for (int o = 0; o < P->nops; ++o)
            for (int p0 = P->op_ptr_h[o]; p0 < P->op_ptr_h[o + 1]; p0 += tc::BN)
                for (int m0 = 0; m0 < M; m0 += mstep)
                    u.push_back({o, (int)(base + p0), std::min(tc::BN, P->op_ptr_h[o + 1] - p0), m0, 0, nk});
        const int nsplit = u.empty() ? 1 : std::max(1, std::min(nk / 3, num_sms() / (int)u.size()));
        for (const tc::Tile& x : u)
            for (int q = 0; q < nsplit; ++q) {
                tc::Tile y = x;
                y.kc0 = nk * q / nsplit;
                y.kc1 = nk * (q + 1) / nsplit;
                t.push_back(y);
            }
        lt.push_back((int)t.size());
        base += P->npairs;
    }
    EB_REQUIRE(levels.size() <= (size_t)MAXLEVEL && row0.size() == levels.size() && nrows.size() == levels.size(),
               "internal: chain levels");
    ch.nlev = (int)levels.size();
    ch.lvl_tile = lt;
    ch.row0 = row0;
    ch.nrows = nrows;
    ch.tiles.alloc(std::max<size_t>(t.size(), 1) * sizeof(tc::Tile) / sizeof(int));
    if (!t.empty()) EB_CUDA(cudaMemcpyAsync(ch.tiles.p, t.data(), t.size() * sizeof(tc::Tile), cudaMemcpyHostToDevice, s));
    ch.bar.alloc(4 + 2 * (MAXLEVEL + 1));          // counter, pad, then level timestamps (u64)
    EB_CUDA(cudaStreamSynchronize(s));
}

void tc_chain_run(const Chain& ch, const CUtensorMap& Ab, const CUtensorMap& As, const double* X, int ldx, float* Xb,
                  float* Xs, int M, int K, double* Y, int ldy, int64_t tail_row0, int64_t tail_rows, cudaStream_t s) {
    if (ch.nlev == 0 && tail_rows <= 0) return;
    ChainArgs ca{};
    ca.nlev = ch.nlev;
    for (int i = 0; i <= ch.nlev; ++i) ca.lvl_tile[i] = ch.lvl_tile[i];
    for (int i = 0; i < ch.nlev; ++i) {
        ca.row0[i] = ch.row0[i];
        ca.nrows[i] = ch.nrows[i];
    }
    ca.tail_row0 = tail_row0;
    ca.tail_rows = tail_rows;
    static bool attr = false;
    if (!attr) {
        EB_CUDA(cudaFuncSetAttribute(tc::tc_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     tc::fast::SMEM_BYTES));
        attr = true;
    }
    EB_CUDA(cudaMemsetAsync(ch.bar.p, 0, sizeof(unsigned), s));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(num_sms());                 // one CTA per SM (its shared memory allows no more)
    cfg.blockDim = dim3(tc::fast::THREADS);
    cfg.dynamicSmemBytes = tc::fast::SMEM_BYTES;
    cfg.stream = s;
    // The grid barrier needs every CTA resident: one CTA per SM always fits an idle SM, and
    // the only concurrent kernels (the stream-B P2P kernels) never wait on this one, so CTAs
    // not yet resident start as those leave.  EBEM_CHAIN_COOP=1 launches cooperatively (the
    // driver then checks residency; measured 0.2-0.4 ms slower end to end)
    static const bool coop = std::getenv("EBEM_CHAIN_COOP") && std::atoi(std::getenv("EBEM_CHAIN_COOP")) == 1;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = coop ? 1 : 0;
    EB_CUDA(cudaLaunchKernelEx(&cfg, tc::tc_chain_kernel, Ab, As, X, ldx, Xb, Xs,
                               reinterpret_cast<const tc::Tile*>(ch.tiles.p), (const int2*)ch.pairs.p, M, K, Y, ldy, ca,
                               (unsigned*)ch.bar.p));
    EB_CHECK_LAUNCH();
    static const bool trace = std::getenv("EBEM_CHAIN_TRACE") != nullptr;
    if (trace) {
        std::vector<unsigned long long> ts(ch.nlev + 1);
        EB_CUDA(cudaMemcpyAsync(ts.data(), ch.bar.p + 2, sizeof(unsigned long long) * (ch.nlev + 1),
                                cudaMemcpyDeviceToHost, s));
        EB_CUDA(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[chain %s] levels (us):", tail_rows > 0 ? "up" : "down");
        for (int i = 0; i < ch.nlev; ++i)
            std::fprintf(stderr, " %d:%.1f(%d tiles)", i, (ts[i + 1] - ts[i]) * 1e-3, ch.lvl_tile[i + 1] - ch.lvl_tile[i]);
        std::fprintf(stderr, "\n");
    }
}

}  // namespace ebem
