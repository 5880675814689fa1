// KIFMM evaluation (Sec. 2.2) on the tree built by tree.cu:
//   upward   : S2M (sources -> upward check potential, fp32 pair loop, TF32 split fused)
//              -> z = Q_u1^T q;  M2M (z_P += M2M_c z_C, level by level, fine to coarse)
//   downward : M2L (w_B += M2L_o z_A, all levels in one launch, grouped by translation o),
//              S2L for the X entries not summed directly -> w += Q_d1^T q,
//              L2L (w_C += L2L_c w_P, coarse to fine)
//   leaves   : phi = r R^-1 z / w (fp64, DMMA); near field = U list + the X / W / V entries
//              that are cheaper summed directly (reading R11), on a second stream beside
//              M2L; far field = L2T + M2T from phi, plus the near buffer, scattered to the
//              caller's target order.
// Translations run on tcgen05 3xTF32 (tc_gemm.cu); precision choices in DESIGN.md Sec. 5.
#include <chrono>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "fmm.cuh"
#include "p2p.cuh"

namespace ebem {

int64_t launch_count();

struct BoxGeo {
    double ox, oy, oz, side;
    __device__ __forceinline__ void center(const int* anchor, const int* level, int b, double& cx, double& cy,
                                           double& cz, double& r) const {
        const double h = side * __hiloint2double((1023 - level[b]) << 20, 0);   // side 2^-level, exact
        cx = ox + (anchor[3 * b] + 0.5) * h;
        cy = oy + (anchor[3 * b + 1] + 0.5) * h;
        cz = oz + (anchor[3 * b + 2] + 0.5) * h;
        r = 0.5 * h;
    }
};

// round-to-nearest TF32 (the tensor-core operand split, as tc_gemm.cu's split kernel)
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// ------------------------------------------------------------------ check potentials
// Entry i: target = check surface of box tbox[i] (radius factor rad), sources = the
// sources of boxes sidx[soff[i] .. soff[i+1]) (or of tbox[i] itself when soff is null).
// Output Q[i][3 nc] (fp32).  PAPER.md line 147: the approximation sum_i phi_i K(x_i, y)
// is fitted to the sources' field on a check surface.
#ifndef EBEM_CP_TILE
#define EBEM_CP_TILE 64
#endif
constexpr int CP_T = 256, CP_TILE = EBEM_CP_TILE;

// one thread per check point (KPT points per thread when the surface has more than CP_T),
// accumulators in registers, sources streamed through shared memory
template <bool SL, bool DL, int KPT>
__global__ void __launch_bounds__(CP_T)
check_potential_kernel(const int* __restrict__ tbox, const int* __restrict__ soff, const int* __restrict__ sidx,
                       const int* __restrict__ sbeg, const int* __restrict__ send, const int* __restrict__ anchor,
                       const int* __restrict__ level, BoxGeo geo, double rad, const float* __restrict__ sc, int nc,
                       const float4* __restrict__ rec, KConst kc, float* __restrict__ Q, float* __restrict__ Qb,
                       float* __restrict__ Qs, int ldq, const int* __restrict__ ssplit, int smode,
                       __half* __restrict__ Qhb, __half* __restrict__ Qhs, float* __restrict__ Qhinv, int ldqh) {
    __shared__ float4 srec[CP_TILE * REC_DISP];
    __shared__ float wmax[CP_T / 32];
    const int i = blockIdx.x;
    const int b = tbox[i];
    double cx, cy, cz, r;
    geo.center(anchor, level, b, cx, cy, cz, r);
    const float R = (float)(rad * r);
    float x[KPT], y[KPT], z[KPT], acc[KPT][3];
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
        const int k = min((int)(threadIdx.x + q * blockDim.x), nc - 1);
        // coordinates relative to the box centre: absolute fp32 check points would carry an
        // error of ulp(|x|), which is not small against a deep box (a level-20 box is
        // ~1e-6 of the root)
        x[q] = R * sc[3 * k];
        y[q] = R * sc[3 * k + 1];
        z[q] = R * sc[3 * k + 2];
        acc[q][0] = acc[q][1] = acc[q][2] = 0.f;
    }
    const int e0 = soff ? soff[i] : 0, e1 = soff ? soff[i + 1] : 1;
    for (int e = e0; e < e1; ++e) {
        const int a = soff ? sidx[e] : b;
        for (int s0 = sbeg[a]; s0 < send[a]; s0 += CP_TILE) {
            const int cnt = min(CP_TILE, send[a] - s0);
            __syncthreads();
            for (int q = threadIdx.x; q < cnt * REC_DISP; q += blockDim.x) {
                float4 v = rec[(int64_t)s0 * REC_DISP + q];
                if (q % REC_DISP == 0) {            // source position, shifted in fp64
                    v.x = (float)((double)v.x - cx);
                    v.y = (float)((double)v.y - cy);
                    v.z = (float)((double)v.z - cz);
                }
                srec[q] = v;
            }
            __syncthreads();
            // (check points never coincide with sources: SAFE = false)
            if (SL && DL && smode) {
                // BEM sources grouped by panel type (tree_partition_sources): each source
                // carries only one layer, so each part runs the one-kernel loop
                const int cs = min(max(ssplit[a] - s0, 0), cnt);
                const float4* s2 = srec + cs * REC_DISP;
                if (smode == 1) {
                    pair_loop_multi<true, false, false, KPT, false>(srec, cs, x, y, z, kc, acc);
                    pair_loop_multi<false, true, false, KPT, false>(s2, cnt - cs, x, y, z, kc, acc);
                } else {
                    pair_loop_multi<false, true, false, KPT, false>(srec, cs, x, y, z, kc, acc);
                    pair_loop_multi<true, false, false, KPT, false>(s2, cnt - cs, x, y, z, kc, acc);
                }
            } else {
                pair_loop_multi<SL, DL, false, KPT, false>(srec, cnt, x, y, z, kc, acc);
            }
        }
    }
    if (Qhb) {
        // FP16 operands for the Q2Z contraction (tc_gemm.cu, reading R14): the box's check
        // potentials scaled by one power of two (largest magnitude in [2^12, 2^13)), head and
        // remainder written as halves, the factor undoing the scale per row
        float amax = 0.f;
#pragma unroll
        for (int q = 0; q < KPT; ++q)
            if ((int)(threadIdx.x + q * blockDim.x) < nc)
                amax = fmaxf(amax, fmaxf(fabsf(acc[q][0]), fmaxf(fabsf(acc[q][1]), fabsf(acc[q][2]))));
#pragma unroll
        for (int off = 16; off; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
        __syncthreads();                       // (srec reads done; wmax free)
        if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = amax;
        __syncthreads();
        amax = 0.f;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) amax = fmaxf(amax, wmax[w]);
        const float scl = pow2_scale(amax);
        if (threadIdx.x == 0) Qhinv[i] = 1.f / scl;
#pragma unroll
        for (int q = 0; q < KPT; ++q) {
            const int k = threadIdx.x + q * blockDim.x;
            if (k < nc) {
                const int64_t o = (int64_t)i * ldqh + 3 * k;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float a = acc[q][c] * scl;
                    const __half h = __float2half_rn(a);
                    Qhb[o + c] = h;
                    Qhs[o + c] = __float2half_rn(a - __half2float(h));
                }
            }
        }
        return;
    }
#pragma unroll
    for (int q = 0; q < KPT; ++q) {
        const int k = threadIdx.x + q * blockDim.x;
        if (k < nc) {
            const int64_t o = (int64_t)i * ldq + 3 * k;
            if (Qb) {              // tensor-core path: the TF32 head / remainder split, fused
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float h = tf32_rna(acc[q][c]);
                    Qb[o + c] = h;
                    Qs[o + c] = tf32_rna(acc[q][c] - h);
                }
            } else {
                Q[o] = acc[q][0];
                Q[o + 1] = acc[q][1];
                Q[o + 2] = acc[q][2];
            }
        }
    }
}

// ------------------------------------------------------------------ leaf evaluation
// Two warp-per-leaf kernels (a CTA holds EV_WARPS independent leaves; leaves carry ~24
// targets on surfaces, so a whole CTA per leaf left most lanes idle):
//   far_eval : L2T (own downward equivalent density) + M2T (W list) in fp64 from phi,
//              result (fp32) into the sorted far-field buffer;
//   near_eval: U-list near field in fp32 (sources staged per warp in shared memory),
//              plus the far field, scattered to the caller's target order.
constexpr int EV_WARPS = 4;
// far field (L2T, M2T) in fp64 from this multipole order on; fp32 below (its rounding,
// amplified by the cancelling equivalent densities, stays under the truncation error).
// Inside GMRES the BEM operator always uses fp64: the fp32 rounding is not linear in the
// density, and Krylov iterations stall at that level (observed at tol 1e-6).
constexpr int FAR_FP64_MIN_P = 9;

// T = double: fp64 evaluation (p >= 9, where fp32 rounding of the cancelling terms
// sum_k K(x, y_k) phi_k would exceed the truncation error); T = float for p <= 8.
template <class T>
__device__ __forceinline__ T far_rinv(T r2);
template <>
__device__ __forceinline__ float far_rinv<float>(float r2) { return rsqrtf(r2); }
template <>
__device__ __forceinline__ double far_rinv<double>(double r2) {
    // fp32 seed (relative error < 2^-22) + one Newton step (error ~1.5 e^2 < 1e-13, far below
    // what the fp64 accumulation protects); r2 > 0: the equivalent surfaces never reach a target
    const double ri = (double)rsqrtf((float)r2);
    const double h = 0.5 * r2;
    return ri * fma(-h * ri, ri, 1.5);
}

// fp64 far field (p >= 9 and GMRES): the unit equivalent surface is held once per CTA in
// fp64 shared memory and scaled per box in the inner loop, so a warp stages only its box's
// densities (3 ne doubles); lane groups as in the fp32 kernel.
template <bool STRESS, int TPT, class NT, class OT>
__device__ __forceinline__ void far_round_f64(int t0, int t_beg, int t_end, int L, int b, int own, int nfar,
                                              const int* __restrict__ widx, int wbeg, const double* __restrict__ PHID,
                                              int l2t, const double* __restrict__ PHIU,
                                              const int* __restrict__ phiu_slot, const int* __restrict__ anchor,
                                              const int* __restrict__ level, const BoxGeo& geo,
                                              const double* __restrict__ sse, int ne, const float* __restrict__ trg,
                                              const KConst& kc, double cfar, double* ph, int lane,
                                              const NT* __restrict__ near, const int* __restrict__ trg_perm,
                                              OT* __restrict__ out) {
    constexpr int NC = STRESS ? 6 : 3;
    const int G = 32 / L, grp = lane / L, l = lane % L;
    int tc[TPT];
#pragma unroll
    for (int j = 0; j < TPT; ++j) {
        const int t = t0 + l + L * j;
        tc[j] = t < t_end ? t : t_beg;
    }
    double acc[TPT][NC];
#pragma unroll
    for (int j = 0; j < TPT; ++j)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[j][c] = 0.0;
    const double a1 = kc.a1d, aa = kc.ad;
    for (int e = 0; e < nfar; ++e) {
        const bool is_own = own && e == 0;
        const int a = is_own ? b : widx[wbeg + e - own];
        const double* phi = is_own ? PHID + (int64_t)l2t * 3 * ne
                                   : (phiu_slot[a] >= 0 ? PHIU + (int64_t)phiu_slot[a] * 3 * ne : nullptr);
        if (!phi) continue;
        double cx, cy, cz, r;
        geo.center(anchor, level, a, cx, cy, cz, r);
        const double R = (is_own ? RAD_DE : RAD_UE) * r;
        __syncwarp();
        for (int k = lane; k < 3 * ne; k += 32) ph[k] = cfar * phi[k];
        __syncwarp();
        double x[TPT], y[TPT], z[TPT];
#pragma unroll
        for (int j = 0; j < TPT; ++j) {
            x[j] = (double)trg[3 * tc[j]] - cx;
            y[j] = (double)trg[3 * tc[j] + 1] - cy;
            z[j] = (double)trg[3 * tc[j] + 2] - cz;
        }
        for (int k = grp; k < ne; k += G) {
            const double qx = R * sse[3 * k], qy = R * sse[3 * k + 1], qz = R * sse[3 * k + 2];
            const double fx = ph[3 * k], fy = ph[3 * k + 1], fz = ph[3 * k + 2];
#pragma unroll
            for (int j = 0; j < TPT; ++j) {
                const double dx = x[j] - qx, dy = y[j] - qy, dz = z[j] - qz;
                const double ri = far_rinv<double>(dx * dx + dy * dy + dz * dz);
                if (!STRESS)
                    acc_U<double>(dx, dy, dz, ri, fx, fy, fz, a1, acc[j]);
                else
                    acc_D<double>(dx, dy, dz, ri, fx, fy, fz, aa, acc[j]);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < TPT; ++j)
#pragma unroll
        for (int c = 0; c < NC; ++c)
            for (int off = L; off < 32; off <<= 1) acc[j][c] += __shfl_xor_sync(0xffffffffu, acc[j][c], off);
    if (grp == 0)
#pragma unroll
        for (int j = 0; j < TPT; ++j) {
            const int t = t0 + l + L * j;
            if (t < t_end) {
                OT* o = out + (int64_t)trg_perm[t] * NC;
#pragma unroll
                for (int c = 0; c < NC; ++c) o[c] = (OT)(acc[j][c] + (double)near[(int64_t)t * NC + c]);
            }
        }
}

// Lane groups for the warp-per-leaf kernels.  A leaf holds nt targets (~31 on average on
// the benchmark surfaces, 1..64 in general); one lane per target left a quarter of the lanes
// idle.  The warp is split into G = 32 / L groups of L lanes; each group takes every G-th
// source and each lane TPT targets (t0 + l + L j), with L * TPT >= nt as tight as possible,
// and the groups' partial sums are added by shuffles at the end.  Returns TPT (1..4; 0 when
// nt exceeds 128, then a 32 x 4 round is used and repeated).
#ifndef LG_TMAX
#define LG_TMAX 4
#endif
#ifndef NEAR_TILE
#define NEAR_TILE 32          // sources staged per warp
#endif
#ifndef NEAR_TMAX_STRESS
#define NEAR_TMAX_STRESS 3
#endif
__device__ __forceinline__ int lane_groups(int nt, int& L) {
    if (nt > 32 * LG_TMAX) {
        L = 32;
        return LG_TMAX;
    }
    int best = 1 << 30, tpt = LG_TMAX;
    L = 32;
    for (int l = 32; l >= 4; l >>= 1) {
        const int t = (nt + l - 1) / l;
        if (t <= LG_TMAX && l * t < best) {   // strict: ties keep the larger group (fewer shuffles)
            best = l * t;
            L = l;
            tpt = t;
        }
    }
    return tpt;
}

template <int TM>
__device__ __forceinline__ int lane_groups_max(int nt, int& L) {
    if (nt > 32 * TM) {
        L = 32;
        return TM;
    }
    int best = 1 << 30, tpt = TM;
    L = 32;
    for (int l = 32; l >= 4; l >>= 1) {
        const int t = (nt + l - 1) / l;
        if (t <= TM && l * t < best) {
            best = l * t;
            L = l;
            tpt = t;
        }
    }
    return tpt;
}

template <int NC, int TPT>
__device__ __forceinline__ void reduce_groups(float (*acc)[NC], int L) {
    for (int off = L; off < 32; off <<= 1)
#pragma unroll
        for (int j = 0; j < TPT; ++j)
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[j][c] += __shfl_xor_sync(0xffffffffu, acc[j][c], off);
}

// fp32 far field (p <= 8 matvec): phi arrives pre-scaled in fp32 (PHI GEMM epilogue), so a
// box costs one coalesced copy of its equivalent points / densities into the warp's shared
// slice; each lane then evaluates TPT targets against them (TPT = 2 for leaves with more
// than 32 targets: every staged point is read once for both).
template <bool STRESS, int TPT>
__device__ __forceinline__ void far_round_f32(int t0, int t_beg, int t_end, int L, int b, int own, int nfar,
                                              const int* __restrict__ widx, int wbeg, const float4* __restrict__ PHIDF,
                                              int l2t, const float4* __restrict__ PHIUF,
                                              const int* __restrict__ phiu_slot, const int* __restrict__ anchor,
                                              const int* __restrict__ level, const BoxGeo& geo,
                                              const float4* __restrict__ se4, int ne, const float* __restrict__ trg,
                                              const KConst& kc, float4* ey, float4* ph, int lane,
                                              const float* __restrict__ near, const int* __restrict__ trg_perm,
                                              float* __restrict__ out) {
    constexpr int NC = STRESS ? 6 : 3;
    const int G = 32 / L, grp = lane / L, l = lane % L;
    int tc[TPT];
#pragma unroll
    for (int j = 0; j < TPT; ++j) {
        const int t = t0 + l + L * j;
        tc[j] = t < t_end ? t : t_beg;
    }
    float acc[TPT][NC];
#pragma unroll
    for (int j = 0; j < TPT; ++j)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[j][c] = 0.f;
    for (int e = 0; e < nfar; ++e) {
        const bool is_own = own && e == 0;
        const int a = is_own ? b : widx[wbeg + e - own];
        const float4* phi = is_own ? PHIDF + (int64_t)l2t * ne
                                   : (phiu_slot[a] >= 0 ? PHIUF + (int64_t)phiu_slot[a] * ne : nullptr);
        if (!phi) continue;
        double cx, cy, cz, r;
        geo.center(anchor, level, a, cx, cy, cz, r);
        const float R = (float)((is_own ? RAD_DE : RAD_UE) * r);
        __syncwarp();
        for (int k = lane; k < ne; k += 32) {
            const float4 u = se4[k];
            ey[k] = make_float4(R * u.x, R * u.y, R * u.z, 0.f);
            ph[k] = phi[k];
        }
        __syncwarp();
        float x[TPT], y[TPT], z[TPT];
#pragma unroll
        for (int j = 0; j < TPT; ++j) {          // relative to the box centre, in fp64
            x[j] = (float)((double)trg[3 * tc[j]] - cx);
            y[j] = (float)((double)trg[3 * tc[j] + 1] - cy);
            z[j] = (float)((double)trg[3 * tc[j] + 2] - cz);
        }
#pragma unroll 2
        for (int k = grp; k < ne; k += G) {      // this group's share of the equivalent points
            const float4 q = ey[k], f = ph[k];
#pragma unroll
            for (int j = 0; j < TPT; ++j) {
                const float dx = x[j] - q.x, dy = y[j] - q.y, dz = z[j] - q.z;
                const float ri = rsqrtf(fmaf(dz, dz, fmaf(dy, dy, dx * dx)));
                if (!STRESS)
                    acc_U<float>(dx, dy, dz, ri, f.x, f.y, f.z, kc.a1, acc[j]);
                else
                    acc_D<float>(dx, dy, dz, ri, f.x, f.y, f.z, kc.a, acc[j]);
            }
        }
    }
    reduce_groups<NC, TPT>(acc, L);
    if (grp == 0)
#pragma unroll
        for (int j = 0; j < TPT; ++j) {
            const int t = t0 + l + L * j;
            if (t < t_end) {
                float* o = out + (int64_t)trg_perm[t] * NC;
#pragma unroll
                for (int c = 0; c < NC; ++c) o[c] = acc[j][c] + near[(int64_t)t * NC + c];
            }
        }
}

#ifndef FAR64_TMAX
#define FAR64_TMAX 4
#endif
template <bool STRESS, class NT, class OT>
__global__ void __launch_bounds__(32 * EV_WARPS)
far_eval_f64_kernel(int n_eval, const int* __restrict__ eval_box, const int* __restrict__ l2t_slot,
                    const double* __restrict__ PHID, const double* __restrict__ PHIU,
                    const int* __restrict__ phiu_slot, const int* __restrict__ woff, const int* __restrict__ widx,
                    const int* __restrict__ tbeg, const int* __restrict__ tend, const int* __restrict__ anchor,
                    const int* __restrict__ level, BoxGeo geo, const double* __restrict__ se, int ne,
                    const float* __restrict__ trg, KConst kc, double cfar, const NT* __restrict__ near,
                    const int* __restrict__ trg_perm, OT* __restrict__ out) {
    extern __shared__ double dsm[];
    double* sse = dsm;                                      // [3 ne] unit surface (CTA)
    for (int k = threadIdx.x; k < 3 * ne; k += blockDim.x) sse[k] = se[k];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * EV_WARPS + warp;
    if (i >= n_eval) return;                                 // warp-uniform; no CTA barriers below
    double* ph = dsm + 3 * ne + (size_t)warp * 3 * ne;
    const int b = eval_box[i];
    const int t_beg = tbeg[b], t_end = tend[b];
    const int l2t = l2t_slot[i];
    const int own = l2t >= 0 ? 1 : 0;
    const int nfar = own + (woff[b + 1] - woff[b]);
    for (int t0 = t_beg; t0 < t_end;) {
        int L;
        // fp64: up to 4 targets per lane (2 for the 6-component stress sums): independent
        // Newton/accumulation chains hide the DFMA latency
        const int tpt = STRESS ? lane_groups_max<2>(t_end - t0, L) : lane_groups_max<FAR64_TMAX>(t_end - t0, L);
#define EB_FAR64(T)                                                                                                  \
    far_round_f64<STRESS, T, NT, OT>(t0, t_beg, t_end, L, b, own, nfar, widx, woff[b], PHID, l2t, PHIU, phiu_slot,   \
                                     anchor, \
                             level, geo, sse, ne, trg, kc, cfar, ph, lane, near, trg_perm, out)
        if (tpt == 1) EB_FAR64(1);
        else if (STRESS || tpt == 2) EB_FAR64(2);
#if FAR64_TMAX >= 3
        else if (tpt == 3) EB_FAR64(3);
#endif
#if FAR64_TMAX >= 4
        else EB_FAR64(4);
#endif
#undef EB_FAR64
        t0 += L * tpt;
    }
}

template <bool STRESS>
__global__ void __launch_bounds__(32 * EV_WARPS)
far_eval_f32_kernel(int n_eval, const int* __restrict__ eval_box, const int* __restrict__ l2t_slot,
                    const float4* __restrict__ PHIDF, const float4* __restrict__ PHIUF,
                    const int* __restrict__ phiu_slot, const int* __restrict__ woff, const int* __restrict__ widx,
                    const int* __restrict__ tbeg, const int* __restrict__ tend, const int* __restrict__ anchor,
                    const int* __restrict__ level, BoxGeo geo, const float4* __restrict__ se4, int ne,
                    const float* __restrict__ trg, KConst kc, const float* __restrict__ near,
                    const int* __restrict__ trg_perm, float* __restrict__ out) {
    extern __shared__ float4 fsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * EV_WARPS + warp;
    if (i >= n_eval) return;                       // warp-uniform; no CTA barriers below
    float4* ey = fsm + (size_t)warp * 2 * ne;
    float4* ph = ey + ne;
    const int b = eval_box[i];
    const int t_beg = tbeg[b], t_end = tend[b];
    const int l2t = l2t_slot[i];
    const int own = l2t >= 0 ? 1 : 0;
    const int nfar = own + (woff[b + 1] - woff[b]);
    for (int t0 = t_beg; t0 < t_end;) {
        int L;
        const int tpt = lane_groups(t_end - t0, L);
#define EB_FAR(T)                                                                                                   \
    far_round_f32<STRESS, T>(t0, t_beg, t_end, L, b, own, nfar, widx, woff[b], PHIDF, l2t, PHIUF, phiu_slot, anchor, \
                             level, geo, se4, ne, trg, kc, ey, ph, lane, near, trg_perm, out)
        switch (tpt) {
            case 1: EB_FAR(1); break;
            case 2: EB_FAR(2); break;
#if LG_TMAX >= 3
            case 3: EB_FAR(3); break;
#endif
#if LG_TMAX >= 4
            case 4: EB_FAR(4); break;
#endif
#if LG_TMAX > 4
            case 5: EB_FAR(5); break;
            case 6: EB_FAR(6); break;
            case 7: EB_FAR(7); break;
            case 8: EB_FAR(8); break;
#endif
            default: EB_FAR(LG_TMAX); break;
        }
#undef EB_FAR
        t0 += L * tpt;
    }
}

// near field: U-list sources staged 32 at a time per warp (record stride R + 1 float4, so
// the groups' different records fall in different banks); lane groups as above
template <bool SL, bool DL, bool STRESS, int TPT>
__device__ __forceinline__ void near_round(int t0, int t_beg, int t_end, int L, int b, const int* __restrict__ uoff,
                                           const int* __restrict__ uidx, const int* __restrict__ sbeg,
                                           const int* __restrict__ send, const float* __restrict__ trg,
                                           const float4* __restrict__ rec, const KConst& kc,
                                           float* __restrict__ near, float4* srec, int lane) {
    constexpr int NC = STRESS ? 6 : 3;
    constexpr int R = STRESS ? REC_STRESS : REC_DISP;
    constexpr int RS = R + 1;
    const int G = 32 / L, grp = lane / L, l = lane % L;
    float x[TPT], y[TPT], z[TPT], acc[TPT][NC];
#pragma unroll
    for (int j = 0; j < TPT; ++j) {
        const int t = t0 + l + L * j;
        const int tc = t < t_end ? t : t_beg;
        x[j] = trg[3 * tc];
        y[j] = trg[3 * tc + 1];
        z[j] = trg[3 * tc + 2];
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[j][c] = 0.f;
    }
    for (int e = uoff[b]; e < uoff[b + 1]; ++e) {
        const int a = uidx[e];
        for (int s0 = sbeg[a]; s0 < send[a]; s0 += NEAR_TILE) {
            const int cnt = min(NEAR_TILE, send[a] - s0);
            __syncwarp();
            for (int q = lane; q < cnt * R; q += 32) srec[(q / R) * RS + q % R] = rec[(int64_t)s0 * R + q];
            __syncwarp();
            if (a == b) pair_loop_strided<SL, DL, STRESS, TPT, RS, true>(srec, cnt, grp, G, x, y, z, kc, acc);
            else pair_loop_strided<SL, DL, STRESS, TPT, RS, false>(srec, cnt, grp, G, x, y, z, kc, acc);
        }
    }
    reduce_groups<NC, TPT>(acc, L);
    if (grp == 0)
#pragma unroll
        for (int j = 0; j < TPT; ++j) {
            const int t = t0 + l + L * j;
            if (t < t_end)
#pragma unroll
                for (int c = 0; c < NC; ++c)   // acc_DS accumulates half of the diagonal
                    near[(int64_t)t * NC + c] = (STRESS && SL && DL && c < 3) ? 2.f * acc[j][c] : acc[j][c];
        }
}

template <bool SL, bool DL, bool STRESS>
__global__ void __launch_bounds__(32 * EV_WARPS)
near_eval_kernel(int n_eval, const int* __restrict__ eval_box, const int* __restrict__ uoff,
                 const int* __restrict__ uidx, const int* __restrict__ sbeg, const int* __restrict__ send,
                 const int* __restrict__ tbeg, const int* __restrict__ tend, const float* __restrict__ trg,
                 const float4* __restrict__ rec, KConst kc, float* __restrict__ near) {
    constexpr int R = STRESS ? REC_STRESS : REC_DISP;
    __shared__ float4 srec_all[EV_WARPS][NEAR_TILE * (R + 1)];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * EV_WARPS + warp;
    if (i >= n_eval) return;
    float4* srec = srec_all[warp];
    const int b = eval_box[i];
    const int t_beg = tbeg[b], t_end = tend[b];
    for (int t0 = t_beg; t0 < t_end;) {
        int L;
#define EB_NEAR(T)                                                                                                   \
    near_round<SL, DL, STRESS, T>(t0, t_beg, t_end, L, b, uoff, uidx, sbeg, send, trg, rec, kc, near, srec, lane)
        if constexpr (STRESS) {     // 6-component sums: fewer targets per lane keep registers down
            const int tpt = lane_groups_max<NEAR_TMAX_STRESS>(t_end - t0, L);
            if (tpt == 1) EB_NEAR(1);
#if NEAR_TMAX_STRESS >= 3
            else if (tpt == 3) EB_NEAR(3);
#endif
#if NEAR_TMAX_STRESS >= 4
            else if (tpt == 4) EB_NEAR(4);
#endif
            else EB_NEAR(2);
            t0 += L * tpt;
        } else {
        const int tpt = lane_groups(t_end - t0, L);
        switch (tpt) {
            case 1: EB_NEAR(1); break;
            case 2: EB_NEAR(2); break;
#if LG_TMAX >= 3
            case 3: EB_NEAR(3); break;
#endif
#if LG_TMAX >= 4
            case 4: EB_NEAR(4); break;
#endif
#if LG_TMAX > 4
            case 5: EB_NEAR(5); break;
            case 6: EB_NEAR(6); break;
            case 7: EB_NEAR(7); break;
            case 8: EB_NEAR(8); break;
#endif
            default: EB_NEAR(LG_TMAX); break;
        }
#undef EB_NEAR
        t0 += L * tpt;
        }
    }
}

// Packed lane groups (FFMA2 pair loops, packed.cuh): groups of L lanes, each lane NP PAIRS of
// targets (t0 + l + L j, j = 0 .. 2 NP - 1; pack k = targets 2k, 2k + 1), L * 2 NP >= nt as
// tight as possible; on ties the smaller group (more targets per lane: each staged source
// record is read once for more targets).  Returns NP (NPMAX and L = 32 when nt exceeds
// 64 NPMAX: rounds are repeated).
template <int NPMAX>
__device__ __forceinline__ int lane_groups_packed(int nt, int& L) {
    if (nt > 64 * NPMAX) {
        L = 32;
        return NPMAX;
    }
    int best = 1 << 30, np = NPMAX;
    L = 32;
    for (int l = 32; l >= 4; l >>= 1) {
        const int t = (nt + 2 * l - 1) / (2 * l);
        if (t <= NPMAX && 2 * l * t <= best) {
            best = 2 * l * t;
            L = l;
            np = t;
        }
    }
    return np;
}

template <int NC, int NP>
__device__ __forceinline__ void reduce_groups_packed(F2 (*acc)[NC], int L) {
    for (int off = L; off < 32; off <<= 1)
#pragma unroll
        for (int k = 0; k < NP; ++k)
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                acc[k][c].v.x += __shfl_xor_sync(0xffffffffu, acc[k][c].v.x, off);
                acc[k][c].v.y += __shfl_xor_sync(0xffffffffu, acc[k][c].v.y, off);
            }
}

// near field with the packed pair loop: as near_round, two targets per FP32 instruction
template <bool SL, bool DL, bool STRESS, int NP>
__device__ __forceinline__ void near_round_p(int t0, int t_beg, int t_end, int L, int b, const int* __restrict__ uoff,
                                             const int* __restrict__ uidx, const int* __restrict__ sbeg,
                                             const int* __restrict__ send, const float* __restrict__ trg,
                                             const float4* __restrict__ rec, const KConst2& kc,
                                             float* __restrict__ near, float4* srec, int lane) {
    constexpr int NC = STRESS ? 6 : 3;
    constexpr int R = STRESS ? REC_STRESS : REC_DISP;
    constexpr int RS = R + 1;
    const int G = 32 / L, grp = lane / L, l = lane % L;
    F2 x[NP], y[NP], z[NP], acc[NP][NC];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const int ta = t0 + l + L * (2 * k), tb = ta + L;
        const int ca = ta < t_end ? ta : t_beg, cb = tb < t_end ? tb : t_beg;
        x[k] = F2(trg[3 * ca], trg[3 * cb]);
        y[k] = F2(trg[3 * ca + 1], trg[3 * cb + 1]);
        z[k] = F2(trg[3 * ca + 2], trg[3 * cb + 2]);
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[k][c] = F2(0.f);
    }
    for (int e = uoff[b]; e < uoff[b + 1]; ++e) {
        const int a = uidx[e];
        for (int s0 = sbeg[a]; s0 < send[a]; s0 += NEAR_TILE) {
            const int cnt = min(NEAR_TILE, send[a] - s0);
            __syncwarp();
            for (int q = lane; q < cnt * R; q += 32) srec[(q / R) * RS + q % R] = rec[(int64_t)s0 * R + q];
            __syncwarp();
            if (a == b) pair_loop_packed<SL, DL, STRESS, NP, RS, true>(srec, cnt, grp, G, x, y, z, kc, acc);
            else pair_loop_packed<SL, DL, STRESS, NP, RS, false>(srec, cnt, grp, G, x, y, z, kc, acc);
        }
    }
    reduce_groups_packed<NC, NP>(acc, L);
    if (grp == 0)
#pragma unroll
        for (int k = 0; k < NP; ++k)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int t = t0 + l + L * (2 * k + h);
                if (t < t_end)
#pragma unroll
                    for (int c = 0; c < NC; ++c) {   // acc_DS accumulates half of the diagonal
                        const float v = h ? acc[k][c].v.y : acc[k][c].v.x;
                        near[(int64_t)t * NC + c] = (STRESS && SL && DL && c < 3) ? 2.f * v : v;
                    }
            }
}

#ifndef NEAR_NPMAX
#define NEAR_NPMAX 4
#endif
template <bool SL, bool DL, bool STRESS>
__global__ void __launch_bounds__(32 * EV_WARPS)
near_eval_p_kernel(int n_eval, const int* __restrict__ eval_box, const int* __restrict__ uoff,
                   const int* __restrict__ uidx, const int* __restrict__ sbeg, const int* __restrict__ send,
                   const int* __restrict__ tbeg, const int* __restrict__ tend, const float* __restrict__ trg,
                   const float4* __restrict__ rec, KConst kc1, float* __restrict__ near) {
    constexpr int R = STRESS ? REC_STRESS : REC_DISP;
    constexpr int NPM = STRESS ? 2 : NEAR_NPMAX;       // 6-component sums: fewer pairs per lane
    __shared__ float4 srec_all[EV_WARPS][NEAR_TILE * (R + 1)];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * EV_WARPS + warp;
    if (i >= n_eval) return;
    const KConst2 kc(kc1);
    float4* srec = srec_all[warp];
    const int b = eval_box[i];
    const int t_beg = tbeg[b], t_end = tend[b];
    for (int t0 = t_beg; t0 < t_end;) {
        int L;
        const int np = lane_groups_packed<NPM>(t_end - t0, L);
#define EB_NEARP(N) \
    near_round_p<SL, DL, STRESS, N>(t0, t_beg, t_end, L, b, uoff, uidx, sbeg, send, trg, rec, kc, near, srec, lane)
        if (np == 1) EB_NEARP(1);
        else if (np == 2 || NPM == 2) EB_NEARP(2);
        else if (np == 3) EB_NEARP(3);
        else EB_NEARP(NPM);
#undef EB_NEARP
        t0 += 2 * L * np;
    }
}

// EBEM_M2L_F16: 0 = M2L operands in TF32; 1 = FP16 for the full-chain M2L (p <= 8 matvec, GMRES
// solves with tol >= 1e-6); 2 = FP16 for the drained (precise) M2L too
static int m2l_f16_level() {
    static const int lv = std::getenv("EBEM_M2L_F16") ? std::atoi(std::getenv("EBEM_M2L_F16")) : 2;
    return lv;
}
static bool ml_f16_on() {      // EBEM_ML_F16=0: M2M / L2L stay in TF32
    static const bool on = !(std::getenv("EBEM_ML_F16") && std::atoi(std::getenv("EBEM_ML_F16")) == 0);
    return on;
}
// EBEM_M2L_MC=cs: the full-chain two-slice M2L on clusters of cs CTAs sharing the operator tiles
// by TMA multicast (tc_pairs_mc_kernel); 0 / 1: one CTA per tile
static int m2l_mc_cs() {
    static const int cs = std::getenv("EBEM_M2L_MC") ? std::atoi(std::getenv("EBEM_M2L_MC")) : 0;
    return cs == 2 || cs == 4 ? cs : 1;
}
static bool m2l_use_f16(const Tree& t) { return t.m2l_f16 && (t.tc_fast || m2l_f16_level() >= 2); }
// precise M2L (p >= 9, GMRES) on the two-slice fast-kernel data flow with drained groups;
// EBEM_M2L_DRAIN=0 selects the one-slice precise kernel instead
static bool m2l_drain_fast() {
    static const bool on = !(std::getenv("EBEM_M2L_DRAIN") && std::atoi(std::getenv("EBEM_M2L_DRAIN")) == 0);
    return on;
}
// the M2L tile table for the tree's current accumulation mode (tc_fast) and operand type
static void build_m2l_tiles(Tree& t) {
    const Plan& P = *t.plan;
    const bool fastflow = t.tc_fast || m2l_drain_fast();
    const int mode = fastflow ? tc_fast_tile_mode(P.me) : 0;
    tc_build_tiles(t.m2l, P.me, P.me, mode, fastflow && m2l_use_f16(t) ? 64 : 32,
                   t.tc_fast && mode == 1 ? m2l_mc_cs() : 1);
}

// ------------------------------------------------------------------ M2L pair table (device)
struct OffIndex {
    int v[343];
};

__device__ __forceinline__ bool m2l_valid(int b, int a, const int* __restrict__ up, const int* __restrict__ leaf,
                                          const int* __restrict__ nsub, const int* __restrict__ tsub, double vdir) {
    if (up[a] < 0) return false;
    return !(vdir > 0.0 && leaf[b] && leaf[a] && (double)nsub[a] * tsub[b] < vdir);
}

__global__ void m2l_count_kernel(int nb, const int* __restrict__ voff, const int* __restrict__ vidx,
                                 const int* __restrict__ dn, const int* __restrict__ up, const int* __restrict__ leaf,
                                 const int* __restrict__ nsub, const int* __restrict__ tsub, double vdir,
                                 int* __restrict__ cnt) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int c = 0;
    if (dn[b] >= 0)
        for (int e = voff[b]; e < voff[b + 1]; ++e) c += m2l_valid(b, vidx[e], up, leaf, nsub, tsub, vdir);
    cnt[b] = c;
}

__global__ void m2l_fill_kernel(int nb, const int* __restrict__ voff, const int* __restrict__ vidx,
                                const int* __restrict__ dn, const int* __restrict__ up, const int* __restrict__ leaf,
                                const int* __restrict__ nsub, const int* __restrict__ tsub, double vdir,
                                const int* __restrict__ anchor, OffIndex oi, const int* __restrict__ pos,
                                long long* __restrict__ keys, int* __restrict__ src, int* __restrict__ ord,
                                int* __restrict__ opcount, int* __restrict__ bad) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb || dn[b] < 0) return;
    int k = pos[b];
    for (int e = voff[b]; e < voff[b + 1]; ++e) {
        const int a = vidx[e];
        if (!m2l_valid(b, a, up, leaf, nsub, tsub, vdir)) continue;
        const int ox = anchor[3 * a] - anchor[3 * b], oy = anchor[3 * a + 1] - anchor[3 * b + 1],
                  oz = anchor[3 * a + 2] - anchor[3 * b + 2];
        const bool in = ox >= -3 && ox <= 3 && oy >= -3 && oy <= 3 && oz >= -3 && oz <= 3;
        const int o = in ? oi.v[(ox + 3) * 49 + (oy + 3) * 7 + (oz + 3)] : -1;
        if (o < 0) {
            atomicExch(bad, 1);
            continue;
        }
        keys[k] = ((long long)o << 32) | (long long)dn[b];
        src[k] = up[a];
        ord[k] = k;
        atomicAdd(&opcount[o], 1);
        ++k;
    }
}

__global__ void m2l_gather_kernel(int64_t n, const long long* __restrict__ keys, const int* __restrict__ ord,
                                  const int* __restrict__ src, int2* __restrict__ pairs) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) pairs[i] = make_int2((int)(keys[i] & 0xffffffffLL), src[ord[i]]);
}

static void build_m2l_pairs(Tree& t, int nb, double vdir, cudaStream_t s) {
    const Plan& P = *t.plan;
    OpPairs& M = t.m2l;
    M.nops = NV_OFFSETS;
    DBuf<int> cnt(nb + 1), pos(nb + 1);
    m2l_count_kernel<<<ceil_div(nb, 256), 256, 0, s>>>(nb, t.lst_off[1].p, t.lst_idx[1].p, t.dn_slot.p, t.up_slot.p,
                                                       t.is_leaf.p, t.nsrc_sub.p, t.ntrg_sub.p, vdir, cnt.p);
    EB_CHECK_LAUNCH();
    const int64_t n = exclusive_scan_i32(cnt.p, pos.p, nb, s);
    M.npairs = n;
    DBuf<long long> keys(std::max<int64_t>(n, 1));
    DBuf<int> src(std::max<int64_t>(n, 1)), ord(std::max<int64_t>(n, 1)), opcount(NV_OFFSETS + 1), bad(1);
    opcount.zero(s);
    bad.zero(s);
    OffIndex oi;
    std::memcpy(oi.v, P.off_index, sizeof(oi.v));
    m2l_fill_kernel<<<ceil_div(nb, 256), 256, 0, s>>>(nb, t.lst_off[1].p, t.lst_idx[1].p, t.dn_slot.p, t.up_slot.p,
                                                      t.is_leaf.p, t.nsrc_sub.p, t.ntrg_sub.p, vdir, t.anchor.p, oi,
                                                      pos.p, keys.p, src.p, ord.p, opcount.p, bad.p);
    EB_CHECK_LAUNCH();
    radix_sort_pairs(keys.p, ord.p, n, 32 + 9, s);     // operator (9 bits) over target row (32)
    M.pairs.alloc(std::max<int64_t>(n, 1));
    if (n) {
        m2l_gather_kernel<<<ceil_div(n, 256), 256, 0, s>>>(n, keys.p, ord.p, src.p, M.pairs.p);
        EB_CHECK_LAUNCH();
    }
    std::vector<int> oc(NV_OFFSETS + 1, 0);
    int hbad = 0;
    d2h(oc.data(), opcount.p, NV_OFFSETS, s);
    d2h(&hbad, bad.p, 1, s);
    EB_CUDA(cudaStreamSynchronize(s));
    EB_REQUIRE(!hbad, "internal: V-list offset outside the 7^3 stencil");
    M.op_ptr_h.assign(NV_OFFSETS + 1, 0);
    M.max_per_op = 0;
    for (int o = 0; o < NV_OFFSETS; ++o) {
        M.op_ptr_h[o + 1] = M.op_ptr_h[o] + oc[o];
        M.max_per_op = std::max(M.max_per_op, oc[o]);
    }
    M.op_ptr.alloc(NV_OFFSETS + 1);
    h2d(M.op_ptr.p, M.op_ptr_h.data(), NV_OFFSETS + 1, s);
    EB_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ leaf lists (device)
// Per target leaf b: the near list (sources summed directly: the U list, the V entries cheaper
// direct (reading R11), the X entries when b is cheaper direct, the W entries whose box holds
// few sources) and the M2T list (the other W entries), in that order -- the order the near
// field sums them.  Pass 1 counts (and the near sources per leaf for the work counts), pass 2
// fills at the scanned offsets.
struct NearRule {
    int xw_direct, v_dir_on, nc;
    double w_thresh, v_thresh;   // w_direct: nsub < w_thresh; v_direct: nsub * tsub < v_thresh
};

template <bool FILL>
__global__ void leaf_lists_kernel(int nb, const int* __restrict__ leaf, const int* __restrict__ nsub,
                                  const int* __restrict__ tsub, const int* __restrict__ uoff,
                                  const int* __restrict__ uidx, const int* __restrict__ voff,
                                  const int* __restrict__ vidx, const int* __restrict__ woff,
                                  const int* __restrict__ widx, const int* __restrict__ xoff,
                                  const int* __restrict__ xidx, NearRule r, int* __restrict__ ncnt,
                                  int* __restrict__ mcnt, int* __restrict__ nsrc, const int* __restrict__ npos,
                                  const int* __restrict__ mpos, int* __restrict__ nidx, int* __restrict__ midx) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) {                               // the last CSR entry: counts 0 before the scan
        if (!FILL && b == nb) ncnt[b] = mcnt[b] = 0;
        return;
    }
    int n = 0, m = 0, ns = 0;
    const int np0 = FILL ? npos[b] : 0, mp0 = FILL ? mpos[b] : 0;
    auto put_n = [&](int a) {
        if (FILL) nidx[np0 + n] = a;
        ++n;
        ns += nsub[a];
    };
    if (leaf[b] && tsub[b] > 0) {
        for (int e = uoff[b]; e < uoff[b + 1]; ++e) put_n(uidx[e]);
        for (int e = voff[b]; e < voff[b + 1]; ++e) {
            const int a = vidx[e];
            if (nsub[a] > 0 && r.v_dir_on && leaf[a] && (double)nsub[a] * tsub[b] < r.v_thresh) put_n(a);
        }
        if (r.xw_direct && tsub[b] < r.nc)
            for (int e = xoff[b]; e < xoff[b + 1]; ++e)
                if (nsub[xidx[e]] > 0) put_n(xidx[e]);
        for (int e = woff[b]; e < woff[b + 1]; ++e) {
            const int a = widx[e];
            if (nsub[a] == 0) continue;
            if (r.xw_direct && nsub[a] < r.w_thresh) put_n(a);
            else {
                if (FILL) midx[mp0 + m] = a;
                ++m;
            }
        }
    }
    if (!FILL) {
        ncnt[b] = n;
        mcnt[b] = m;
        nsrc[b] = ns;
    }
}

// ------------------------------------------------------------------ schedule (host)
void schedule_tree(Tree& t, cudaStream_t s) {
    const Plan& P = *t.plan;
    static const bool timing = std::getenv("EBEM_BUILD_TIMING") != nullptr;
    auto tick = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!timing) return;
        EB_CUDA(cudaStreamSynchronize(s));
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[ebem schedule] %-18s %.2f ms\n", what,
                std::chrono::duration<double, std::milli>(now - tick).count());
        tick = now;
    };
    const int nb = t.nboxes;
    auto dl = [&](const DBuf<int>& d, size_t n) {
        std::vector<int> h(n);
        if (n) d2h(h.data(), d.p, n, s);
        return h;
    };
    std::vector<int> level = dl(t.level, nb), parent = dl(t.parent, nb), child = dl(t.child, 8 * (size_t)nb),
                     leaf = dl(t.is_leaf, nb), nsub = dl(t.nsrc_sub, nb), tsub = dl(t.ntrg_sub, nb),
                     anchor = dl(t.anchor, 3 * (size_t)nb);
    std::vector<int> off[4], idx[4];
    for (int k = 2; k < 4; ++k) {            // W, X (the U and V lists stay on the device)
        off[k] = dl(t.lst_off[k], nb + 1);
        idx[k] = dl(t.lst_idx[k], t.lst_n[k]);
    }
    EB_CUDA(cudaStreamSynchronize(s));
    t.nleaves = 0;
    for (int b = 0; b < nb; ++b) t.nleaves += leaf[b];

    std::vector<int> up(nb, -1), dn(nb, -1);
    t.n_up = t.n_dn = 0;
    for (int b = 0; b < nb; ++b) {
        if (level[b] >= 2 && nsub[b] > 0) up[b] = t.n_up++;
        if (level[b] >= 2 && tsub[b] > 0) dn[b] = t.n_dn++;
    }
    t.up_lstart.assign(t.nlevels + 1, 0);
    t.dn_lstart.assign(t.nlevels + 1, 0);
    for (int b = 0; b < nb; ++b) {
        if (up[b] >= 0) t.up_lstart[level[b] + 1] = up[b] + 1;
        if (dn[b] >= 0) t.dn_lstart[level[b] + 1] = dn[b] + 1;
    }
    for (int l = 1; l <= t.nlevels; ++l) {
        t.up_lstart[l] = std::max(t.up_lstart[l], t.up_lstart[l - 1]);
        t.dn_lstart[l] = std::max(t.dn_lstart[l], t.dn_lstart[l - 1]);
    }
    t.up_slot.alloc(nb);
    t.dn_slot.alloc(nb);
    h2d(t.up_slot.p, up.data(), nb, s);
    h2d(t.dn_slot.p, dn.data(), nb, s);

    lap("download+slots");
    // S2M on leaves carrying z; check potential rows are s2m indices
    std::vector<int> s2m;
    std::vector<int> op1;
    std::vector<int2> pr;
    for (int b = 0; b < nb; ++b)
        if (leaf[b] && up[b] >= 0) {
            pr.push_back(make_int2(up[b], (int)s2m.size()));
            s2m.push_back(b);
        }
    t.n_s2m = (int)s2m.size();
    t.s2m_box.alloc(std::max<size_t>(s2m.size(), 1));
    h2d(t.s2m_box.p, s2m.data(), s2m.size(), s);
    op1.assign(pr.size(), 0);
    build_op_pairs(t.q2z_up, 1, op1, pr, s);

    // M2M per parent level
    t.m2m.clear();
    t.m2m.resize(t.nlevels);
    for (int l = 2; l < t.nlevels; ++l) {
        std::vector<int> op;
        std::vector<int2> p2;
        for (int b = t.level_start[l]; b < t.level_start[l + 1]; ++b) {
            if (leaf[b] || up[b] < 0) continue;
            for (int c = 0; c < 8; ++c) {
                int ch = child[8 * b + c];
                if (ch >= 0 && up[ch] >= 0) {
                    op.push_back(c);
                    p2.push_back(make_int2(up[b], up[ch]));
                }
            }
        }
        build_op_pairs(t.m2m[l], 8, op, p2, s);
    }

    // X- and W-list interactions that are cheaper done directly (reading in DESIGN.md):
    // X (source leaf A -> box B): when B is a leaf with fewer targets than check points, A's
    // sources go straight to B's targets instead of to B's check surface; W (A's equivalent
    // density -> B's targets): when A holds fewer sources than equivalent points, its sources
    // go straight to B's targets.  Exact, and fewer pair interactions either way.
    // EBEM_XW_DIRECT=0 keeps the paper's S2L / M2T for every entry.
    const bool xw_direct = !(std::getenv("EBEM_XW_DIRECT") && std::atoi(std::getenv("EBEM_XW_DIRECT")) == 0);
    auto x_direct = [&](int b) { return xw_direct && leaf[b] && tsub[b] < P.nc; };
    const double wf = std::getenv("EBEM_W_DIRECT_F") ? std::atof(std::getenv("EBEM_W_DIRECT_F")) : t.w_direct;
    // (w_direct(a): xw_direct && nsub[a] < wf n_e -- applied by leaf_lists_kernel)
    // V-list pairs of two leaves with few points: one M2L costs ~ (3 n_e)^2 tensor-core MACs
    // (x3 for 3xTF32) plus its share of the fp64 state; summing the nsrc x ntrg pairs directly
    // is cheaper below ~kappa (3 n_e)^2 pair interactions.  kappa measured with the FP16
    // translations and the branch-free epilogue (the cheaper the M2L, the lower the optimum):
    // 1M beam, p = 6: 3.78 / 3.76 / 3.77 / 3.78 / 3.81 / 3.82 ms at kappa = 0.00475 / 0.005 /
    // 0.00525 / 0.0055 / 0.006 / 0.0065; configs[3], p = 8: 6.68 / 6.53 / 6.58 / 6.66 / 6.76 ms at
    // 0.0025 / 0.003 / 0.0035 / 0.004 / 0.0045.  (TF32 translations: 0.006 for both.)
    const double kappa = std::getenv("EBEM_V_DIRECT") ? std::atof(std::getenv("EBEM_V_DIRECT"))
                                                      : (P.p <= 6 ? 0.005 : 0.003);
    // (only with the fp32 far field, p <= 8: at p >= 9 the fp32 direct sums would exceed the
    // fp64 far field's error, measured 1.5e-6 vs 5.5e-7 at p = 10)
    // (v_direct(b, a): both leaves, nsub[a] tsub[b] < kappa (3 n_e)^2 -- leaf_lists_kernel and
    // the M2L pair table)
    const bool v_dir_on = xw_direct && P.p < FAR_FP64_MIN_P;

    // S2L: boxes with X-list leaves that hold sources
    std::vector<int> s2l, xoff(1, 0), xidx;
    pr.clear();
    for (int b = 0; b < nb; ++b) {
        if (dn[b] < 0 || x_direct(b)) continue;
        int cnt = 0;
        for (int e = off[3][b]; e < off[3][b + 1]; ++e)
            if (nsub[idx[3][e]] > 0) {
                xidx.push_back(idx[3][e]);
                ++cnt;
            }
        if (cnt) {
            pr.push_back(make_int2(dn[b], (int)s2l.size()));
            s2l.push_back(b);
            xoff.push_back((int)xidx.size());
        }
    }
    t.n_s2l = (int)s2l.size();
    t.s2l_box.alloc(std::max<size_t>(s2l.size(), 1));
    h2d(t.s2l_box.p, s2l.data(), s2l.size(), s);
    t.x_src_off.alloc(xoff.size());
    h2d(t.x_src_off.p, xoff.data(), xoff.size(), s);
    t.x_src_idx.alloc(std::max<size_t>(xidx.size(), 1));
    h2d(t.x_src_idx.p, xidx.data(), xidx.size(), s);
    op1.assign(pr.size(), 0);
    build_op_pairs(t.q2z_dn, 1, op1, pr, s);

    lap("s2m/m2m/s2l");
    // M2L, all levels, grouped by translation vector: built on the device (the host loop over
    // the 1.2 M V entries and its counting sort took 6 ms of a 1M-point build); the pair
    // order is the host one: operator-major, target rows ascending within an operator
    build_m2l_pairs(t, nb, v_dir_on ? kappa * (double)P.me * P.me : -1.0, s);

    lap("m2l pairs");
    // L2L per child level
    t.l2l.clear();
    t.l2l.resize(t.nlevels);
    for (int l = 3; l < t.nlevels; ++l) {
        std::vector<int> op;
        std::vector<int2> p2;
        for (int b = t.level_start[l]; b < t.level_start[l + 1]; ++b) {
            if (dn[b] < 0) continue;
            int par = parent[b];
            if (dn[par] < 0) continue;
            int oc = ((anchor[3 * b] & 1) << 2) | ((anchor[3 * b + 1] & 1) << 1) | (anchor[3 * b + 2] & 1);
            op.push_back(oc);
            p2.push_back(make_int2(dn[b], dn[par]));
        }
        build_op_pairs(t.l2l[l], 8, op, p2, s);
    }

    lap("l2l");
    // leaf evaluation: near list (U + direct V / X / W) and M2T list (the other W entries), on
    // the device; the host keeps the M2T list (PHI_U slots) and the near sources per leaf
    std::vector<int> ev, l2t, phid_box, phiu_box, phiu(nb, -1);
    std::vector<int> moff(nb + 1, 0), midx, near_ns(nb);
    {
        const NearRule rule{xw_direct ? 1 : 0, v_dir_on ? 1 : 0, P.nc, wf * P.ne,
                            v_dir_on ? kappa * (double)P.me * P.me : 0.0};
        DBuf<int> ncnt(nb + 1), mcnt(nb + 1), nsrc(nb);
        leaf_lists_kernel<false><<<ceil_div(nb + 1, 128), 128, 0, s>>>(
            nb, t.is_leaf.p, t.nsrc_sub.p, t.ntrg_sub.p, t.lst_off[0].p, t.lst_idx[0].p, t.lst_off[1].p, t.lst_idx[1].p,
            t.lst_off[2].p, t.lst_idx[2].p, t.lst_off[3].p, t.lst_idx[3].p, rule, ncnt.p, mcnt.p, nsrc.p, nullptr,
            nullptr, nullptr, nullptr);
        EB_CHECK_LAUNCH();
        t.near_off.alloc(nb + 1);
        t.m2t_off.alloc(nb + 1);
        const int64_t nn = exclusive_scan_i32(ncnt.p, t.near_off.p, nb + 1, s);
        const int64_t nm = exclusive_scan_i32(mcnt.p, t.m2t_off.p, nb + 1, s);
        t.near_idx.alloc(std::max<int64_t>(nn, 1));
        t.m2t_idx.alloc(std::max<int64_t>(nm, 1));
        leaf_lists_kernel<true><<<ceil_div(nb, 128), 128, 0, s>>>(
            nb, t.is_leaf.p, t.nsrc_sub.p, t.ntrg_sub.p, t.lst_off[0].p, t.lst_idx[0].p, t.lst_off[1].p, t.lst_idx[1].p,
            t.lst_off[2].p, t.lst_idx[2].p, t.lst_off[3].p, t.lst_idx[3].p, rule, nullptr, nullptr, nullptr,
            t.near_off.p, t.m2t_off.p, t.near_idx.p, t.m2t_idx.p);
        EB_CHECK_LAUNCH();
        midx.resize(nm);
        d2h(moff.data(), t.m2t_off.p, nb + 1, s);
        d2h(midx.data(), t.m2t_idx.p, nm, s);
        d2h(near_ns.data(), nsrc.p, nb, s);
        EB_CUDA(cudaStreamSynchronize(s));
    }
    lap("  near/m2t lists");
    std::vector<double> phid_scale, phiu_scale;
    std::vector<int2> prd, pru;
    auto half = [&](int b) { return t.side / (double)(1 << level[b]) * 0.5; };
    for (int b = 0; b < nb; ++b) {
        if (!leaf[b] || tsub[b] == 0) continue;
        ev.push_back(b);
        if (dn[b] >= 0) {
            l2t.push_back((int)phid_box.size());
            prd.push_back(make_int2((int)phid_box.size(), dn[b]));
            phid_scale.push_back(half(b));
            phid_box.push_back(b);
        } else {
            l2t.push_back(-1);
        }
        for (int e = moff[b]; e < moff[b + 1]; ++e) {
            int a = midx[e];
            if (up[a] >= 0 && phiu[a] < 0) {
                phiu[a] = (int)phiu_box.size();
                pru.push_back(make_int2(phiu[a], up[a]));
                phiu_scale.push_back(half(a));
                phiu_box.push_back(a);
            }
        }
    }
    lap("  eval/phi slots");
    // algorithmic work counts for the phase profiler
    {
        const double nc = P.nc, ne = P.ne;
        t.w_s2m_inter = t.w_s2m_src = t.w_s2l_inter = t.w_s2l_src = 0;
        t.w_p2p_inter = t.w_p2p_src = t.w_l2t_inter = t.w_m2t_inter = 0;
        for (int b : s2m) { t.w_s2m_src += nsub[b]; t.w_s2m_inter += nsub[b] * nc; }
        for (size_t i = 0; i + 1 < xoff.size(); ++i)
            for (int e = xoff[i]; e < xoff[i + 1]; ++e) { t.w_s2l_src += nsub[xidx[e]]; t.w_s2l_inter += nsub[xidx[e]] * nc; }
        for (size_t i = 0; i < ev.size(); ++i) {
            const int b = ev[i];
            const double ns = near_ns[b];
            t.w_p2p_src += ns;
            t.w_p2p_inter += ns * tsub[b];
            if (l2t[i] >= 0) t.w_l2t_inter += ne * tsub[b];
            for (int e = moff[b]; e < moff[b + 1]; ++e)
                if (phiu[midx[e]] >= 0) t.w_m2t_inter += ne * tsub[b];
        }
        t.w_m2m_pairs = t.w_l2l_pairs = 0;
        for (auto& x : t.m2m) t.w_m2m_pairs += x.npairs;
        for (auto& x : t.l2l) t.w_l2l_pairs += x.npairs;
        t.w_m2l_ops = 0;
        for (int o = 0; o < t.m2l.nops; ++o) t.w_m2l_ops += t.m2l.op_ptr_h[o + 1] > t.m2l.op_ptr_h[o];
    }
    lap("  work counts");
    // leaves in order of decreasing pair work, so that the warp-per-leaf kernels end on small
    // leaves instead of an SM-wide tail behind the largest: the near-field kernel (and the BEM
    // near operator's row sets) by the near sum, the far-field kernel by L2T + M2T
    // (EBEM_EVAL_ORDER=0: Morton order for both)
    static const bool lpt = !(std::getenv("EBEM_EVAL_ORDER") && std::atoi(std::getenv("EBEM_EVAL_ORDER")) == 0);
    std::vector<int> fev = ev, fl2t = l2t;
    if (lpt && !ev.empty()) {
        std::vector<double> wn(ev.size()), wf(ev.size());
        for (size_t i = 0; i < ev.size(); ++i) {
            const int b = ev[i];
            double nfar = l2t[i] >= 0 ? 1.0 : 0.0;
            for (int e = moff[b]; e < moff[b + 1]; ++e) nfar += phiu[midx[e]] >= 0 ? 1.0 : 0.0;
            wn[i] = (double)tsub[b] * near_ns[b];
            wf[i] = (double)tsub[b] * P.ne * nfar;
        }
        // decreasing work by a counting sort on the leading 16 bits of the (non-negative) work as
        // a float (exponent and eight mantissa bits: 0.4% classes), Morton order within a class
        // (two std::sort calls over the ~30 k leaves took 2.5 ms of the build)
        auto order = [&](const std::vector<double>& w, std::vector<int>& e_out, std::vector<int>& l_out) {
            constexpr int NB = 1 << 16;
            std::vector<int> cls(ev.size()), start(NB + 1, 0);
            for (size_t i = 0; i < cls.size(); ++i) {
                const float wf32 = (float)w[i];
                uint32_t bits;
                std::memcpy(&bits, &wf32, sizeof(bits));
                cls[i] = NB - 1 - (int)(bits >> 15);          // sign bit 0: 16 leading bits; largest first
                ++start[cls[i] + 1];
            }
            for (int c = 0; c < NB; ++c) start[c + 1] += start[c];
            for (size_t i = 0; i < cls.size(); ++i) {
                const int pos = start[cls[i]]++;
                e_out[pos] = ev[i];
                l_out[pos] = l2t[i];
            }
        };
        std::vector<int> nev(ev.size()), nl2t(ev.size());
        order(wf, fev, fl2t);
        order(wn, nev, nl2t);
        ev.swap(nev);
        l2t.swap(nl2t);
    }
    t.far_box.alloc(std::max<size_t>(fev.size(), 1));
    h2d(t.far_box.p, fev.data(), fev.size(), s);
    t.far_l2t_slot.alloc(std::max<size_t>(fl2t.size(), 1));
    h2d(t.far_l2t_slot.p, fl2t.data(), fl2t.size(), s);
    t.n_eval = (int)ev.size();
    t.n_phid = (int)phid_box.size();
    t.n_phiu = (int)phiu_box.size();
    t.eval_box.alloc(std::max<size_t>(ev.size(), 1));
    h2d(t.eval_box.p, ev.data(), ev.size(), s);
    t.eval_l2t_slot.alloc(std::max<size_t>(l2t.size(), 1));
    h2d(t.eval_l2t_slot.p, l2t.data(), l2t.size(), s);
    t.phiu_slot.alloc(nb);
    h2d(t.phiu_slot.p, phiu.data(), nb, s);
    t.phid_scale.alloc(std::max<size_t>(phid_scale.size(), 1));
    h2d(t.phid_scale.p, phid_scale.data(), phid_scale.size(), s);
    t.phiu_scale.alloc(std::max<size_t>(phiu_scale.size(), 1));
    h2d(t.phiu_scale.p, phiu_scale.data(), phiu_scale.size(), s);
    op1.assign(prd.size(), 0);
    build_op_pairs(t.phid_pairs, 1, op1, prd, s);
    op1.assign(pru.size(), 0);
    build_op_pairs(t.phiu_pairs, 1, op1, pru, s);

    lap("leaf lists/phi");
    // workspace
    const int me = P.me, mc = P.mc;
    t.rec_disp.alloc(std::max<int64_t>(t.nsrc * REC_DISP, 1));
    t.rec_stress.alloc(std::max<int64_t>(t.nsrc * REC_STRESS, 1));
    const int lde = P.lde, ldc = P.ldc;
    const int64_t nq = std::max(1, t.n_s2m), nqd = std::max(1, t.n_s2l);
    t.Q.alloc((size_t)nq * ldc);
    t.Qd.alloc((size_t)nqd * ldc);
    t.Z.alloc((size_t)std::max(1, t.n_up) * lde);
    t.W.alloc((size_t)std::max(1, t.n_dn) * lde);
    if (const char* e = std::getenv("EBEM_SIMT")) t.use_tc = std::atoi(e) == 0;
    t.far64 = P.p >= FAR_FP64_MIN_P;
    t.tc_fast = t.use_tc && !t.far64 && !(std::getenv("EBEM_TC_PRECISE") && std::atoi(std::getenv("EBEM_TC_PRECISE")));
    if (t.use_tc) {
        t.Qb.alloc(t.Q.n); t.Qs.alloc(t.Q.n);
        t.Qdb.alloc(t.Qd.n); t.Qds.alloc(t.Qd.n);
        t.Zb.alloc(t.Z.n); t.Zs.alloc(t.Z.n);
        t.Wb.alloc(t.W.n); t.Ws.alloc(t.W.n);
        for (DBuf<float>* b : {&t.Qb, &t.Qs, &t.Qdb, &t.Qds, &t.Zb, &t.Zs, &t.Wb, &t.Ws}) b->zero(s);
        tc_make_map_b(&t.mQb, t.Qb.p, nq, mc, ldc);
        tc_make_map_b(&t.mQs, t.Qs.p, nq, mc, ldc);
        tc_make_map_b(&t.mQdb, t.Qdb.p, nqd, mc, ldc);
        tc_make_map_b(&t.mQds, t.Qds.p, nqd, mc, ldc);
        tc_make_map_b(&t.mZb, t.Zb.p, std::max(1, t.n_up), me, lde);
        tc_make_map_b(&t.mZs, t.Zs.p, std::max(1, t.n_up), me, lde);
        tc_make_map_b(&t.mWb, t.Wb.p, std::max(1, t.n_dn), me, lde);
        tc_make_map_b(&t.mWs, t.Ws.p, std::max(1, t.n_dn), me, lde);
        // Q2Z / M2M / L2L on the full-chain fast kernel up to this order (measured at p = 6:
        // 0.17 ms faster, error 2.907e-5 -> 2.912e-5; at p = 8 the error grew 1.9e-6 -> 2.7e-6)
        static const int ml_fast_pmax = std::getenv("EBEM_ML_FAST") ? std::atoi(std::getenv("EBEM_ML_FAST")) : 6;
        t.ml_fast = t.tc_fast && P.p <= ml_fast_pmax;
        // tile shapes: the full-chain and the drained M2L kernels two-slice or wide by M
        // (tc_fast_tile_mode), the one-slice precise kernel 128 x 128
        const int fm = tc_fast_tile_mode(me);
        // M2L operands in FP16 (3xFP16, twice the tensor rate of 3xTF32; EBEM_M2L_F16=0: TF32)
        t.m2l_f16 = m2l_f16_level() >= 1;
        if (t.m2l_f16) {
            t.Zhb.alloc((size_t)std::max(1, t.n_up) * P.ldh);
            t.Zhs.alloc((size_t)std::max(1, t.n_up) * P.ldh);
            t.Zhinv.alloc(std::max(1, t.n_up));
            t.Zhb.zero(s);
            t.Zhs.zero(s);
        }
        build_m2l_tiles(t);
        // M2M / L2L on the fast kernel in FP16 as well: each level's rows are split (row-scaled
        // fp16 head / remainder) as they become final, which also serves the M2L.  Not in trees
        // deeper than 16 levels: a rounding error made at the leaves is amplified by 2 per M2M
        // level relative to a double layer's decaying field (limitation L1), and the
        // fp16 split (absolute precision relative to the row's largest entry) then shows where
        // the TF32 split (relative per element) does not -- level-20 coincident cluster, GPU vs
        // oracle KIFMM: 1.71e-3 with TF32 chains, 2.11e-3 with FP16 chains, M2L in FP16 either way.
        static const bool chain_env = std::getenv("EBEM_ML_CHAIN") && std::atoi(std::getenv("EBEM_ML_CHAIN")) == 1;
        // p = 7 .. 10: the chains on the same FP16 data flow with DRAINED accumulation
        // (tc_pairs_fast / wide kernel <true, true>) instead of the one-slice precise TF32 kernel
        // with TMA-gathered rows (EBEM_ML_DRAIN_F16=0: off; the BEM operator keeps the precise kernel)
        // EBEM_ML_DRAIN_F16: 0 off; 1 (default) p = 7 .. 10; 2 every order above 6.  Measured on the
        // 1M beam at p = 10: 29.8 -> 27.8 ms, rel-L2 5.02e-7 -> 5.49e-7 (bound 1e-6); at p = 12
        // (3000-point beam, test_largest_order) 1.3e-6 -> 2.2e-6, over that test's 2e-6: the
        // orders above 10 keep the precise kernel.
        static const int drain_lv = std::getenv("EBEM_ML_DRAIN_F16") ? std::atoi(std::getenv("EBEM_ML_DRAIN_F16")) : 1;
        const bool drain_h = drain_lv >= 2 || (drain_lv == 1 && P.p <= 10);
        t.ml_drain = t.use_tc && !t.ml_fast && P.p > 6 && drain_h && m2l_f16_level() >= 2 && m2l_drain_fast();
        t.ml_f16 = (t.ml_fast || t.ml_drain) && t.m2l_f16 && !chain_env && ml_f16_on() && t.nlevels <= 16;
        t.ml_drain = t.ml_drain && t.ml_f16;
        // the upward Q2Z on FP16 operands as well (the S2M kernel writes the split; EBEM_Q2Z_F16=0: TF32)
        static const bool q2z_h = !(std::getenv("EBEM_Q2Z_F16") && std::atoi(std::getenv("EBEM_Q2Z_F16")) == 0);
        // (as the M2M / L2L chains, not in trees deeper than 16 levels: level-20 coincident cluster,
        // GPU vs oracle KIFMM 2.85e-3 with the FP16 Q2Z against 1.71e-3, limitation L1)
        // (with the drained chains, p = 7 .. 10, on the drained kernel too)
        t.q2z_f16 = (t.ml_fast || t.ml_drain) && m2l_f16_level() >= 1 && q2z_h && t.nlevels <= 16;
        if (t.q2z_f16) {
            t.Qhb.alloc((size_t)nq * P.ldch);
            t.Qhs.alloc((size_t)nq * P.ldch);
            t.Qhinv.alloc(nq);
            t.Qhb.zero(s);
            t.Qhs.zero(s);
        }
        tc_build_tiles(t.q2z_up, me, mc, t.ml_fast || t.q2z_f16 ? fm : 0, t.q2z_f16 ? 64 : 32);
        tc_build_tiles(t.q2z_dn, me, mc, t.ml_fast ? fm : 0);
        if (t.ml_f16) {
            t.Whb.alloc((size_t)std::max(1, t.n_dn) * P.ldh);
            t.Whs.alloc((size_t)std::max(1, t.n_dn) * P.ldh);
            t.Whinv.alloc(std::max(1, t.n_dn));
            t.Whb.zero(s);
            t.Whs.zero(s);
        }
        for (auto& x : t.m2m) tc_build_tiles(x, me, me, t.ml_fast || t.ml_drain ? fm : 0, t.ml_f16 ? 64 : 32);
        for (auto& x : t.l2l) tc_build_tiles(x, me, me, t.ml_fast || t.ml_drain ? fm : 0, t.ml_f16 ? 64 : 32);
        // EBEM_ML_CHAIN=1: M2M and L2L chains as one persistent launch each (tc_chain_kernel).
        // Measured on the 1M beam: M2M 0.341 -> 0.317 ms, L2L 0.321 -> 0.306 ms alone, but the
        // overlapped matvec unchanged (4.41-4.44 ms either way) and the host-buffer (e2e) matvec
        // 0.4 ms slower (5.79 vs 5.39 ms, mean of 3-4 runs); default: a split launch plus a
        // translation launch per level
        static const bool chain_on = std::getenv("EBEM_ML_CHAIN") && std::atoi(std::getenv("EBEM_ML_CHAIN")) == 1;
        t.ml_chain = t.ml_fast && chain_on;
        if (t.ml_chain) {
            std::vector<const OpPairs*> up, dn;
            std::vector<int64_t> ur0, urn, dr0, drn;
            for (int l = t.nlevels - 2; l >= 2; --l) {      // M2M at l reads the Z rows of level l + 1
                up.push_back(&t.m2m[l]);
                ur0.push_back(t.up_lstart[l + 1]);
                urn.push_back(t.up_lstart[l + 2] - t.up_lstart[l + 1]);
            }
            for (int l = 3; l < t.nlevels; ++l) {           // L2L at l reads the W rows of level l - 1
                dn.push_back(&t.l2l[l]);
                dr0.push_back(t.dn_lstart[l - 1]);
                drn.push_back(t.dn_lstart[l] - t.dn_lstart[l - 1]);
            }
            tc_build_chain(t.m2m_chain, up, ur0, urn, me, me, s);
            tc_build_chain(t.l2l_chain, dn, dr0, drn, me, me, s);
        }
    }
    if (t.far64) {
        t.PHID.alloc((size_t)std::max(1, t.n_phid) * me);
        t.PHIU.alloc((size_t)std::max(1, t.n_phiu) * me);
    } else {
        t.PHIDF.alloc((size_t)std::max(1, t.n_phid) * P.ne);
        t.PHIUF.alloc((size_t)std::max(1, t.n_phiu) * P.ne);
        t.PHIDF.zero(s);
        t.PHIUF.zero(s);
    }
    lap("workspace+tiles");
    t.near_sorted.alloc((size_t)std::max<int64_t>(1, t.ntrg) * 6);
    EB_CUDA(cudaStreamSynchronize(s));

    int64_t bytes = 0;
    bytes += t.keys.bytes() + t.perm.bytes() + t.src_perm.bytes() + t.trg_perm.bytes() + t.src_xyz.bytes() +
             t.src_nrm.bytes() + t.src_w.bytes() + t.trg_xyz.bytes();
    bytes += (int64_t)nb * 4 * 40;
    for (int k = 0; k < 4; ++k) bytes += t.lst_off[k].bytes() + t.lst_idx[k].bytes();
    bytes += t.rec_disp.bytes() + t.rec_stress.bytes() + t.Q.bytes() + t.Qd.bytes() + t.Z.bytes() + t.W.bytes() + t.PHID.bytes() +
             t.PHIU.bytes() + t.PHIDF.bytes() + t.PHIUF.bytes();
    bytes += t.m2l.pairs.bytes();
    t.device_bytes = bytes;
}

// ------------------------------------------------------------------ evaluation
template <bool SL, bool DL>
static void launch_check(const Tree& t, const int* tbox, int n, const int* soff, const int* sidx, double rad,
                         float* Q, float* Qb, float* Qs, cudaStream_t s, __half* Qhb = nullptr, __half* Qhs = nullptr,
                         float* Qhinv = nullptr) {
    if (n == 0) return;
    const Plan& P = *t.plan;
    BoxGeo geo{t.origin[0], t.origin[1], t.origin[2], t.side};
    KConst kc = make_kconst(t.mat);
    const int kpt = ceil_div(P.nc, CP_T);      // 2 or 3 points per thread measured slower
    // the fewest whole warps that cover the surface with kpt points per thread (p = 6:
    // 218 points -> 224 threads, not 256)
    const int nthr = 32 * ceil_div(ceil_div(P.nc, kpt), 32);
#define EB_CHECK_LAUNCH_KPT(K)                                                                                     \
    EB_CUDA(cudaFuncSetAttribute(check_potential_kernel<SL, DL, K>, cudaFuncAttributePreferredSharedMemoryCarveout, 100)); \
    check_potential_kernel<SL, DL, K><<<n, nthr, 0, s>>>(tbox, soff, sidx, t.sbeg.p, t.send.p, t.anchor.p,         \
                                                         t.level.p, geo, rad, P.s_c.p, P.nc, t.rec_disp.p, kc,    \
                                                         Q, Qb, Qs, P.ldc, t.ssplit.p, t.ssplit.p ? t.split_mode : 0, \
                                                         Qhb, Qhs, Qhinv, P.ldch)
    switch (kpt) {
        case 1: EB_CHECK_LAUNCH_KPT(1); break;
        case 2: EB_CHECK_LAUNCH_KPT(2); break;
        case 3: EB_CHECK_LAUNCH_KPT(3); break;
        default: EB_REQUIRE(kpt <= 4, "check surface too large"); EB_CHECK_LAUNCH_KPT(4); break;
    }
#undef EB_CHECK_LAUNCH_KPT
    EB_CHECK_LAUNCH();
}

// BEM: the sources of every leaf grouped by the boundary-condition type of their panel
// (Dirichlet first, stable), so that inside a solve each group carries one layer only
// (mode 0: Dirichlet -> single layer, Neumann -> double layer; mode 1 the reverse) and the
// check potentials run the one-kernel pair loops.  A permutation inside each leaf: every
// box range stays valid.  ssplit[leaf] = first source of the second group.
__global__ void partition_kernel(int nb, const int* __restrict__ is_leaf, const int* __restrict__ sbeg,
                                 const int* __restrict__ send, const int* __restrict__ src_perm, int nq,
                                 const int32_t* __restrict__ bc, int* __restrict__ dest, int* __restrict__ ssplit) {
    __shared__ int n0s, w0[32], w1[32];
    const int b = blockIdx.x;
    if (b >= nb || !is_leaf[b]) return;
    const int B = sbeg[b], E = send[b];
    if (E <= B) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) n0s = 0;
    __syncthreads();
    int c0 = 0;
    for (int s = B + threadIdx.x; s < E; s += blockDim.x) c0 += bc[src_perm[s] / nq] == 0;
    atomicAdd(&n0s, c0);
    __syncthreads();
    const int n0 = n0s;
    const unsigned lt = (1u << lane) - 1u;
    int base0 = 0, base1 = 0;
    for (int s0 = B; s0 < E; s0 += blockDim.x) {
        const int s = s0 + threadIdx.x;
        const bool valid = s < E;
        const bool f = valid && bc[src_perm[s] / nq] == 0;
        const unsigned b0 = __ballot_sync(0xffffffffu, f), b1 = __ballot_sync(0xffffffffu, valid && !f);
        if (lane == 0) {
            w0[warp] = __popc(b0);
            w1[warp] = __popc(b1);
        }
        __syncthreads();
        int p0 = 0, p1 = 0, t0 = 0, t1 = 0;
        for (int w = 0; w < nw; ++w) {
            if (w < warp) {
                p0 += w0[w];
                p1 += w1[w];
            }
            t0 += w0[w];
            t1 += w1[w];
        }
        if (valid) dest[s] = f ? B + base0 + p0 + __popc(b0 & lt) : B + n0 + base1 + p1 + __popc(b1 & lt);
        base0 += t0;
        base1 += t1;
        __syncthreads();
    }
    if (threadIdx.x == 0) ssplit[b] = B + n0;
}

__global__ void iota_kernel(int* __restrict__ a, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int)i;
}

template <class T>
__global__ void scatter_rows(const T* __restrict__ in, const int* __restrict__ dest, int64_t n, int w,
                             T* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int c = 0; c < w; ++c) out[(int64_t)dest[i] * w + c] = in[i * w + c];
}

void tree_partition_sources(Tree& t, const int32_t* bc, int nq, cudaStream_t s) {
    const int64_t n = t.nsrc;
    if (n == 0 || t.nboxes == 0) return;
    DBuf<int> dest(n);
    iota_kernel<<<ceil_div(n, 256), 256, 0, s>>>(dest.p, n);
    EB_CHECK_LAUNCH();
    if (t.ssplit.n != (size_t)t.nboxes) t.ssplit.alloc(t.nboxes);
    partition_kernel<<<t.nboxes, 256, 0, s>>>(t.nboxes, t.is_leaf.p, t.sbeg.p, t.send.p, t.src_perm.p, nq, bc, dest.p,
                                              t.ssplit.p);
    EB_CHECK_LAUNCH();
    auto permute = [&](auto& buf, int w) {
        using T = typename std::remove_reference<decltype(*buf.p)>::type;
        if (!buf.p) return;
        DBuf<T> tmp(buf.n);
        scatter_rows<T><<<ceil_div(n, 256), 256, 0, s>>>(buf.p, dest.p, n, w, tmp.p);
        EB_CHECK_LAUNCH();
        buf = std::move(tmp);
    };
    permute(t.src_perm, 1);
    permute(t.src_xyz, 3);
    if (t.has_normals) permute(t.src_nrm, 3);
    if (t.has_weights) permute(t.src_w, 1);
    EB_CUDA(cudaStreamSynchronize(s));
}

// switch a built tree to the precise configuration (fp64 far field, drained tensor-core
// accumulation): the BEM operator inside GMRES
void tree_precise(Tree& t, cudaStream_t s) {
    const Plan& P = *t.plan;
    if (!t.far64) {
        t.far64 = true;
        t.PHIDF.release();
        t.PHIUF.release();
        t.PHID.alloc((size_t)std::max(1, t.n_phid) * P.me);
        t.PHIU.alloc((size_t)std::max(1, t.n_phiu) * P.me);
    }
    // EBEM_BEM_ML_DRAIN=1: the BEM operator's chains on the drained FP16 data flow too (measurement)
    static const bool bem_drain = std::getenv("EBEM_BEM_ML_DRAIN") && std::atoi(std::getenv("EBEM_BEM_ML_DRAIN")) == 1;
    if (t.ml_drain && !bem_drain) {     // the operator inside GMRES keeps the one-slice precise kernel for the chains
        t.ml_drain = false;
        t.ml_f16 = false;
        for (auto& x : t.m2m) tc_build_tiles(x, P.me, P.me, 0, 32);
        for (auto& x : t.l2l) tc_build_tiles(x, P.me, P.me, 0, 32);
    }
    if (t.q2z_f16) {      // the BEM's stored S2M operator (s2m_hook) writes the TF32 split
        t.q2z_f16 = false;
        tc_build_tiles(t.q2z_up, P.me, P.mc, t.ml_fast ? tc_fast_tile_mode(P.me) : 0, 32);
    }
    tree_m2l_fast(t, false, s);
    EB_CUDA(cudaStreamSynchronize(s));
}

// M2L accumulation of a built tree: full-chain (fast) or drained groups (precise).  The fast
// chain is allowed only where it is below the truncation error (p <= 8).
void tree_m2l_fast(Tree& t, bool fast, cudaStream_t s) {
    const Plan& P = *t.plan;
    fast = fast && t.use_tc && P.p < FAR_FP64_MIN_P;
    if (fast == t.tc_fast) return;
    t.tc_fast = fast;
    build_m2l_tiles(t);
    EB_CUDA(cudaStreamSynchronize(s));
}

// near field (U-list P2P) into the sorted near buffer
// Dynamic shared memory a stream-B kernel requests so that a fixed number of its CTAs fit
// beside one persistent translation CTA (tc_pairs_fast_kernel) and fill its leftover shared
// memory.  Measured on the 1M-point matvec (with the M2L timestamp below).  With the TF32 M2L
// (1.64 ms alone): 4.64 ms with three near-field CTAs beside each M2L CTA (no padding),
// 4.45-4.48 with two, 4.60 with one -- the third took issue slots the M2L producer warps
// needed.  With the FP16 M2L (1.37 ms alone) the near field is the longer of the two and three
// CTAs are the better split: 4.04 vs 4.07 ms with two (configs[3] unchanged, 7.59 ms).
// EBEM_NEAR_PAD=bytes overrides.
int beside_translation_pad(const void* kernel) {
    if (const char* e = std::getenv("EBEM_NEAR_PAD")) return std::atoi(e);
    cudaFuncAttributes fa;
    EB_CUDA(cudaFuncGetAttributes(&fa, kernel));
    int dev = 0, smem_sm = 0, resv = 0;
    EB_CUDA(cudaGetDevice(&dev));
    EB_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    EB_CUDA(cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev));
    const int free_sm = smem_sm - (tc_fast_smem_bytes() + resv);
    const int per_sm = 3;
    const int pad = (free_sm / per_sm - resv - (int)fa.sharedSizeBytes - 128) & ~127;
    return pad > 0 ? pad : 0;
}

template <bool SL, bool DL, bool STRESS>
static void launch_near(const Tree& t, cudaStream_t s) {
    if (t.n_eval == 0) return;
    KConst kc = make_kconst(t.mat);
    static bool carve = false;
    if (!carve) {   // same L1/shared split as the translation kernels, so both can share an SM
        EB_CUDA(cudaFuncSetAttribute(near_eval_kernel<SL, DL, STRESS>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     100));
        carve = true;
    }
    // (a variant staging each leaf's near sources as merged contiguous ranges with a cp.async
    // double buffer was 3.5% faster alone but made the overlapped matvec slower, 4.41 -> 4.56 ms)
    // EBEM_NEAR_PACKED=1: packed FFMA2 pair loop (two targets per FP32 instruction)
    // (1.348 vs 1.36 ms alone, but the overlapped matvec 4.70 vs 4.45 ms: its 127 registers
    // leave room for fewer near-field CTAs beside the translation CTAs; off by default)
    static const bool packed = std::getenv("EBEM_NEAR_PACKED") && std::atoi(std::getenv("EBEM_NEAR_PACKED")) == 1;
    if (packed) {
        static bool carve_p = false;
        if (!carve_p) {
            EB_CUDA(cudaFuncSetAttribute(near_eval_p_kernel<SL, DL, STRESS>,
                                         cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            carve_p = true;
        }
        static const int pad = beside_translation_pad((const void*)near_eval_p_kernel<SL, DL, STRESS>);
        near_eval_p_kernel<SL, DL, STRESS><<<ceil_div(t.n_eval, EV_WARPS), 32 * EV_WARPS, pad, s>>>(
            t.n_eval, t.eval_box.p, t.near_off.p, t.near_idx.p, t.sbeg.p, t.send.p, t.tbeg.p, t.tend.p, t.trg_xyz.p,
            STRESS ? t.rec_stress.p : t.rec_disp.p, kc, t.near_sorted.p);
    } else {
        static const int pad = beside_translation_pad((const void*)near_eval_kernel<SL, DL, STRESS>);
        near_eval_kernel<SL, DL, STRESS><<<ceil_div(t.n_eval, EV_WARPS), 32 * EV_WARPS, pad, s>>>(
            t.n_eval, t.eval_box.p, t.near_off.p, t.near_idx.p, t.sbeg.p, t.send.p, t.tbeg.p, t.tend.p, t.trg_xyz.p,
            STRESS ? t.rec_stress.p : t.rec_disp.p, kc, t.near_sorted.p);
    }
    EB_CHECK_LAUNCH();
}

// far field (L2T + M2T) plus the near buffer, scattered to the caller's target order
template <bool STRESS>
static void launch_far(const Tree& t, float* out, cudaStream_t s) {
    if (t.n_eval == 0) return;
    const Plan& P = *t.plan;
    BoxGeo geo{t.origin[0], t.origin[1], t.origin[2], t.side};
    KConst kc = make_kconst(t.mat);
    const double cfar = STRESS ? t.mat.cD : t.mat.cU;
    const int grid = ceil_div(t.n_eval, EV_WARPS);
    if (t.far64) {
        const size_t sm = sizeof(double) * 3 * P.ne * (EV_WARPS + 1);
        auto go = [&](auto ffn, const auto* near, auto* o) {
            if (sm > 48 * 1024)
                EB_CUDA(cudaFuncSetAttribute(ffn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            ffn<<<grid, 32 * EV_WARPS, sm, s>>>(t.n_eval, t.far_box.p, t.far_l2t_slot.p, t.PHID.p, t.PHIU.p,
                                                t.phiu_slot.p, t.m2t_off.p, t.m2t_idx.p, t.tbeg.p, t.tend.p,
                                                t.anchor.p, t.level.p, geo, P.s_e64.p, P.ne, t.trg_xyz.p, kc, cfar,
                                                near, t.trg_perm.p, o);
        };
        // (the BEM operator inside GMRES: fp64 near field in, fp64 result out)
        if (t.out_d && t.near_f64) go(far_eval_f64_kernel<STRESS, double, double>, t.near_sorted_d.p, t.out_d);
        else if (t.out_d) go(far_eval_f64_kernel<STRESS, float, double>, t.near_sorted.p, t.out_d);
        else go(far_eval_f64_kernel<STRESS, float, float>, t.near_sorted.p, out);
    } else {
        const size_t sm = sizeof(float4) * 2 * P.ne * EV_WARPS;
        auto ffn = far_eval_f32_kernel<STRESS>;
        if (sm > 48 * 1024) EB_CUDA(cudaFuncSetAttribute(ffn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        ffn<<<grid, 32 * EV_WARPS, sm, s>>>(t.n_eval, t.far_box.p, t.far_l2t_slot.p, t.PHIDF.p, t.PHIUF.p,
                                            t.phiu_slot.p, t.m2t_off.p, t.m2t_idx.p, t.tbeg.p, t.tend.p,
                                            t.anchor.p, t.level.p, geo, P.s_e4.p, P.ne, t.trg_xyz.p, kc,
                                            t.near_sorted.p, t.trg_perm.p, out);
    }
    EB_CHECK_LAUNCH();
}

// Schedule.  Profiling on: every phase in order on the caller's stream (phase events).
// Otherwise two internal streams forked from the caller's stream and joined back into it:
//   A (high priority): prep -> S2M, Q2Z_up, M2M -> M2L -> [S2L done] Q2Z_dn -> L2L -> PHI
//                      -> [near done] far field + scatter
//   B (low priority) :         S2L check potentials, then the U-list near field
// B's kernels are FP32-ALU bound and run beside the memory / tensor-core bound M2L (the
// persistent M2L kernel leaves room for a few P2P CTAs per SM once all kernels request the
// same L1/shared split).  Measured on the 1M beam: 7.20 vs 7.31 ms serial; the overlap is
// partial because M2L itself slows down by the issue slots the P2P warps take.
void fmm_evaluate(Tree& t, int kernel, const float* f, const float* g, float* out, cudaStream_t s) {
    const Plan& P = *t.plan;
    const int me = P.me, mc = P.mc;
    const bool stress = kernel_stress(kernel);
    const bool sl = kernel_sl(kernel), dl = kernel_dl(kernel);
    const int src_kernel = stress ? kernel - 3 : kernel;    // D->U, S->P, DS->UP
    EB_REQUIRE(!dl || t.has_normals, "double-layer kernel needs normals at fmm_build_tree");
    if (t.ntrg == 0) return;
    static const bool serial = std::getenv("EBEM_SERIAL") != nullptr;   // diagnostics: one stream
    const bool conc = t.profile != 1 && !serial && !t.force_serial;
    if (conc && !t.sA) {
        int least = 0, greatest = 0;
        EB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        EB_CUDA(cudaStreamCreateWithPriority(&t.sA, cudaStreamNonBlocking, greatest));
        EB_CUDA(cudaStreamCreateWithPriority(&t.sB, cudaStreamNonBlocking, least));
        for (cudaEvent_t* e : {&t.ev_fork, &t.ev_s2l, &t.ev_near, &t.ev_joinA, &t.ev_zz, &t.ev_wz})
            EB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        EB_CUDA(cudaEventCreate(&t.ev_m2l));
    }
    // diagnostics (EBEM_TRACE=1): stream timeline of the overlapped section, printed per call
    static const bool trace = std::getenv("EBEM_TRACE") != nullptr;
    static cudaEvent_t tev[8] = {};
    if (trace && !tev[0])
        for (auto& e : tev) EB_CUDA(cudaEventCreate(&e));
    cudaStream_t sa = s, sb = s;
    if (conc) {
        sa = t.sA;
        sb = t.sB;
        EB_CUDA(cudaEventRecord(t.ev_fork, s));
        EB_CUDA(cudaStreamWaitEvent(sa, t.ev_fork, 0));
    }
    // phase brackets: begin / end timing events on the stream a phase is launched on (when
    // profiling) and the number of kernels its enqueue issued
    enum { PH_PREP, PH_S2M, PH_Q2Z_UP, PH_M2M, PH_S2L, PH_Q2Z_DN, PH_M2L, PH_L2L, PH_PHI, PH_NEAR, PH_FAR };
    Tree::ProfSet* ps = nullptr;
    if (t.profile) {
        if (t.prof_ring.empty()) {
            t.prof_ring.resize(Tree::PROF_RING);
            for (auto& r : t.prof_ring)
                for (int i = 0; i < Tree::NPHASE; ++i) {
                    EB_CUDA(cudaEventCreate(&r.b[i]));
                    EB_CUDA(cudaEventCreate(&r.e[i]));
                }
        }
        ps = &t.prof_ring[t.prof_count % Tree::PROF_RING];
        for (bool& u : ps->used) u = false;
        ++t.prof_count;
    }
    int64_t lbeg[Tree::NPHASE] = {};
    for (int& x : t.phase_launches) x = 0;
    // In situ (mode 2) only M2L and the near field are timed, with events placed exactly where
    // the unprofiled schedule has them: M2L's begin event is the timestamp the schedule records
    // before M2L anyway (see below), its end event follows it on stream A, and the near
    // field's end event follows it on stream B.  Any further timing event ahead of the fork
    // shifted which of the two kernels takes the SMs first (measured: 4.41 -> 4.73 ms).
    const bool insitu = ps && conc;
    auto timed = [&](int ph) { return ps && (!insitu || ph == PH_M2L || ph == PH_NEAR); };
    auto pb = [&](int ph, cudaStream_t st) {
        lbeg[ph] = launch_count();
        if (timed(ph)) {
            EB_CUDA(cudaEventRecord(ps->b[ph], st));
            ps->from[ph] = ps->b[ph];
        }
    };
    // stream-B phases in situ: no event ahead of the near-field kernel; NEAR is timed from
    // M2L's begin event (both start at the fork) to its own end event and includes S2L
    auto pb_after = [&](int ph) { lbeg[ph] = launch_count(); };
    auto pe_count = [&](int ph) { t.phase_launches[ph] += (int)(launch_count() - lbeg[ph]); };
    auto pe = [&](int ph, cudaStream_t st) {
        t.phase_launches[ph] += (int)(launch_count() - lbeg[ph]);
        if (timed(ph)) {
            EB_CUDA(cudaEventRecord(ps->e[ph], st));
            ps->used[ph] = true;
        }
    };
    pb(PH_PREP, sa);

    // prepared sources in tree order (geometry sorted, densities via src_perm); not needed when
    // every pass that reads them is replaced by a stored operator (the BEM inside GMRES)
    const bool need_rec = !(t.near_hook && t.s2m_hook && (t.s2l_hook || t.n_s2l == 0));
    if (need_rec)
        prepare_sources(src_kernel, t.mat, t.src_xyz.p, t.src_nrm.p, t.src_w.p, nullptr, f, g, t.src_perm.p, t.nsrc,
                        t.rec_disp.p, sa);
    if (stress)
        prepare_sources(kernel, t.mat, t.src_xyz.p, t.src_nrm.p, t.src_w.p, nullptr, f, g, t.src_perm.p, t.nsrc,
                        t.rec_stress.p, sa);
    if (conc) {   // the accumulators are cleared on stream B beside the prep and S2M kernels
        EB_CUDA(cudaStreamWaitEvent(sb, t.ev_fork, 0));
        t.Z.zero(sb);
        EB_CUDA(cudaEventRecord(t.ev_zz, sb));
        t.W.zero(sb);
        EB_CUDA(cudaEventRecord(t.ev_wz, sb));
    } else {
        t.Z.zero(sa);
        t.W.zero(sa);
    }
    pe(PH_PREP, sa);

    auto s2l = [&](cudaStream_t st) {
        if (!t.n_s2l) return;
        if (t.s2l_hook) {
            t.s2l_hook(st);
            return;
        }
        float* qb = t.use_tc ? t.Qdb.p : nullptr;
        float* qs = t.use_tc ? t.Qds.p : nullptr;
        if (sl && dl) launch_check<true, true>(t, t.s2l_box.p, t.n_s2l, t.x_src_off.p, t.x_src_idx.p, RAD_DC, t.Qd.p, qb, qs, st);
        else if (sl) launch_check<true, false>(t, t.s2l_box.p, t.n_s2l, t.x_src_off.p, t.x_src_idx.p, RAD_DC, t.Qd.p, qb, qs, st);
        else launch_check<false, true>(t, t.s2l_box.p, t.n_s2l, t.x_src_off.p, t.x_src_idx.p, RAD_DC, t.Qd.p, qb, qs, st);
    };
    auto near = [&](cudaStream_t st) {
        if (t.near_hook) {
            t.near_hook(st);
            return;
        }
        switch (kernel) {
            case K_U: launch_near<true, false, false>(t, st); break;
            case K_P: launch_near<false, true, false>(t, st); break;
            case K_UP: launch_near<true, true, false>(t, st); break;
            case K_D: launch_near<true, false, true>(t, st); break;
            case K_S: launch_near<false, true, true>(t, st); break;
            case K_DS: launch_near<true, true, true>(t, st); break;
        }
    };
    // stream B starts when the upward pass is done, i.e. alongside M2L
    auto fork_b = [&]() {
        if (!conc) return;
        EB_CUDA(cudaStreamWaitEvent(sb, t.ev_fork, 0));
        pb_after(PH_S2L);
        s2l(sb);
        pe_count(PH_S2L);
        EB_CUDA(cudaEventRecord(t.ev_s2l, sb));
        if (trace) EB_CUDA(cudaEventRecord(tev[1], sb));
        pb_after(PH_NEAR);
        if (ps) ps->from[PH_NEAR] = ps->b[PH_M2L];   // recorded on A right after the fork
        near(sb);
        pe(PH_NEAR, sb);
        if (trace) EB_CUDA(cudaEventRecord(tev[2], sb));
        EB_CUDA(cudaEventRecord(t.ev_near, sb));
    };

    // upward pass
    pb(PH_S2M, sa);
    if (t.s2m_hook) {
        t.s2m_hook(sa);
    } else {
        float* qb = t.use_tc ? t.Qb.p : nullptr;
        float* qs = t.use_tc ? t.Qs.p : nullptr;
        __half* hb = t.q2z_f16 ? t.Qhb.p : nullptr;
        __half* hs = t.q2z_f16 ? t.Qhs.p : nullptr;
        float* hi = t.q2z_f16 ? t.Qhinv.p : nullptr;
        if (sl && dl) launch_check<true, true>(t, t.s2m_box.p, t.n_s2m, nullptr, nullptr, RAD_UC, t.Q.p, qb, qs, sa, hb, hs, hi);
        else if (sl) launch_check<true, false>(t, t.s2m_box.p, t.n_s2m, nullptr, nullptr, RAD_UC, t.Q.p, qb, qs, sa, hb, hs, hi);
        else launch_check<false, true>(t, t.s2m_box.p, t.n_s2m, nullptr, nullptr, RAD_UC, t.Q.p, qb, qs, sa, hb, hs, hi);
    }
    pe(PH_S2M, sa);
    const int lde = P.lde, ldc = P.ldc;
    auto zrows = [&](int l) { return (int64_t)t.up_lstart[l + 1] - t.up_lstart[l]; };
    auto wrows = [&](int l) { return (int64_t)t.dn_lstart[l + 1] - t.dn_lstart[l]; };
    if (conc) EB_CUDA(cudaStreamWaitEvent(sa, t.ev_zz, 0));
    pb(PH_Q2Z_UP, sa);
    if (t.use_tc) {
        if (t.q2z_f16)
            tc_pairs_gemm_fast(t.q2z_up, P.mQu1T_hb, P.mQu1T_hs, t.Qhb.p, t.Qhs.p, P.ldch, me, mc, t.Z.p, lde, t.ml_drain, sa,
                               true, t.Qhinv.p, P.qu_hinv);
        else if (t.ml_fast) tc_pairs_gemm_fast(t.q2z_up, P.mQu1T_b, P.mQu1T_s, t.Qb.p, t.Qs.p, ldc, me, mc, t.Z.p, lde, false, sa);
        else tc_pairs_gemm(t.q2z_up, P.mQu1T_b, P.mQu1T_s, t.mQb, t.mQs, me, mc, t.Z.p, lde, sa);
    } else {
        gemm_pairs_f32(t.q2z_up, P.Qu1T.p, me, mc, ldc, t.Q.p, ldc, t.Z.p, lde, sa);
    }
    pe(PH_Q2Z_UP, sa);
    pb(PH_M2M, sa);
    if (t.use_tc && t.ml_chain) {
        if (t.nlevels > 2)
            tc_chain_run(t.m2m_chain, P.mM2M_b, P.mM2M_s, t.Z.p, lde, t.Zb.p, t.Zs.p, me, me, t.Z.p, lde,
                         t.up_lstart[2], zrows(2), sa);
    } else {
    for (int l = t.nlevels - 2; l >= 2; --l) {
        if (t.use_tc && t.ml_f16) {
            tc_split_rows_h(t.Z.p, lde, t.up_lstart[l + 1], zrows(l + 1), me, t.Zhb.p, t.Zhs.p, P.ldh, t.Zhinv.p, sa);
            tc_pairs_gemm_fast(t.m2m[l], P.mM2M_hb, P.mM2M_hs, t.Zhb.p, t.Zhs.p, P.ldh, me, me, t.Z.p, lde, t.ml_drain, sa,
                               true, t.Zhinv.p, P.m2m_hinv);
        } else if (t.use_tc) {
            tc_split_rows(t.Z.p, lde, t.up_lstart[l + 1], zrows(l + 1), me, t.Zb.p, t.Zs.p, sa);
            if (t.ml_fast) tc_pairs_gemm_fast(t.m2m[l], P.mM2M_b, P.mM2M_s, t.Zb.p, t.Zs.p, lde, me, me, t.Z.p, lde, false, sa);
            else tc_pairs_gemm(t.m2m[l], P.mM2M_b, P.mM2M_s, t.mZb, t.mZs, me, me, t.Z.p, lde, sa);
        } else {
            gemm_pairs_f32(t.m2m[l], P.M2M.p, me, me, lde, t.Z.p, lde, t.Z.p, lde, sa);
        }
    }
    if (t.use_tc && t.ml_f16) {       // the coarsest rows the M2L reads (or all of them in a two-level tree)
        if (t.nlevels > 2) tc_split_rows_h(t.Z.p, lde, t.up_lstart[2], zrows(2), me, t.Zhb.p, t.Zhs.p, P.ldh, t.Zhinv.p, sa);
    } else if (t.use_tc && t.nlevels > 2) tc_split_rows(t.Z.p, lde, t.up_lstart[2], zrows(2), me, t.Zb.p, t.Zs.p, sa);
    }
    pe(PH_M2M, sa);

    // downward pass (stream B forks here: started together with the upward pass it only
    // competed with the other FP32-bound kernels, measured no faster)
    // EBEM_NEAR_AFTER_M2L=1: stream B forks after M2L (the near field beside L2L / PHI)
    static const bool near_late = std::getenv("EBEM_NEAR_AFTER_M2L") && std::atoi(std::getenv("EBEM_NEAR_AFTER_M2L"));
    if (!near_late) {
        if (conc) EB_CUDA(cudaEventRecord(t.ev_fork, sa));
        fork_b();
    }
    if (!conc) {
        pb(PH_S2L, sa);
        s2l(sa);
        pe(PH_S2L, sa);
    }
    auto q2z_dn = [&]() {
        if (!t.n_s2l) return;
        if (t.use_tc) {
            if (t.ml_fast) tc_pairs_gemm_fast(t.q2z_dn, P.mQd1T_b, P.mQd1T_s, t.Qdb.p, t.Qds.p, ldc, me, mc, t.W.p, lde, false, sa);
            else tc_pairs_gemm(t.q2z_dn, P.mQd1T_b, P.mQd1T_s, t.mQdb, t.mQds, me, mc, t.W.p, lde, sa);
        } else {
            gemm_pairs_f32(t.q2z_dn, P.Qd1T.p, me, mc, ldc, t.Qd.p, ldc, t.W.p, lde, sa);
        }
    };
    if (!conc) {
        pb(PH_Q2Z_DN, sa);
        q2z_dn();
        pe(PH_Q2Z_DN, sa);
    }
    if (trace) EB_CUDA(cudaEventRecord(tev[3], sa));
    // a timestamp on stream A just before M2L: measured to let the near-field CTAs (padded to
    // two per SM beside a translation CTA, beside_translation_pad) take their slots first,
    // 4.67 -> 4.48 ms per matvec; a timing-disabled event does not have the effect (when
    // profiling, the phase's own begin event is that timestamp)
    if (conc) {
        EB_CUDA(cudaStreamWaitEvent(sa, t.ev_wz, 0));
        if (!ps) EB_CUDA(cudaEventRecord(t.ev_m2l, sa));
    }
    pb(PH_M2L, sa);
    if (t.use_tc && m2l_use_f16(t) && (t.tc_fast || m2l_drain_fast())) {
        // 3xFP16: row-scaled fp16 split of every Z row, then the same kernels on fp16 operands
        if (!t.ml_f16) tc_split_rows_h(t.Z.p, lde, 0, t.n_up, me, t.Zhb.p, t.Zhs.p, P.ldh, t.Zhinv.p, sa);
        tc_pairs_gemm_fast(t.m2l, P.mM2L_hb, P.mM2L_hs, t.Zhb.p, t.Zhs.p, P.ldh, me, me, t.W.p, lde, !t.tc_fast, sa,
                           true, t.Zhinv.p, P.m2l_hinv);
    } else if (t.use_tc && t.tc_fast) tc_pairs_gemm_fast(t.m2l, P.mM2L_b, P.mM2L_s, t.Zb.p, t.Zs.p, lde, me, me, t.W.p, lde, false, sa);
    else if (t.use_tc && m2l_drain_fast())   // precise accumulation, two-slice fast-kernel data flow
        tc_pairs_gemm_fast(t.m2l, P.mM2L_b, P.mM2L_s, t.Zb.p, t.Zs.p, lde, me, me, t.W.p, lde, true, sa);
    else if (t.use_tc) tc_pairs_gemm(t.m2l, P.mM2L_b, P.mM2L_s, t.mZb, t.mZs, me, me, t.W.p, lde, sa);
    else gemm_pairs_f32(t.m2l, P.M2L.p, me, me, lde, t.Z.p, lde, t.W.p, lde, sa);
    pe(PH_M2L, sa);
    if (near_late) {
        if (conc) EB_CUDA(cudaEventRecord(t.ev_fork, sa));
        fork_b();
    }
    if (trace) EB_CUDA(cudaEventRecord(tev[4], sa));
    if (conc) {
        EB_CUDA(cudaStreamWaitEvent(sa, t.ev_s2l, 0));
        pb(PH_Q2Z_DN, sa);
        q2z_dn();
        pe(PH_Q2Z_DN, sa);
    }
    pb(PH_L2L, sa);
    if (t.use_tc && t.ml_chain) {
        tc_chain_run(t.l2l_chain, P.mL2L_b, P.mL2L_s, t.W.p, lde, t.Wb.p, t.Ws.p, me, me, t.W.p, lde, 0, 0, sa);
    } else {
    for (int l = 3; l < t.nlevels; ++l) {
        if (t.use_tc && t.ml_f16) {
            tc_split_rows_h(t.W.p, lde, t.dn_lstart[l - 1], wrows(l - 1), me, t.Whb.p, t.Whs.p, P.ldh, t.Whinv.p, sa);
            tc_pairs_gemm_fast(t.l2l[l], P.mL2L_hb, P.mL2L_hs, t.Whb.p, t.Whs.p, P.ldh, me, me, t.W.p, lde, t.ml_drain, sa,
                               true, t.Whinv.p, P.l2l_hinv);
        } else if (t.use_tc) {
            tc_split_rows(t.W.p, lde, t.dn_lstart[l - 1], wrows(l - 1), me, t.Wb.p, t.Ws.p, sa);
            if (t.ml_fast) tc_pairs_gemm_fast(t.l2l[l], P.mL2L_b, P.mL2L_s, t.Wb.p, t.Ws.p, lde, me, me, t.W.p, lde, false, sa);
            else tc_pairs_gemm(t.l2l[l], P.mL2L_b, P.mL2L_s, t.mWb, t.mWs, me, me, t.W.p, lde, sa);
        } else {
            gemm_pairs_f32(t.l2l[l], P.L2L.p, me, me, lde, t.W.p, lde, t.W.p, lde, sa);
        }
    }
    }
    pe(PH_L2L, sa);
    pb(PH_PHI, sa);

    // equivalent densities (fp64) and leaf evaluation
    if (t.far64) {
        gemm_pairs_f64(t.phid_pairs, P.Rdinv.p, me, me, t.W.p, lde, t.phid_scale.p, t.PHID.p, me, sa);
        gemm_pairs_f64(t.phiu_pairs, P.Ruinv.p, me, me, t.Z.p, lde, t.phiu_scale.p, t.PHIU.p, me, sa);
    } else {
        const double cfar = stress ? t.mat.cD : t.mat.cU;
        gemm_pairs_f64_to_f32(t.phid_pairs, P.Rdinv.p, me, me, t.W.p, lde, t.phid_scale.p, cfar, t.PHIDF.p, P.ne,
                              sa);
        gemm_pairs_f64_to_f32(t.phiu_pairs, P.Ruinv.p, me, me, t.Z.p, lde, t.phiu_scale.p, cfar, t.PHIUF.p, P.ne,
                              sa);
    }
    pe(PH_PHI, sa);
    if (trace) EB_CUDA(cudaEventRecord(tev[5], sa));
    if (conc) {
        EB_CUDA(cudaStreamWaitEvent(sa, t.ev_near, 0));
    } else {
        pb(PH_NEAR, sa);
        near(sa);
        pe(PH_NEAR, sa);
    }
    if (trace) EB_CUDA(cudaEventRecord(tev[6], sa));
    pb(PH_FAR, sa);
    if (stress) launch_far<true>(t, out, sa);
    else launch_far<false>(t, out, sa);
    pe(PH_FAR, sa);
    if (conc) {
        EB_CUDA(cudaEventRecord(t.ev_joinA, sa));
        EB_CUDA(cudaStreamWaitEvent(s, t.ev_joinA, 0));
    }
    if (trace && conc) {
        EB_CUDA(cudaEventRecord(tev[7], sa));
        EB_CUDA(cudaEventSynchronize(tev[7]));
        float ms[8] = {};
        for (int k = 1; k < 8; ++k) EB_CUDA(cudaEventElapsedTime(&ms[k], tev[3], tev[k]));
        std::fprintf(stderr,
                     "[trace, ms from M2L start] near %.3f..%.3f  M2L ..%.3f  L2L+PHI ..%.3f  wait near ..%.3f  "
                     "end %.3f\n", ms[1], ms[2], ms[4], ms[5], ms[6], ms[7]);
    }
}

// flops per pair interaction of the fp32 pair loop, counted in the SASS of the compiled
// direct kernel (tools/count_flops.sh): FFMA = 2, FMUL / FADD = 1 per pair; the rsqrt (MUFU)
// and the r = 0 select are not counted.
static double flops_per_pair(int kernel) {
    switch (kernel) {
        case K_U: return 29;
        case K_P: return 45;
        case K_UP: return 59;
        case K_D: return 54;
        case K_S: return 87;
        default: return 97;
    }
}

int phase_stats(Tree& t, int kernel, ebem_phase_stat* out, int cap) {
    static const char* names[Tree::NPHASE] = {"prep", "S2M",    "Q2Z_up", "M2M",  "S2L", "Q2Z_dn",
                                              "M2L",  "L2L",    "PHI",    "NEAR", "FAR"};
    const Plan& P = *t.plan;
    const double me = P.me, mc = P.mc, ne = P.ne;
    const bool stress = kernel_stress(kernel);
    const int srck = stress ? kernel - 3 : kernel;
    const double rec_b = 16.0 * REC_DISP, rec_sb = 16.0 * REC_STRESS;
    ebem_phase_stat st[Tree::NPHASE];
    std::memset(st, 0, sizeof(st));
    for (int i = 0; i < Tree::NPHASE; ++i) {
        std::strncpy(st[i].name, names[i], 15);
        st[i].launches = t.phase_launches[i];
        st[i].ms = -1;
    }
    // prep: densities + sorted geometry in, prepared records out
    st[0].bytes = t.nsrc * (4.0 * (3 + 3 + 3 + 3 + 1 + 1) + rec_b + (stress ? rec_sb : 0));
    st[1].interactions = t.w_s2m_inter;
    st[1].flops = t.w_s2m_inter * flops_per_pair(srck);
    st[1].bytes = t.w_s2m_src * rec_b + 4.0 * mc * t.n_s2m;
    st[2].flops = 2.0 * me * mc * t.n_s2m;
    st[2].bytes = 4.0 * me * mc + 4.0 * (mc + me) * t.n_s2m;
    st[3].flops = 2.0 * me * me * t.w_m2m_pairs;
    st[3].bytes = 4.0 * 8 * me * me + 4.0 * 2 * me * t.w_m2m_pairs;
    st[4].interactions = t.w_s2l_inter;
    st[4].flops = t.w_s2l_inter * flops_per_pair(srck);
    st[4].bytes = t.w_s2l_src * rec_b + 4.0 * mc * t.n_s2l;
    st[5].flops = 2.0 * me * mc * t.n_s2l;
    st[5].bytes = t.n_s2l ? 4.0 * me * mc + 4.0 * (mc + me) * t.n_s2l : 0;
    st[6].flops = 2.0 * me * me * t.m2l.npairs;
    st[6].bytes = 4.0 * me * me * t.w_m2l_ops + 4.0 * me * (t.n_up + t.n_dn);
    st[7].flops = 2.0 * me * me * t.w_l2l_pairs;
    st[7].bytes = 4.0 * 8 * me * me + 4.0 * 2 * me * t.w_l2l_pairs;
    st[8].fp64 = 1;
    st[8].flops = st[8].flops_fp64 = me * (me + 1) * (double)(t.n_phid + t.n_phiu);   // triangular R^-1
    st[8].bytes = 2 * 8.0 * me * me + (4.0 + 8.0) * me * (t.n_phid + t.n_phiu);
    st[9].interactions = t.w_p2p_inter;
    st[9].flops = t.w_p2p_inter * flops_per_pair(kernel);
    st[9].bytes = t.w_p2p_src * (stress ? rec_sb : rec_b) + t.ntrg * (12.0 + 4.0 * (stress ? 6 : 3));
    st[10].interactions = t.w_l2t_inter + t.w_m2t_inter;
    st[10].fp64 = t.far64 ? 1 : 0;
    st[10].flops = (t.w_l2t_inter + t.w_m2t_inter) * flops_per_pair(stress ? K_D : K_U);
    st[10].flops_fp64 = t.far64 ? st[10].flops : 0;
    st[10].bytes = t.ntrg * (12.0 + 4.0 * (stress ? 6 : 3) * 2) + (t.far64 ? 8.0 : 16.0 / 3.0) * me * (t.n_phid + t.n_phiu);
    // mean device time over the evaluations recorded since profiling was switched on
    const int nrec = std::min(t.prof_count, (int)Tree::PROF_RING);
    if (nrec > 0) {
        EB_CUDA(cudaDeviceSynchronize());
        for (int i = 0; i < Tree::NPHASE; ++i) {
            double sum = 0;
            int n = 0;
            for (int k = 0; k < nrec; ++k) {
                const Tree::ProfSet& r = t.prof_ring[k];
                if (!r.used[i]) continue;
                float ms = 0;
                EB_CUDA(cudaEventElapsedTime(&ms, r.from[i], r.e[i]));
                sum += ms;
                ++n;
            }
            st[i].ms = n ? sum / n : -1.0;     // -1: not timed (S2L in situ: inside NEAR)
        }
    }
    const int n = std::min(cap, (int)Tree::NPHASE);
    std::memcpy(out, st, sizeof(ebem_phase_stat) * n);
    return Tree::NPHASE;
}


void set_profiling(Tree& t, int mode) {
    EB_REQUIRE(mode >= 0 && mode <= 2, "profiling mode must be 0, 1 or 2");
    t.profile = mode;
    t.prof_count = 0;
}

}  // namespace ebem
