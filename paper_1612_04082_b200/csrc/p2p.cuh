// Prepared source records and the shared-memory tiled pair loops used by the direct
// sum (bem_kernel_direct) and by every point-to-point-like FMM pass (near field, S2M,
// S2L).  PAPER.md Eq. fmm_summation: t_i = sum_j K(x_i, y_j, n_j) s_j.
#pragma once
#include "common.cuh"
#include "elastic.cuh"
#include "packed.cuh"

namespace ebem {

enum KernelId { K_U = 0, K_P = 1, K_UP = 2, K_D = 3, K_S = 4, K_DS = 5 };

inline bool kernel_sl(int k) { return k == K_U || k == K_UP || k == K_D || k == K_DS; }
inline bool kernel_dl(int k) { return k == K_P || k == K_UP || k == K_S || k == K_DS; }
inline bool kernel_stress(int k) { return k >= K_D; }
inline int kernel_ncomp(int k) { return kernel_stress(k) ? 6 : 3; }

// Per-source record, 4 float4 (displacement family) or 6 float4 (stress family):
//   disp   : [y.xyz, q=a (n.g)] [f = cU w f, 0] [g = cP w g, 0] [3 n, 0]
//   stress : [y.xyz, ng = n.g]  [f = cD w f, 0] [g = cS w g, 0] [n, 0]
//            [NG_xx, NG_yy, NG_zz, NG_xy] [NG_yz, NG_xz, 0, 0],  NG = a (n g^T + g n^T)
constexpr int REC_DISP = 4;
constexpr int REC_STRESS = 6;

struct KConst {
    float a1, a, a3, nu, b4;
    float ds_k2, ds_k4, ds_k5;   // D+S pair: 1.5 / a, 3 nu, 1.5 a (acc_DS)
    double a1d, ad, nud, b4d;
};

inline KConst make_kconst(const Material& m) {
    KConst k;
    k.a1 = (float)m.a1; k.a = (float)m.a; k.a3 = (float)(m.a / 3.0); k.nu = (float)m.nu; k.b4 = (float)m.b4;
    k.ds_k2 = (float)(1.5 / m.a); k.ds_k4 = (float)(3.0 * m.nu); k.ds_k5 = (float)(1.5 * m.a);
    k.a1d = m.a1; k.ad = m.a; k.nud = m.nu; k.b4d = m.b4;
    return k;
}

// Build prepared records.  Record i takes its geometry (y, nrm, w) from index
// gperm[i] and its densities (f, g) from index dperm[i] (null perm = identity), so the
// FMM can combine tree-ordered geometry with caller-ordered densities.  w/f/g/nrm may
// be null where the kernel does not use them (w null = 1).
void prepare_sources(int kernel, const Material& m, const float* y, const float* nrm,
                     const float* w, const int* gperm, const float* f, const float* g,
                     const int* dperm, int64_t n, float4* rec, cudaStream_t s);

// ------------------------------------------------------------------ pair loops
#ifndef EBEM_PL_UNROLL
#define EBEM_PL_UNROLL 4
#endif
constexpr int PL_UNROLL = EBEM_PL_UNROLL;

// the same, for TPT targets per thread: the source loop is outermost so that each record is
// read from shared memory once for all TPT targets (one LDS.128 per pair at TPT = 4)
// SAFE = false where no staged source can coincide with a target (check surfaces, boxes
// other than the target's own leaf: coincident points share a Morton key and hence a leaf),
// dropping the r = 0 select from the pair (2 of ~43 instructions for U+P).
template <bool SL, bool DL, bool STRESS, int TPT, bool SAFE = true>
__device__ __forceinline__ void pair_loop_multi(const float4* __restrict__ srec, int cnt, const float* x,
                                                const float* y, const float* z, const KConst& kc, float (*acc)[STRESS ? 6 : 3]) {
    constexpr int R = STRESS ? REC_STRESS : REC_DISP;
#pragma unroll PL_UNROLL
    for (int j = 0; j < cnt; ++j) {
        const float4 p = srec[j * R + 0];
        const float4 f = SL ? srec[j * R + 1] : make_float4(0, 0, 0, 0);
        const float4 g = DL ? srec[j * R + 2] : make_float4(0, 0, 0, 0);
        const float4 n = DL ? srec[j * R + 3] : make_float4(0, 0, 0, 0);
        float NG[6] = {0, 0, 0, 0, 0, 0};
        if (STRESS && DL) {
            const float4 t0 = srec[j * R + 4];
            const float4 t1 = srec[j * R + 5];
            NG[0] = t0.x; NG[1] = t0.y; NG[2] = t0.z; NG[3] = t0.w; NG[4] = t1.x; NG[5] = t1.y;
        }
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
            float dx = x[k] - p.x, dy = y[k] - p.y, dz = z[k] - p.z;
            float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            float ri = SAFE ? safe_rinv(r2) : rsqrtf(r2);
            if (!STRESS) {
                if (SL && DL) acc_UP(dx, dy, dz, ri, f.x, f.y, f.z, g.x, g.y, g.z, n.x, n.y, n.z, p.w, kc.a1, kc.a3, acc[k]);
                else if (SL) acc_U(dx, dy, dz, ri, f.x, f.y, f.z, kc.a1, acc[k]);
                else acc_P(dx, dy, dz, ri, g.x, g.y, g.z, n.x, n.y, n.z, p.w, kc.a3, acc[k]);
            } else {
                if (SL && DL) acc_DS(dx, dy, dz, ri, f.x, f.y, f.z, f.w, g.x, g.y, g.z, n.x, n.y, n.z, p.w, NG, kc, acc[k]);
                else if (SL) acc_D(dx, dy, dz, ri, f.x, f.y, f.z, kc.a, acc[k]);
                else acc_S(dx, dy, dz, ri, g.x, g.y, g.z, n.x, n.y, n.z, p.w, NG, kc.a, kc.nu, kc.b4, acc[k]);
            }
        }
    }
}


// Packed variant: NP pairs of targets per thread, each pair evaluated by FFMA2/FMUL2/FADD2
// against the broadcast source record (packed.cuh: half the FP32 issue slots per pair).
// Records j = g, g + G, ... of the tile at stride RS float4 (g = 0, G = 1, RS = R: all).
struct KConst2 {
    F2 a1, a, a3, nu, b4, ds_k2, ds_k4, ds_k5;
    __device__ __forceinline__ explicit KConst2(const KConst& k)
        : a1(k.a1), a(k.a), a3(k.a3), nu(k.nu), b4(k.b4), ds_k2(k.ds_k2), ds_k4(k.ds_k4), ds_k5(k.ds_k5) {}
};

template <bool SL, bool DL, bool STRESS, int NP, int RS, bool SAFE, int UNROLL = 2>
__device__ __forceinline__ void pair_loop_packed(const float4* __restrict__ srec, int cnt, int g, int G, const F2* x,
                                                 const F2* y, const F2* z, const KConst2& kc,
                                                 F2 (*acc)[STRESS ? 6 : 3]) {
#pragma unroll UNROLL
    for (int j = g; j < cnt; j += G) {
        const float4 p = srec[j * RS + 0];
        const float4 f = SL ? srec[j * RS + 1] : make_float4(0, 0, 0, 0);
        const float4 gg = DL ? srec[j * RS + 2] : make_float4(0, 0, 0, 0);
        const float4 n = DL ? srec[j * RS + 3] : make_float4(0, 0, 0, 0);
        F2 NG[6] = {F2(0.f), F2(0.f), F2(0.f), F2(0.f), F2(0.f), F2(0.f)};
        if (STRESS && DL) {
            const float4 t0 = srec[j * RS + 4];
            const float4 t1 = srec[j * RS + 5];
            NG[0] = F2(t0.x); NG[1] = F2(t0.y); NG[2] = F2(t0.z); NG[3] = F2(t0.w); NG[4] = F2(t1.x); NG[5] = F2(t1.y);
        }
        const F2 px(p.x), py(p.y), pz(p.z), pw(p.w);
        const F2 fx(f.x), fy(f.y), fz(f.z), fw(f.w), gx(gg.x), gy(gg.y), gz(gg.z), nx(n.x), ny(n.y), nz(n.z);
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            const F2 dx = x[k] - px, dy = y[k] - py, dz = z[k] - pz;
            const F2 r2 = fmat(dz, dz, fmat(dy, dy, dx * dx));
            const F2 ri = SAFE ? safe_rinv2(r2) : rsqrt2(r2);
            if (!STRESS) {
                if (SL && DL) acc_UP(dx, dy, dz, ri, fx, fy, fz, gx, gy, gz, nx, ny, nz, pw, kc.a1, kc.a3, acc[k]);
                else if (SL) acc_U(dx, dy, dz, ri, fx, fy, fz, kc.a1, acc[k]);
                else acc_P(dx, dy, dz, ri, gx, gy, gz, nx, ny, nz, pw, kc.a3, acc[k]);
            } else {
                if (SL && DL) acc_DS(dx, dy, dz, ri, fx, fy, fz, fw, gx, gy, gz, nx, ny, nz, pw, NG, kc, acc[k]);
                else if (SL) acc_D(dx, dy, dz, ri, fx, fy, fz, kc.a, acc[k]);
                else acc_S(dx, dy, dz, ri, gx, gy, gz, nx, ny, nz, pw, NG, kc.a, kc.nu, kc.b4, acc[k]);
            }
        }
    }
}

#ifndef NEAR_UNROLL1
#define NEAR_UNROLL1 2
#endif
#ifndef NEAR_UNROLL2
#define NEAR_UNROLL2 2
#endif
// the same for a lane group: records j = g, g + G, ... of the staged tile (stride RS float4),
// TPT targets per thread
template <bool SL, bool DL, bool STRESS, int TPT, int RS, bool SAFE = true>
__device__ __forceinline__ void pair_loop_strided(const float4* __restrict__ srec, int cnt, int g, int G,
                                                  const float* x, const float* y, const float* z, const KConst& kc,
                                                  float (*acc)[STRESS ? 6 : 3]) {
    // independent pair evaluations in flight per lane = TPT x unroll
    constexpr int UN = TPT == 1 ? NEAR_UNROLL1 : (TPT == 2 ? NEAR_UNROLL2 : 2);
#pragma unroll UN
    for (int j = g; j < cnt; j += G) {
        const float4 p = srec[j * RS + 0];
        const float4 f = SL ? srec[j * RS + 1] : make_float4(0, 0, 0, 0);
        const float4 gg = DL ? srec[j * RS + 2] : make_float4(0, 0, 0, 0);
        const float4 n = DL ? srec[j * RS + 3] : make_float4(0, 0, 0, 0);
        float NG[6] = {0, 0, 0, 0, 0, 0};
        if (STRESS && DL) {
            const float4 t0 = srec[j * RS + 4];
            const float4 t1 = srec[j * RS + 5];
            NG[0] = t0.x; NG[1] = t0.y; NG[2] = t0.z; NG[3] = t0.w; NG[4] = t1.x; NG[5] = t1.y;
        }
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
            float dx = x[k] - p.x, dy = y[k] - p.y, dz = z[k] - p.z;
            float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            float ri = SAFE ? safe_rinv(r2) : rsqrtf(r2);
            if (!STRESS) {
                if (SL && DL) acc_UP(dx, dy, dz, ri, f.x, f.y, f.z, gg.x, gg.y, gg.z, n.x, n.y, n.z, p.w, kc.a1, kc.a3, acc[k]);
                else if (SL) acc_U(dx, dy, dz, ri, f.x, f.y, f.z, kc.a1, acc[k]);
                else acc_P(dx, dy, dz, ri, gg.x, gg.y, gg.z, n.x, n.y, n.z, p.w, kc.a3, acc[k]);
            } else {
                if (SL && DL) acc_DS(dx, dy, dz, ri, f.x, f.y, f.z, f.w, gg.x, gg.y, gg.z, n.x, n.y, n.z, p.w, NG, kc, acc[k]);
                else if (SL) acc_D(dx, dy, dz, ri, f.x, f.y, f.z, kc.a, acc[k]);
                else acc_S(dx, dy, dz, ri, gg.x, gg.y, gg.z, n.x, n.y, n.z, p.w, NG, kc.a, kc.nu, kc.b4, acc[k]);
            }
        }
    }
}

}  // namespace ebem
