// Pairwise accumulation of the four elastostatic kernels (Sec. 2.1).
//
//   U_ij  = ((3-4nu) d_ij + r_i r_j) / (16 pi (1-nu) G r)                        Eq. disp_1
//   P_ij  = [dr/dn ((1-2nu) d_ij + 3 r_i r_j) - (1-2nu)(r_i n_j - r_j n_i)] / (8 pi (1-nu) r^2)
//                                                                                Eq. disp_2
//   D_kij = -[(1-2nu)(d_ki r_j + d_kj r_i - d_ij r_k) + 3 r_i r_j r_k] / (8 pi (1-nu) r^2)
//                                                                Eq. stress_2, reading R2
//   S_kij = G/(4 pi (1-nu) r^3){3 dr/dn[(1-2nu) d_ij r_k + nu(d_ki r_j + d_kj r_i) - 5 r_i r_j r_k]
//           + 3nu(n_i r_j r_k + n_j r_i r_k) + (1-2nu)(3 n_k r_i r_j + n_j d_ki + n_i d_kj)
//           - (1-4nu) n_k d_ij}                                  Eq. stress_3, reading R3
//
// with r_i = d_i / r, d = target - source (reading R1).  Everything is written in the
// un-normalised d and powers of rinv = 1/r so that one rsqrt per pair suffices, and the
// per-source constants (panel weight w, kernel prefactor, n.g, the symmetric n (x) g
// tensor) are folded into a prepared source record once per source, not per pair.
//
// Outputs: displacement u[3]; stress s[6] in Voigt order (xx, yy, zz, xy, yz, xz).
#pragma once

namespace ebem {

template <class T>
__device__ __forceinline__ T rsqrt_t(T x);
template <>
__device__ __forceinline__ float rsqrt_t<float>(float x) { return rsqrtf(x); }
template <>
__device__ __forceinline__ double rsqrt_t<double>(double x) { return rsqrt(x); }

// fused multiply-add for both precisions (the accumulations below are written as FMA
// chains into the accumulator, so the compiler emits one FFMA per term)
__device__ __forceinline__ float fmat(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmat(double a, double b, double c) { return fma(a, b, c); }

// rinv with the self pair (r == 0) excluded: PAPER.md line 189, the own panel is
// handled by the local pass, never by the sum.
template <class T>
__device__ __forceinline__ T safe_rinv(T r2) {
    T ri = rsqrt_t<T>(r2);
    return r2 > T(0) ? ri : T(0);
}

// single layer: u_i += rinv (a1 f_i) + d_i (d.f) rinv^3,  f = cU w f (prepared)
template <class T>
__device__ __forceinline__ void acc_U(T dx, T dy, T dz, T ri, T fx, T fy, T fz, T a1, T* u) {
    T ri2 = ri * ri;
    T df = fmat(dz, fz, fmat(dy, fy, dx * fx));
    T s = df * ri2 * ri;
    T t = a1 * ri;
    u[0] = fmat(t, fx, fmat(s, dx, u[0]));
    u[1] = fmat(t, fy, fmat(s, dy, u[1]));
    u[2] = fmat(t, fz, fmat(s, dz, u[2]));
}

// double layer: g = cP w g, q = a (n.g), n3 = 3 n (all prepared per source):
// u_i += a rinv^3 [(d.n) g_i + (d.g) n_i] + rinv^3 [3 (d.n)(d.g) rinv^2 - q] d_i
// written with a3 = a/3 so every output update is one FFMA (FFMA-dense inner loop)
template <class T>
__device__ __forceinline__ void acc_P(T dx, T dy, T dz, T ri, T gx, T gy, T gz, T n3x, T n3y, T n3z,
                                      T q, T a3, T* u) {
    T ri2 = ri * ri;
    T ri3 = ri2 * ri;
    T dn3 = fmat(dz, n3z, fmat(dy, n3y, dx * n3x));   // 3 (d.n)
    T dg = fmat(dz, gz, fmat(dy, gy, dx * gx));
    T ar3 = a3 * ri3;
    T A = dn3 * ar3;                                  // a (d.n) rinv^3
    T B = dg * ar3;                                   // a (d.g) rinv^3 / 3   (multiplies n3)
    T C = ri3 * fmat(dn3 * dg, ri2, -q);
    u[0] = fmat(A, gx, fmat(B, n3x, fmat(C, dx, u[0])));
    u[1] = fmat(A, gy, fmat(B, n3y, fmat(C, dy, u[1])));
    u[2] = fmat(A, gz, fmat(B, n3z, fmat(C, dz, u[2])));
}

// both layers at once (U + P): the two d-terms share one coefficient, S = (d.f) rinv^3 + C,
// 37 FP32 instructions per pair with d and r^2 instead of 41 for acc_U + acc_P
template <class T>
__device__ __forceinline__ void acc_UP(T dx, T dy, T dz, T ri, T fx, T fy, T fz, T gx, T gy, T gz, T n3x, T n3y,
                                       T n3z, T q, T a1, T a3, T* u) {
    T ri2 = ri * ri;
    T ri3 = ri2 * ri;
    T df = fmat(dz, fz, fmat(dy, fy, dx * fx));
    T dn3 = fmat(dz, n3z, fmat(dy, n3y, dx * n3x));
    T dg = fmat(dz, gz, fmat(dy, gy, dx * gx));
    T ar3 = a3 * ri3;
    T A = dn3 * ar3;
    T B = dg * ar3;
    T S = fmat(df, ri3, ri3 * fmat(dn3 * dg, ri2, -q));
    T t = a1 * ri;
    u[0] = fmat(t, fx, fmat(A, gx, fmat(B, n3x, fmat(S, dx, u[0]))));
    u[1] = fmat(t, fy, fmat(A, gy, fmat(B, n3y, fmat(S, dy, u[1]))));
    u[2] = fmat(t, fz, fmat(A, gz, fmat(B, n3z, fmat(S, dz, u[2]))));
}

// stress of a single layer: f = cD w f (prepared, cD = -1/(8 pi (1-nu))):
// s_ij += a rinv^3 (f_i d_j + f_j d_i - d_ij (d.f)) + 3 rinv^5 (d.f) d_i d_j
template <class T>
__device__ __forceinline__ void acc_D(T dx, T dy, T dz, T ri, T fx, T fy, T fz, T a, T* s) {
    T ri2 = ri * ri;
    T ri3 = ri2 * ri;
    T df = fmat(dz, fz, fmat(dy, fy, dx * fx));
    T A = a * ri3;
    T B = T(3) * df * ri3 * ri2;
    T Ad = A * df;
    // v_i = A f_i + (B/2) d_i:  s_ij += v_i d_j + v_j d_i - Ad d_ij
    T hB = T(0.5) * B;
    T vx = fmat(hB, dx, A * fx), vy = fmat(hB, dy, A * fy), vz = fmat(hB, dz, A * fz);
    s[0] = fmat(T(2) * vx, dx, s[0] - Ad);
    s[1] = fmat(T(2) * vy, dy, s[1] - Ad);
    s[2] = fmat(T(2) * vz, dz, s[2] - Ad);
    s[3] = fmat(vx, dy, fmat(vy, dx, s[3]));
    s[4] = fmat(vy, dz, fmat(vz, dy, s[4]));
    s[5] = fmat(vx, dz, fmat(vz, dx, s[5]));
}

// stress of a double layer: g = cS w g, ng = n.g, NG = a (n (x) g + g (x) n) (prepared):
// s_ij += u_i d_j + u_j d_i + rinv^3 NG_ij + Cdelta d_ij with
//   u_i = (Cdd/2) d_i + Cgd g_i + Cnd n_i,  Cdd = rinv^5 (3 a ng - 15 (d.n)(d.g) rinv^2),
//   Cgd = 3 nu (d.n) rinv^5,  Cnd = 3 nu (d.g) rinv^5,
//   Cdelta = 3 a (d.n)(d.g) rinv^5 - (1 - 4 nu) ng rinv^3
template <class T>
__device__ __forceinline__ void acc_S(T dx, T dy, T dz, T ri, T gx, T gy, T gz, T nx, T ny, T nz,
                                      T ng, const T* NG, T a, T nu, T b4, T* s) {
    T ri2 = ri * ri;
    T ri3 = ri2 * ri;
    T ri5 = ri3 * ri2;
    T dn = dx * nx + dy * ny + dz * nz;
    T dg = dx * gx + dy * gy + dz * gz;
    T dndg = dn * dg;
    T hCdd = T(0.5) * ri5 * (T(3) * a * ng - T(15) * dndg * ri2);
    T Cgd = T(3) * nu * dn * ri5;
    T Cnd = T(3) * nu * dg * ri5;
    T Cdl = T(3) * a * dndg * ri5 - b4 * ng * ri3;
    T ux = fmat(Cnd, nx, fmat(Cgd, gx, hCdd * dx));
    T uy = fmat(Cnd, ny, fmat(Cgd, gy, hCdd * dy));
    T uz = fmat(Cnd, nz, fmat(Cgd, gz, hCdd * dz));
    s[0] = fmat(T(2) * ux, dx, fmat(ri3, NG[0], s[0] + Cdl));
    s[1] = fmat(T(2) * uy, dy, fmat(ri3, NG[1], s[1] + Cdl));
    s[2] = fmat(T(2) * uz, dz, fmat(ri3, NG[2], s[2] + Cdl));
    s[3] = fmat(ux, dy, fmat(uy, dx, fmat(ri3, NG[3], s[3])));
    s[4] = fmat(uy, dz, fmat(uz, dy, fmat(ri3, NG[4], s[4])));
    s[5] = fmat(ux, dz, fmat(uz, dx, fmat(ri3, NG[5], s[5])));
}

// both stress kernels at once (D + S), re-associated for the FP32 pipe (63 instead of ~71
// instructions per pair).  Per source the record carries (prepare_kernel, K_DS):
//   f' = a cD w f,  q1 = 1.5 a (n.g),  q2n = -0.5 (1 - 4 nu)(n.g),  g = cS w g,  n,
//   NGh = a (n_i g_i) on the diagonal (half of NG_ii), a (n_i g_j + n_j g_i) off it,
// and the DIAGONAL accumulators s[0..2] hold HALF the stress (the caller doubles them):
//   w   = (hCdd + hB) d + rinv^3 f' + 3 nu rinv^5 [(d.n) g + (d.g) n]
//   hCdd + hB = rinv^5 [q1 - 7.5 (d.n)(d.g) rinv^2 + (1.5 / a)(d.f')]
//   s_ii/2 += w_i d_i + rinv^3 NGh_ii + Cdelta / 2,  Cdelta / 2 = 1.5 a (d.n)(d.g) rinv^5
//             + rinv^3 (q2n - 0.5 d.f')
//   s_ij   += w_i d_j + w_j d_i + rinv^3 NG_ij
// which is D (v = A f + (B/2) d, diagonal -A (d.f), A = a rinv^3, B = 3 (d.f) rinv^5) plus
// S (acc_S above) term by term.
template <class T, class KC>
__device__ __forceinline__ void acc_DS(T dx, T dy, T dz, T ri, T fx, T fy, T fz, T q2n, T gx, T gy, T gz, T nx,
                                       T ny, T nz, T q1, const T* NG, const KC& kc, T* s) {
    T ri2 = ri * ri;
    T ri3 = ri2 * ri;
    T ri5 = ri3 * ri2;
    T df = fmat(dz, fz, fmat(dy, fy, dx * fx));          // d.f' = a d.f
    T dn = fmat(dz, nz, fmat(dy, ny, dx * nx));
    T dg = fmat(dz, gz, fmat(dy, gy, dx * gx));
    T dndg = dn * dg;
    T hd = ri5 * fmat(kc.ds_k2, df, fmat(T(-7.5), dndg * ri2, q1));
    T c3 = kc.ds_k4 * ri5;
    T Cgd = dn * c3, Cnd = dg * c3;
    T hCdl = fmat(kc.ds_k5, dndg * ri5, ri3 * fmat(T(-0.5), df, q2n));
    T wx = fmat(Cnd, nx, fmat(Cgd, gx, fmat(ri3, fx, hd * dx)));
    T wy = fmat(Cnd, ny, fmat(Cgd, gy, fmat(ri3, fy, hd * dy)));
    T wz = fmat(Cnd, nz, fmat(Cgd, gz, fmat(ri3, fz, hd * dz)));
    s[0] = fmat(wx, dx, fmat(ri3, NG[0], s[0] + hCdl));
    s[1] = fmat(wy, dy, fmat(ri3, NG[1], s[1] + hCdl));
    s[2] = fmat(wz, dz, fmat(ri3, NG[2], s[2] + hCdl));
    s[3] = fmat(wx, dy, fmat(wy, dx, fmat(ri3, NG[3], s[3])));
    s[4] = fmat(wy, dz, fmat(wz, dy, fmat(ri3, NG[4], s[4])));
    s[5] = fmat(wx, dz, fmat(wz, dx, fmat(ri3, NG[5], s[5])));
}

}  // namespace ebem
