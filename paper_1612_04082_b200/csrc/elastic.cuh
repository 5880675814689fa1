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
    T df = dx * fx + dy * fy + dz * fz;
    T s = df * ri2 * ri;
    T t = a1 * ri;
    u[0] += t * fx + s * dx;
    u[1] += t * fy + s * dy;
    u[2] += t * fz + s * dz;
}

// double layer: g = cP w g (prepared), q = a (n.g) (prepared):
// u_i += a rinv^3 [(d.n) g_i + (d.g) n_i] + [3 (d.n)(d.g) rinv^5 - q rinv^3] d_i
template <class T>
__device__ __forceinline__ void acc_P(T dx, T dy, T dz, T ri, T gx, T gy, T gz, T nx, T ny, T nz,
                                      T q, T a, T* u) {
    T ri2 = ri * ri;
    T ri3 = ri2 * ri;
    T dn = dx * nx + dy * ny + dz * nz;
    T dg = dx * gx + dy * gy + dz * gz;
    T ar3 = a * ri3;
    T A = dn * ar3;
    T B = dg * ar3;
    T C = (T(3) * dn * dg) * (ri3 * ri2) - q * ri3;
    u[0] += A * gx + B * nx + C * dx;
    u[1] += A * gy + B * ny + C * dy;
    u[2] += A * gz + B * nz + C * dz;
}

// stress of a single layer: f = cD w f (prepared, cD = -1/(8 pi (1-nu))):
// s_ij += a rinv^3 (f_i d_j + f_j d_i - d_ij (d.f)) + 3 rinv^5 (d.f) d_i d_j
template <class T>
__device__ __forceinline__ void acc_D(T dx, T dy, T dz, T ri, T fx, T fy, T fz, T a, T* s) {
    T ri2 = ri * ri;
    T ri3 = ri2 * ri;
    T df = dx * fx + dy * fy + dz * fz;
    T A = a * ri3;
    T B = T(3) * df * ri3 * ri2;
    T Ad = A * df;
    T bx = B * dx, by = B * dy, bz = B * dz;
    T ax = A * fx, ay = A * fy, az = A * fz;
    s[0] += T(2) * ax * dx - Ad + bx * dx;
    s[1] += T(2) * ay * dy - Ad + by * dy;
    s[2] += T(2) * az * dz - Ad + bz * dz;
    s[3] += ax * dy + ay * dx + bx * dy;
    s[4] += ay * dz + az * dy + by * dz;
    s[5] += ax * dz + az * dx + bx * dz;
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
    T ux = hCdd * dx + Cgd * gx + Cnd * nx;
    T uy = hCdd * dy + Cgd * gy + Cnd * ny;
    T uz = hCdd * dz + Cgd * gz + Cnd * nz;
    s[0] += T(2) * ux * dx + ri3 * NG[0] + Cdl;
    s[1] += T(2) * uy * dy + ri3 * NG[1] + Cdl;
    s[2] += T(2) * uz * dz + ri3 * NG[2] + Cdl;
    s[3] += ux * dy + uy * dx + ri3 * NG[3];
    s[4] += uy * dz + uz * dy + ri3 * NG[4];
    s[5] += ux * dz + uz * dx + ri3 * NG[5];
}

}  // namespace ebem
