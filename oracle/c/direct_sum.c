/* Oracle: O(N^2) fp64 direct sum of PAPER.md Eq. fmm_summation, plain C.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by oracle/cdirect.py for tests/, smoke() and the
 * cpu_baseline leg of bench.py.  Shares nothing with the CUDA product path.
 *
 * Same kernels and readings as oracle/kernels.py (R1: rh = (target - source)/r;
 * R2: D with -1/(8 pi (1-nu) r^2); R3: S carries G), written out term by term:
 *   U_ij  = ((3-4nu) d_ij + r_i r_j) / (16 pi (1-nu) G r)                    Eq. disp_1
 *   P_ij  = [dr/dn ((1-2nu) d_ij + 3 r_i r_j) - (1-2nu)(r_i n_j - r_j n_i)]
 *           / (8 pi (1-nu) r^2)                                                Eq. disp_2
 *   D_kij = -[(1-2nu)(d_ki r_j + d_kj r_i - d_ij r_k) + 3 r_i r_j r_k]
 *           / (8 pi (1-nu) r^2)                                                Eq. stress_2
 *   S_kij = G/(4 pi (1-nu) r^3) { 3 dr/dn [(1-2nu) d_ij r_k + nu (d_ki r_j + d_kj r_i)
 *           - 5 r_i r_j r_k] + 3 nu (n_i r_j r_k + n_j r_i r_k)
 *           + (1-2nu)(3 n_k r_i r_j + n_j d_ki + n_i d_kj) - (1-4nu) n_k d_ij }  Eq. stress_3
 * out_i = sum_j w_j [K(x_i, y_j) s_j] over pairs with r != 0; stress in Voigt order
 * (xx, yy, zz, xy, yz, xz).  Kernel ids: 0 U, 1 P, 2 U+P, 3 D, 4 S, 5 D+S.
 */
#include <math.h>

static inline double dlt(int a, int b) { return a == b ? 1.0 : 0.0; }

void oracle_direct_sum(int kernel, const double *trg, long ntrg, const double *src,
                       const double *nrm, const double *w, const double *f, const double *g,
                       long nsrc, double K, double G, double *out)
{
    const double PI = 3.14159265358979323846;
    const double nu = (3.0 * K - 2.0 * G) / (2.0 * (3.0 * K + G));
    const int sl = (kernel == 0 || kernel == 2 || kernel == 3 || kernel == 5);
    const int dl = (kernel == 1 || kernel == 2 || kernel == 4 || kernel == 5);
    const int stress = (kernel >= 3);
    static const int VI[6] = {0, 1, 2, 0, 1, 0}, VJ[6] = {0, 1, 2, 1, 2, 2};
#pragma omp parallel for schedule(dynamic, 16)
    for (long t = 0; t < ntrg; ++t) {
        double acc[9] = {0};
        for (long s = 0; s < nsrc; ++s) {
            double d[3], r2 = 0.0;
            for (int a = 0; a < 3; ++a) { d[a] = trg[3 * t + a] - src[3 * s + a]; r2 += d[a] * d[a]; }
            if (r2 == 0.0) continue;
            double r = sqrt(r2), rh[3] = {d[0] / r, d[1] / r, d[2] / r};
            double ws = w ? w[s] : 1.0;
            double fs[3] = {0, 0, 0}, gs[3] = {0, 0, 0}, n[3] = {0, 0, 0}, drdn = 0.0;
            for (int a = 0; a < 3; ++a) {
                if (sl) fs[a] = f[3 * s + a] * ws;
                if (dl) { gs[a] = g[3 * s + a] * ws; n[a] = nrm[3 * s + a]; drdn += rh[a] * n[a]; }
            }
            if (!stress) {
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) {
                        if (sl)
                            acc[i] += ((3.0 - 4.0 * nu) * dlt(i, j) + rh[i] * rh[j])
                                      / (16.0 * PI * (1.0 - nu) * G * r) * fs[j];
                        if (dl)
                            acc[i] += (drdn * ((1.0 - 2.0 * nu) * dlt(i, j) + 3.0 * rh[i] * rh[j])
                                       - (1.0 - 2.0 * nu) * (rh[i] * n[j] - rh[j] * n[i]))
                                      / (8.0 * PI * (1.0 - nu) * r2) * gs[j];
                    }
            } else {
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j)
                        for (int k = 0; k < 3; ++k) {
                            if (sl)
                                acc[3 * i + j] += -((1.0 - 2.0 * nu) * (dlt(k, i) * rh[j] + dlt(k, j) * rh[i]
                                                                        - dlt(i, j) * rh[k])
                                                    + 3.0 * rh[i] * rh[j] * rh[k])
                                                  / (8.0 * PI * (1.0 - nu) * r2) * fs[k];
                            if (dl)
                                acc[3 * i + j] += G / (4.0 * PI * (1.0 - nu) * r2 * r)
                                    * (3.0 * drdn * ((1.0 - 2.0 * nu) * dlt(i, j) * rh[k]
                                                     + nu * (dlt(k, i) * rh[j] + dlt(k, j) * rh[i])
                                                     - 5.0 * rh[i] * rh[j] * rh[k])
                                       + 3.0 * nu * (n[i] * rh[j] * rh[k] + n[j] * rh[i] * rh[k])
                                       + (1.0 - 2.0 * nu) * (3.0 * n[k] * rh[i] * rh[j] + n[j] * dlt(k, i)
                                                             + n[i] * dlt(k, j))
                                       - (1.0 - 4.0 * nu) * n[k] * dlt(i, j))
                                    * gs[k];
                        }
            }
        }
        if (!stress)
            for (int i = 0; i < 3; ++i) out[3 * t + i] = acc[i];
        else
            for (int v = 0; v < 6; ++v) out[6 * t + v] = acc[3 * VI[v] + VJ[v]];
    }
}
