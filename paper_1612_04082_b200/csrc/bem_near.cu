// BEM near-field operator held in HBM (bem_gmres_solve).
//
// In the collocation BEM (PAPER.md Eq. num2, l. 175; 16-point panel quadrature, l. 187) every
// target's near field is the sum of Eq. fmm_summation over the quadrature points of the
// panels in its near boxes, each point carrying the density of its panel: inside a GMRES
// solve the densities change every iteration, the geometry does not.  The near sum is
// therefore the same linear map every iteration,
//     near(t) = sum_{panels j near t} N(t, j) x_j,
//     N(t, j) = sum_{quadrature points q of j in t's near boxes} w_q K_j(t, y_q)   (3 x 3),
// with K_j = -U on Dirichlet panels (the unknown is the traction, entering as -U p) and P
// on Neumann panels (the unknown is the displacement).  Building N once per solve and
// applying it as a dense per-leaf GEMV turns the FP32-bound pair loop over ~16x more
// quadrature points than panels into one HBM read of N (9 floats per target-panel pair):
// the B200-first trade of its 180 GB of HBM3e for arithmetic.  Same sums, re-associated:
// N(t, j) collects exactly the pairs the near-field kernel evaluates (U list plus the
// directly summed X/W/V entries, r = 0 excluded).
//
// Layout: per target leaf i (eval order) the unique panels of its near sources, sorted, are
// its columns; N_i is stored [9][rows][ncol padded to 4] (component-major, so a warp reading
// 128 columns of one row and component is one 512-B run of 16-B loads).
//
// The same construction serves the two other sums over quadrature points whose geometry is
// fixed inside a solve (PanelOp::kind): the upward check potentials of the source leaves
// (S2M: the sources' field on the check surface of their own box) and the
// downward check potentials of the X-list entries (S2L).  Their rows are the n_c check
// points of a box (centre + 2.95 r or 1.05 r times the unit check surface, formed in fp64
// about the box centre), their columns the panels of the box's (or its X-list leaves')
// sources, and the apply writes the TF32 head / remainder split the tensor-core Q2Z reads.
// With all three held in HBM the FMM never touches the 16 quadrature points per panel
// during an iteration: the densities enter as one fp64 vector of panel values.
#include <chrono>
#include <cstdio>
#include <vector>

#include "bem_near.cuh"

namespace ebem {
namespace {

int bits_for(int64_t n) {
    int b = 1;
    while ((int64_t(1) << b) < n) ++b;
    return b;
}

// the source boxes of row set i: CSR indexed by the set (S2L: x_src_off) or by its box
// (near field: near_off is per box id); S2M: the set's own box
struct SetSrc {
    const int* box;
    const int* off;
    const int* idx;
    int by_box;      // 1: off indexed by box id; 2: the box itself is the only source box
    __device__ __forceinline__ int begin(int i) const {
        return by_box == 2 ? 0 : off[by_box ? box[i] : i];
    }
    __device__ __forceinline__ int end(int i) const {
        return by_box == 2 ? 1 : off[(by_box ? box[i] : i) + 1];
    }
    __device__ __forceinline__ int src_box(int i, int e) const { return by_box == 2 ? box[i] : idx[e]; }
};

// check rows are padded to a multiple of 4 (float4 loads of four rows in ck_apply)
__device__ __forceinline__ int set_rows(int kind, int b, const int* tbeg, const int* tend, int nc) {
    return kind == 0 ? tend[b] - tbeg[b] : (nc + 3) & ~3;
}

__global__ void nm_count(int nsets, SetSrc ss, int kind, int nc, const int* __restrict__ sbeg,
                         const int* __restrict__ send, const int* __restrict__ tbeg, const int* __restrict__ tend,
                         int* __restrict__ cnt, int* __restrict__ rows) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nsets) return;
    int c = 0;
    for (int e = ss.begin(i); e < ss.end(i); ++e) {
        const int a = ss.src_box(i, e);
        c += send[a] - sbeg[a];
    }
    cnt[i] = c;
    rows[i] = set_rows(kind, ss.box[i], tbeg, tend, nc);
}

// warp per row set: key = (set << pbits) | panel of the source, value = sorted source
__global__ void nm_fill(int nsets, SetSrc ss, const int* __restrict__ sbeg, const int* __restrict__ send,
                        const int* __restrict__ off, const int* __restrict__ src_perm, int nq, int pbits,
                        long long* __restrict__ keys, int* __restrict__ vals) {
    const int i = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (i >= nsets) return;
    int64_t pos = off[i];
    for (int e = ss.begin(i); e < ss.end(i); ++e) {
        const int a = ss.src_box(i, e);
        const int n = send[a] - sbeg[a];
        for (int j = lane; j < n; j += 32) {
            const int s = sbeg[a] + j;
            keys[pos + j] = ((long long)i << pbits) | (long long)(src_perm[s] / nq);
            vals[pos + j] = s;
        }
        pos += n;
    }
}

__global__ void nm_flags(const long long* __restrict__ keys, int64_t n, int* __restrict__ flag) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) flag[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
}

__global__ void nm_segs(const long long* __restrict__ keys, const int* __restrict__ flag, const int* __restrict__ ex,
                        int64_t n, long long pmask, int* __restrict__ seg_start, int* __restrict__ col_panel) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n || !flag[k]) return;
    seg_start[ex[k]] = (int)k;
    col_panel[ex[k]] = (int)(keys[k] & pmask);
}

// the first entry of a set always starts a segment (its key's set bits differ)
__global__ void nm_cols(int nsets, const int* __restrict__ off, const int* __restrict__ cnt,
                        const int* __restrict__ ex, int* __restrict__ col_first, int* __restrict__ ncol) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nsets) return;
    if (cnt[i] == 0) {
        col_first[i] = 0;
        ncol[i] = 0;
        return;
    }
    const int k0 = off[i], k1 = off[i] + cnt[i];
    col_first[i] = ex[k0];
    ncol[i] = ex[k1] - ex[k0];       // segment starts in [k0, k1)
}

struct RowGeo {   // check points: box centre + rad * r * unit check surface (fp64)
    double ox, oy, oz, side, rad;
    const int* anchor;
    const int* level;
    const float* sc;     // unit check surface [nc * 3]
};

// one CTA per row set; thread per (row, column) with the column fastest (coalesced stores).
// Entry (row, panel) = sum over the panel's quadrature points in the set's source boxes of
// w K(row point, y): -U on Dirichlet panels (the unknown traction enters as -U p), P on
// Neumann panels; r = 0 pairs excluded (R8; only target rows can coincide with sources).
template <int KIND>
__global__ void __launch_bounds__(256)
nm_assemble(int nsets, const int* __restrict__ set_box, const int* __restrict__ tbeg, const int* __restrict__ tend,
            int nc_rows, RowGeo rg, const int* __restrict__ col_first, const int* __restrict__ ncol,
            const long long* __restrict__ moff, const int* __restrict__ seg_start, const int* __restrict__ col_panel,
            const int* __restrict__ vals, const float* __restrict__ sxyz, const float* __restrict__ snrm,
            const float* __restrict__ sw, const float* __restrict__ txyz, const int32_t* __restrict__ bc, float cU,
            float cP, float a1, float a, float* __restrict__ M) {
    const int i = blockIdx.x;
    if (i >= nsets) return;
    const int b = set_box[i];
    const int rows = KIND == 0 ? tend[b] - tbeg[b] : (nc_rows + 3) & ~3, nc = ncol[i], ncp = (nc + 3) & ~3;
    if (nc == 0 || rows == 0) return;
    double cx = 0, cy = 0, cz = 0, R = 0;
    if (KIND == 1) {
        const double h = rg.side * __hiloint2double((1023 - rg.level[b]) << 20, 0);   // side 2^-level
        cx = rg.ox + (rg.anchor[3 * b] + 0.5) * h;
        cy = rg.oy + (rg.anchor[3 * b + 1] + 0.5) * h;
        cz = rg.oz + (rg.anchor[3 * b + 2] + 0.5) * h;
        R = rg.rad * 0.5 * h;
    }
    float* base = M + moff[i];
    const int64_t plane = (int64_t)rows * ncp;
    for (int64_t idx = threadIdx.x; idx < plane; idx += blockDim.x) {
        // near rows: [9][rows][ncp] (column fastest); check rows (hundreds of check points, a
        // few dozen panels): [9][ncp][rows] (row fastest, read a row per thread)
        const int r = KIND == 0 ? (int)(idx / ncp) : (int)(idx % rows);
        const int c = KIND == 0 ? (int)(idx - (int64_t)r * ncp) : (int)(idx / rows);
        if (c >= nc || (KIND == 1 && r >= nc_rows)) {   // padding columns (x staged as 0) / rows
#pragma unroll
            for (int q = 0; q < 9; ++q) base[q * plane + idx] = 0.f;
            continue;
        }
        const int sg = col_first[i] + c;
        const bool dir = bc[col_panel[sg]] == 0;
        double tx, ty, tz;
        if (KIND == 0) {
            const int t = tbeg[b] + r;
            tx = txyz[3 * t];
            ty = txyz[3 * t + 1];
            tz = txyz[3 * t + 2];
        } else {
            tx = cx + R * rg.sc[3 * r];
            ty = cy + R * rg.sc[3 * r + 1];
            tz = cz + R * rg.sc[3 * r + 2];
        }
        float A[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) A[q] = 0.f;
        for (int k = seg_start[sg]; k < seg_start[sg + 1]; ++k) {
            const int s = vals[k];
            // target - source: near rows subtract two fp32 points in fp32 (IEEE subtraction is
            // correctly rounded: bitwise the fp64 difference rounded to fp32); check rows (fp64
            // points, no cancellation far from the origin) in fp64; then fp32 kernel arithmetic
            float d[3];
            if (KIND == 0) {
                d[0] = (float)tx - sxyz[3 * s];
                d[1] = (float)ty - sxyz[3 * s + 1];
                d[2] = (float)tz - sxyz[3 * s + 2];
            } else {
                d[0] = (float)(tx - (double)sxyz[3 * s]);
                d[1] = (float)(ty - (double)sxyz[3 * s + 1]);
                d[2] = (float)(tz - (double)sxyz[3 * s + 2]);
            }
            const float r2 = fmaf(d[2], d[2], fmaf(d[1], d[1], d[0] * d[0]));
            if (r2 == 0.f) continue;                    // R8: r = 0 pairs excluded
            const float ri = rsqrtf(r2), ri2 = ri * ri, ri3 = ri2 * ri;
            if (dir) {   // -U: u_i += a1 / r f_i + d_i (d.f) / r^3 with f = -cU w p
                const float cw = -cU * sw[s];
#pragma unroll
                for (int p = 0; p < 3; ++p)
#pragma unroll
                    for (int q = 0; q < 3; ++q) A[3 * p + q] += cw * ((p == q ? a1 * ri : 0.f) + ri3 * d[p] * d[q]);
            } else {     // P: coefficient of g_j = cP w u_j in acc_P
                const float cw = cP * sw[s];
                const float n[3] = {snrm[3 * s], snrm[3 * s + 1], snrm[3 * s + 2]};
                const float dn = d[0] * n[0] + d[1] * n[1] + d[2] * n[2];
#pragma unroll
                for (int p = 0; p < 3; ++p)
#pragma unroll
                    for (int q = 0; q < 3; ++q)
                        A[3 * p + q] += cw * ((p == q ? a * dn * ri3 : 0.f) + a * ri3 * (n[p] * d[q] - d[p] * n[q]) +
                                              3.f * dn * ri3 * ri2 * d[p] * d[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) base[q * plane + idx] = A[q];
    }
}

// Near rows with the quadrature sources staged in shared memory: the columns are taken in
// tiles of NMA_CT panels whose sources (consecutive in the sorted list) are copied once into
// shared memory (structure of arrays) and read there by every (row, column) item of the tile;
// the entries are the same sums as nm_assemble<0> (the same operations in the same order).
// A tile whose sources exceed NMA_SMAX reads them from global memory.  Measured on configs[4]:
// 375 ms per build with every item gathering its sources from global memory.
constexpr int NMA_T = 256, NMA_CT = 64, NMA_SMAX = 2048;
__global__ void __launch_bounds__(NMA_T)
nm_assemble_near(int nsets, const int* __restrict__ set_box, const int* __restrict__ tbeg,
                 const int* __restrict__ tend, const int* __restrict__ col_first, const int* __restrict__ ncol,
                 const long long* __restrict__ moff, const int* __restrict__ seg_start,
                 const int* __restrict__ col_panel, const int* __restrict__ vals, const float* __restrict__ sxyz,
                 const float* __restrict__ snrm, const float* __restrict__ sw, const float* __restrict__ txyz,
                 const int32_t* __restrict__ bc, float cU, float cP, float a1, float a, float* __restrict__ M) {
    extern __shared__ float ssrc[];                  // [7][NMA_SMAX]: x, y, z, nx, ny, nz, w
    const int i = blockIdx.x;
    if (i >= nsets) return;
    const int b = set_box[i];
    const int rows = tend[b] - tbeg[b], nc = ncol[i], ncp = (nc + 3) & ~3;
    if (nc == 0 || rows == 0) return;
    const int cf = col_first[i];
    float* base = M + moff[i];
    const int64_t plane = (int64_t)rows * ncp;
    for (int c0 = 0; c0 < ncp; c0 += NMA_CT) {
        const int ce = min(ncp, c0 + NMA_CT), cr = min(nc, ce), w = ce - c0;
        const int k0 = c0 < nc ? seg_start[cf + c0] : 0, k1 = c0 < nc ? seg_start[cf + cr] : 0;
        const bool staged = k1 - k0 <= NMA_SMAX;
        __syncthreads();
        if (staged)
            for (int k = k0 + threadIdx.x; k < k1; k += NMA_T) {
                const int sidx = vals[k], o = k - k0;
                ssrc[o] = sxyz[3 * sidx];
                ssrc[NMA_SMAX + o] = sxyz[3 * sidx + 1];
                ssrc[2 * NMA_SMAX + o] = sxyz[3 * sidx + 2];
                ssrc[3 * NMA_SMAX + o] = snrm[3 * sidx];
                ssrc[4 * NMA_SMAX + o] = snrm[3 * sidx + 1];
                ssrc[5 * NMA_SMAX + o] = snrm[3 * sidx + 2];
                ssrc[6 * NMA_SMAX + o] = sw[sidx];
            }
        __syncthreads();
        for (int item = threadIdx.x; item < rows * w; item += NMA_T) {
            const int r = item / w, c = c0 + item % w;
            const int64_t idx = (int64_t)r * ncp + c;
            if (c >= nc) {                                  // padding columns (x staged as 0)
#pragma unroll
                for (int q = 0; q < 9; ++q) base[q * plane + idx] = 0.f;
                continue;
            }
            const int sg = cf + c;
            const bool dir = bc[col_panel[sg]] == 0;
            const int t = tbeg[b] + r;
            const float tx = txyz[3 * t], ty = txyz[3 * t + 1], tz = txyz[3 * t + 2];
            float A[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) A[q] = 0.f;
            for (int k = seg_start[sg]; k < seg_start[sg + 1]; ++k) {
                float px, py, pz, nx, ny, nz, wq;
                if (staged) {
                    const int o = k - k0;
                    px = ssrc[o];
                    py = ssrc[NMA_SMAX + o];
                    pz = ssrc[2 * NMA_SMAX + o];
                    nx = ssrc[3 * NMA_SMAX + o];
                    ny = ssrc[4 * NMA_SMAX + o];
                    nz = ssrc[5 * NMA_SMAX + o];
                    wq = ssrc[6 * NMA_SMAX + o];
                } else {
                    const int sidx = vals[k];
                    px = sxyz[3 * sidx];
                    py = sxyz[3 * sidx + 1];
                    pz = sxyz[3 * sidx + 2];
                    nx = snrm[3 * sidx];
                    ny = snrm[3 * sidx + 1];
                    nz = snrm[3 * sidx + 2];
                    wq = sw[sidx];
                }
                // fp32 difference of two fp32 points (correctly rounded, as nm_assemble<0>)
                const float d[3] = {tx - px, ty - py, tz - pz};
                const float r2 = fmaf(d[2], d[2], fmaf(d[1], d[1], d[0] * d[0]));
                if (r2 == 0.f) continue;                    // R8: r = 0 pairs excluded
                const float ri = rsqrtf(r2), ri2 = ri * ri, ri3 = ri2 * ri;
                if (dir) {
                    const float cw = -cU * wq;
#pragma unroll
                    for (int p = 0; p < 3; ++p)
#pragma unroll
                        for (int q = 0; q < 3; ++q) A[3 * p + q] += cw * ((p == q ? a1 * ri : 0.f) + ri3 * d[p] * d[q]);
                } else {
                    const float cw = cP * wq;
                    const float n[3] = {nx, ny, nz};
                    const float dn = d[0] * n[0] + d[1] * n[1] + d[2] * n[2];
#pragma unroll
                    for (int p = 0; p < 3; ++p)
#pragma unroll
                        for (int q = 0; q < 3; ++q)
                            A[3 * p + q] += cw * ((p == q ? a * dn * ri3 : 0.f) + a * ri3 * (n[p] * d[q] - d[p] * n[q]) +
                                                  3.f * dn * ri3 * ri2 * d[p] * d[q]);
                }
            }
#pragma unroll
            for (int q = 0; q < 9; ++q) base[q * plane + idx] = A[q];
        }
    }
}

constexpr int NM_T = 256, NM_CH = 1024;

__device__ __forceinline__ float tf32_rna_nm(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// check rows: one CTA per row set, a thread per four consecutive check points (16-B loads
// of the [9][ncp][rows padded to 4] layout, contiguous across threads), the set's panel
// densities staged in shared memory, fp64 accumulation, the TF32 split written to Qb / Qs
// CK_G row groups of 4 x CK_T check points per thread, instantiated for the surface at hand
// (p = 8: 386 points, one group: 102 -> ~70 registers and more CTAs in flight)
constexpr int CK_T = 128, CK_CH = 512, CK_GMAX = 2;   // up to CK_GMAX x 4 x CK_T = 1024 check points
template <int CK_G, int UNR>
__global__ void __launch_bounds__(CK_T)
ck_apply(int nsets, int rows, const int* __restrict__ col_first, const int* __restrict__ ncol,
         const long long* __restrict__ moff, const int* __restrict__ col_panel, const float* __restrict__ M,
         const double* __restrict__ x, float* __restrict__ Qb, float* __restrict__ Qs, int ldq) {
    __shared__ double xs[CK_CH][3];
    const int i = blockIdx.x;
    if (i >= nsets) return;
    const int nc = ncol[i], ncp = (nc + 3) & ~3, r4 = (rows + 3) & ~3;
    const float* base = M + moff[i];
    const int64_t plane = (int64_t)r4 * ncp;
    double acc[CK_G][4][3];
#pragma unroll
    for (int h = 0; h < CK_G; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[h][k][0] = acc[h][k][1] = acc[h][k][2] = 0.0;
    for (int c0 = 0; c0 < nc; c0 += CK_CH) {          // uniform over the CTA (barriers inside)
        const int cnt = min(CK_CH, nc - c0);
        __syncthreads();
        for (int c = threadIdx.x; c < cnt; c += CK_T) {
            const int p = col_panel[col_first[i] + c0 + c];
            xs[c][0] = x[3 * p];
            xs[c][1] = x[3 * p + 1];
            xs[c][2] = x[3 * p + 2];
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < CK_G; ++h) {
            const int g = threadIdx.x + h * CK_T;          // rows 4g .. 4g+3
            if (4 * g >= r4) continue;
#pragma unroll UNR
            for (int c = 0; c < cnt; ++c) {
                const double xv[3] = {xs[c][0], xs[c][1], xs[c][2]};
                const float* mc = base + (int64_t)(c0 + c) * r4 + 4 * g;
                float4 v[9];
#pragma unroll
                for (int q = 0; q < 9; ++q) v[q] = __ldcs(reinterpret_cast<const float4*>(mc + q * plane));
#pragma unroll
                for (int p = 0; p < 3; ++p)
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const float4 a = v[3 * p + q];
                        acc[h][0][p] = fma((double)a.x, xv[q], acc[h][0][p]);
                        acc[h][1][p] = fma((double)a.y, xv[q], acc[h][1][p]);
                        acc[h][2][p] = fma((double)a.z, xv[q], acc[h][2][p]);
                        acc[h][3][p] = fma((double)a.w, xv[q], acc[h][3][p]);
                    }
            }
        }
    }
#pragma unroll
    for (int h = 0; h < CK_G; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int r = 4 * (threadIdx.x + h * CK_T) + k;
            if (r < rows)
#pragma unroll
                for (int p = 0; p < 3; ++p) {
                    const float hd = tf32_rna_nm((float)acc[h][k][p]);
                    Qb[(int64_t)i * ldq + 3 * r + p] = hd;
                    Qs[(int64_t)i * ldq + 3 * r + p] = tf32_rna_nm((float)(acc[h][k][p] - (double)hd));
                }
        }
    (void)ncp;
}

// out = N_i x_gathered: one CTA per row set, the set's panel densities staged in shared
// memory NM_CH columns at a time, a warp per row, each lane 4 columns per step (rows padded
// to a multiple of 4 columns: nine 16-B streaming loads per lane).  fp64 densities and fp64
// accumulation of the fp32 operator entries (HBM-bound: the FP64 pipe has room).
// KIND 0: near field rows, written as fp64 to near[sorted target];  KIND 1: check potential
// rows, written as the TF32 head / remainder split to Qb / Qs row i (ld ldq).
template <int KIND>
__global__ void __launch_bounds__(NM_T)
nm_apply(int nsets, const int* __restrict__ set_box, const int* __restrict__ tbeg, const int* __restrict__ tend,
         int nc_rows, const int* __restrict__ col_first, const int* __restrict__ ncol,
         const long long* __restrict__ moff, const int* __restrict__ col_panel, const float* __restrict__ M,
         const double* __restrict__ x, double* __restrict__ near, float* __restrict__ Qb, float* __restrict__ Qs,
         int ldq) {
    __shared__ __align__(16) double xs[3][NM_CH];
    const int i = blockIdx.x;
    if (i >= nsets) return;
    const int b = set_box[i];
    const int rows = KIND == 0 ? tend[b] - tbeg[b] : nc_rows, nc = ncol[i], ncp = (nc + 3) & ~3;
    const int t0 = KIND == 0 ? tbeg[b] : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (nc == 0) {
        for (int q = threadIdx.x; q < 3 * rows; q += NM_T) {
            if (KIND == 0) near[3 * (int64_t)t0 + q] = 0.0;
            else Qb[(int64_t)i * ldq + q] = Qs[(int64_t)i * ldq + q] = 0.f;
        }
        return;
    }
    const float* base = M + moff[i];
    const int64_t plane = (int64_t)rows * ncp;
    double part[3];          // KIND 1, more than one chunk: running row sums are kept in registers
    for (int c0 = 0; c0 < ncp; c0 += NM_CH) {
        const int cnt = min(NM_CH, ncp - c0);
        __syncthreads();
        for (int c = threadIdx.x; c < cnt; c += NM_T) {
            const bool in = c0 + c < nc;
            const int p = in ? col_panel[col_first[i] + c0 + c] : 0;
            xs[0][c] = in ? x[3 * p] : 0.0;
            xs[1][c] = in ? x[3 * p + 1] : 0.0;
            xs[2][c] = in ? x[3 * p + 2] : 0.0;
        }
        __syncthreads();
        for (int r = warp; r < rows; r += NM_T / 32) {
            const float* m = base + (int64_t)r * ncp + c0;
            double acc[3] = {0.0, 0.0, 0.0};
            for (int c = 4 * lane; c < cnt; c += 128) {
                const double* x0 = &xs[0][c];
                const double* x1 = &xs[1][c];
                const double* x2 = &xs[2][c];
                float4 v[9];
#pragma unroll
                for (int q = 0; q < 9; ++q) v[q] = __ldcs(reinterpret_cast<const float4*>(m + q * plane + c));
#pragma unroll
                for (int p = 0; p < 3; ++p) {
                    const float4 a = v[3 * p], bq = v[3 * p + 1], cq = v[3 * p + 2];
                    acc[p] = fma((double)a.x, x0[0], fma((double)a.y, x0[1], fma((double)a.z, x0[2], fma((double)a.w, x0[3], acc[p]))));
                    acc[p] = fma((double)bq.x, x1[0], fma((double)bq.y, x1[1], fma((double)bq.z, x1[2], fma((double)bq.w, x1[3], acc[p]))));
                    acc[p] = fma((double)cq.x, x2[0], fma((double)cq.y, x2[1], fma((double)cq.z, x2[2], fma((double)cq.w, x2[3], acc[p]))));
                }
            }
#pragma unroll
            for (int p = 0; p < 3; ++p)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[p] += __shfl_xor_sync(0xffffffffu, acc[p], o);
            if (lane == 0) {
                if (KIND == 0) {
                    double* o = near + 3 * (int64_t)(t0 + r);
                    for (int p = 0; p < 3; ++p) o[p] = c0 == 0 ? acc[p] : o[p] + acc[p];
                } else {
                    // check rows: the partial of earlier chunks is re-read from the split (exact
                    // for a single chunk, the usual case; rows of many panels add in fp32)
                    float* hb = Qb + (int64_t)i * ldq + 3 * r;
                    float* hs = Qs + (int64_t)i * ldq + 3 * r;
                    for (int p = 0; p < 3; ++p) {
                        const double v = c0 == 0 ? acc[p] : acc[p] + (double)hb[p] + (double)hs[p];
                        const float h = tf32_rna_nm((float)v);
                        hb[p] = h;
                        hs[p] = tf32_rna_nm((float)(v - (double)h));
                    }
                }
            }
        }
    }
    (void)part;
}

__global__ void nm_diff(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n, int* __restrict__ flag) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n && a[k] != b[k]) *flag = 1;
}

__global__ void iota_i(int* __restrict__ a, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

// the row sets of each operator kind on the BEM tree
struct SetDesc {
    int nsets = 0;
    const int* box = nullptr;
    SetSrc src{};
    int kind = 0;       // 0 target rows, 1 check rows
    double rad = 0;
};

SetDesc describe(const Tree& t, PanelOp::Kind k) {
    SetDesc d;
    if (k == PanelOp::NEAR) {
        d.nsets = t.n_eval;
        d.box = t.eval_box.p;
        d.src = SetSrc{t.eval_box.p, t.near_off.p, t.near_idx.p, 1};
    } else if (k == PanelOp::S2M) {
        d.nsets = t.n_s2m;
        d.box = t.s2m_box.p;
        d.src = SetSrc{t.s2m_box.p, nullptr, nullptr, 2};
        d.kind = 1;
        d.rad = RAD_UC;
    } else {
        d.nsets = t.n_s2l;
        d.box = t.s2l_box.p;
        d.src = SetSrc{t.s2l_box.p, t.x_src_off.p, t.x_src_idx.p, 0};
        d.kind = 1;
        d.rad = RAD_DC;
    }
    return d;
}

}  // namespace

bool near_matrix_enabled() {   // read per solve (tests switch it)
    const char* e = std::getenv("EBEM_BEM_NEARMAT");
    return !(e && std::atoi(e) == 0);
}

bool check_matrix_enabled() {   // S2M / S2L operators held in HBM inside GMRES
    const char* e = std::getenv("EBEM_BEM_CHECKMAT");
    return !(e && std::atoi(e) == 0);
}

bool panel_op_build(const Tree& t, PanelOp::Kind kind, int nq, int64_t npanels, const int32_t* bc,
                    const Material& m, PanelOp& N, cudaStream_t s) {
    // reuse when the boundary-condition types are unchanged
    if (N.ready) {
        DBuf<int> flag(1);
        flag.zero(s);
        nm_diff<<<ceil_div(npanels, 256), 256, 0, s>>>(bc, N.bc.p, npanels, flag.p);
        EB_CHECK_LAUNCH();
        int h = 0;
        d2h(&h, flag.p, 1, s);
        EB_CUDA(cudaStreamSynchronize(s));
        if (!h) return true;
    }
    N.release();
    N.kind = kind;
    const auto t_start = std::chrono::steady_clock::now();
    static const bool timing = std::getenv("EBEM_BUILD_TIMING") != nullptr;
    auto tick = t_start;
    auto lap = [&](const char* what) {
        if (!timing) return;
        EB_CUDA(cudaStreamSynchronize(s));
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[panel operator]   %-12s %.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tick).count());
        tick = now;
    };
    const SetDesc sd = describe(t, kind);
    const int ne = sd.nsets;
    if (ne == 0) return false;
    const Plan& P = *t.plan;
    DBuf<int> cnt(ne + 1), rows(ne), off(ne + 1);
    nm_count<<<ceil_div(ne, 256), 256, 0, s>>>(ne, sd.src, sd.kind, P.nc, t.sbeg.p, t.send.p, t.tbeg.p, t.tend.p,
                                              cnt.p, rows.p);
    EB_CHECK_LAUNCH();
    EB_CUDA(cudaMemsetAsync(cnt.p + ne, 0, sizeof(int), s));
    // entry count must fit the int32 scans and the radix sort
    {
        std::vector<int> hc(ne);
        d2h(hc.data(), cnt.p, ne, s);
        EB_CUDA(cudaStreamSynchronize(s));
        int64_t tot = 0;
        for (int v : hc) tot += v;
        if (tot >= (int64_t(1) << 31) - 1) return false;
    }
    const int64_t nent = exclusive_scan_i32(cnt.p, off.p, ne + 1, s);
    lap("count/scan");
    const int pbits = bits_for(std::max<int64_t>(npanels, 2)), lbits = bits_for(std::max(ne, 2));
    if (pbits + lbits > 62) return false;
    DBuf<long long> keys(std::max<int64_t>(nent, 1));
    N.vals.alloc(std::max<int64_t>(nent, 1));
    nm_fill<<<ceil_div((int64_t)ne * 32, 256), 256, 0, s>>>(ne, sd.src, t.sbeg.p, t.send.p, off.p, t.src_perm.p, nq,
                                                           pbits, keys.p, N.vals.p);
    EB_CHECK_LAUNCH();
    lap("fill");
    radix_sort_pairs(keys.p, N.vals.p, nent, pbits + lbits, s);
    lap("sort");
    DBuf<int> flag(nent + 1), ex(nent + 1);
    nm_flags<<<ceil_div(nent, 256), 256, 0, s>>>(keys.p, nent, flag.p);
    EB_CHECK_LAUNCH();
    EB_CUDA(cudaMemsetAsync(flag.p + nent, 0, sizeof(int), s));
    const int64_t nseg = exclusive_scan_i32(flag.p, ex.p, nent + 1, s);
    N.seg_start.alloc(nseg + 1);
    N.col_panel.alloc(std::max<int64_t>(nseg, 1));
    nm_segs<<<ceil_div(nent, 256), 256, 0, s>>>(keys.p, flag.p, ex.p, nent, (1LL << pbits) - 1, N.seg_start.p,
                                               N.col_panel.p);
    EB_CHECK_LAUNCH();
    {
        const int v = (int)nent;
        h2d(N.seg_start.p + nseg, &v, 1, s);
    }
    N.col_first.alloc(ne);
    N.ncol.alloc(ne);
    nm_cols<<<ceil_div(ne, 256), 256, 0, s>>>(ne, off.p, cnt.p, ex.p, N.col_first.p, N.ncol.p);
    EB_CHECK_LAUNCH();
    lap("segments");
    // per-set matrix offsets (int64, host scan of ne values) and the memory check
    std::vector<int> hr(ne), hn(ne);
    d2h(hr.data(), rows.p, ne, s);
    d2h(hn.data(), N.ncol.p, ne, s);
    EB_CUDA(cudaStreamSynchronize(s));
    std::vector<long long> mo(ne);
    long long tot = 0;
    for (int i = 0; i < ne; ++i) {
        mo[i] = tot;
        tot += 9LL * hr[i] * ((hn[i] + 3) & ~3);   // rows padded to 4 columns (16-B aligned)
    }
    size_t fr = 0, tt = 0;
    cache_trim();                              // cached blocks count as free memory here
    EB_CUDA(cudaMemGetInfo(&fr, &tt));
    const double frac = std::getenv("EBEM_BEM_NEARMAT_FRAC") ? std::atof(std::getenv("EBEM_BEM_NEARMAT_FRAC")) : 0.6;
    if ((double)tot * 4.0 > frac * (double)fr) {
        N.release();
        return false;
    }
    lap("offsets/mem");
    N.moff.alloc(ne);
    h2d(N.moff.p, mo.data(), ne, s);
    N.M.alloc(std::max<long long>(tot, 1));
    lap("alloc");
    const RowGeo rg{t.origin[0], t.origin[1], t.origin[2], t.side, sd.rad, t.anchor.p, t.level.p, P.s_c.p};
    auto asm_args = [&](auto fn) {
        fn<<<ne, 256, 0, s>>>(ne, sd.box, t.tbeg.p, t.tend.p, P.nc, rg, N.col_first.p, N.ncol.p, N.moff.p,
                              N.seg_start.p, N.col_panel.p, N.vals.p, t.src_xyz.p, t.src_nrm.p, t.src_w.p, t.trg_xyz.p,
                              bc, (float)m.cU, (float)m.cP, (float)m.a1, (float)m.a, N.M.p);
    };
    if (sd.kind == 0) {
        const size_t sm = sizeof(float) * 7 * NMA_SMAX;
        static bool attr = false;
        if (!attr) {
            EB_CUDA(cudaFuncSetAttribute(nm_assemble_near, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            attr = true;
        }
        nm_assemble_near<<<ne, NMA_T, sm, s>>>(ne, sd.box, t.tbeg.p, t.tend.p, N.col_first.p, N.ncol.p, N.moff.p,
                                               N.seg_start.p, N.col_panel.p, N.vals.p, t.src_xyz.p, t.src_nrm.p,
                                               t.src_w.p, t.trg_xyz.p, bc, (float)m.cU, (float)m.cP, (float)m.a1,
                                               (float)m.a, N.M.p);
    } else {
        asm_args(nm_assemble<1>);
    }
    EB_CHECK_LAUNCH();
    lap("assemble");
    N.vals.release();             // only the build needs the sorted sources
    N.bc.alloc(npanels);
    EB_CUDA(cudaMemcpyAsync(N.bc.p, bc, sizeof(int32_t) * npanels, cudaMemcpyDeviceToDevice, s));
    N.entries = tot;
    N.ready = true;
    EB_CUDA(cudaStreamSynchronize(s));
    if (std::getenv("EBEM_BUILD_TIMING"))
        std::fprintf(stderr, "[panel operator %s] %d sets, %lld quadrature entries, %lld columns, %.2f GB, %.1f ms\n",
                     kind == PanelOp::NEAR ? "near" : kind == PanelOp::S2M ? "S2M" : "S2L", ne, (long long)nent,
                     (long long)nseg, tot * 4.0 / 1e9,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
    return true;
}

void panel_op_apply(const Tree& t, const PanelOp& N, const double* x, double* near, float* Qb, float* Qs, int ldq,
                    cudaStream_t s) {
    const SetDesc sd = describe(t, N.kind);
    if (sd.nsets == 0) return;
    const Plan& P = *t.plan;
    if (sd.kind == 0) {
        static const int pad = beside_translation_pad((const void*)nm_apply<0>);
        nm_apply<0><<<sd.nsets, NM_T, pad, s>>>(sd.nsets, sd.box, t.tbeg.p, t.tend.p, P.nc, N.col_first.p, N.ncol.p,
                                               N.moff.p, N.col_panel.p, N.M.p, x, near, nullptr, nullptr, 0);
    } else {
        EB_REQUIRE(P.nc <= 4 * CK_GMAX * CK_T, "check surface too large for ck_apply");
        static const int unr = std::getenv("EBEM_CK_UNROLL") ? std::atoi(std::getenv("EBEM_CK_UNROLL")) : 4;
        auto go = [&](auto fn) {
            fn<<<sd.nsets, CK_T, 0, s>>>(sd.nsets, P.nc, N.col_first.p, N.ncol.p, N.moff.p, N.col_panel.p, N.M.p, x, Qb,
                                         Qs, ldq);
        };
        if (P.nc <= 4 * CK_T) {
            if (unr == 2) go(ck_apply<1, 2>);
            else go(ck_apply<1, 4>);
        } else {
            go(ck_apply<2, 2>);
        }
    }
    EB_CHECK_LAUNCH();
}

bool near_matrix_build(const Tree& t, int nq, int64_t npanels, const int32_t* bc, const Material& m, NearMat& N,
                       cudaStream_t s) {
    return panel_op_build(t, PanelOp::NEAR, nq, npanels, bc, m, N, s);
}

void near_matrix_apply(const Tree& t, const NearMat& N, const double* x, double* near, cudaStream_t s) {
    panel_op_apply(t, N, x, near, nullptr, nullptr, 0, s);
}

}  // namespace ebem
