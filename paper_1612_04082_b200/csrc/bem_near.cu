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

__global__ void nm_count(int n_eval, const int* __restrict__ eval_box, const int* __restrict__ noff,
                         const int* __restrict__ nidx, const int* __restrict__ sbeg, const int* __restrict__ send,
                         const int* __restrict__ tbeg, const int* __restrict__ tend, int* __restrict__ cnt,
                         int* __restrict__ rows) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_eval) return;
    const int b = eval_box[i];
    int c = 0;
    for (int e = noff[b]; e < noff[b + 1]; ++e) {
        const int a = nidx[e];
        c += send[a] - sbeg[a];
    }
    cnt[i] = c;
    rows[i] = tend[b] - tbeg[b];
}

// warp per target leaf: key = (leaf << pbits) | panel of the source, value = sorted source
__global__ void nm_fill(int n_eval, const int* __restrict__ eval_box, const int* __restrict__ noff,
                        const int* __restrict__ nidx, const int* __restrict__ sbeg, const int* __restrict__ send,
                        const int* __restrict__ off, const int* __restrict__ src_perm, int nq, int pbits,
                        long long* __restrict__ keys, int* __restrict__ vals) {
    const int i = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (i >= n_eval) return;
    const int b = eval_box[i];
    int64_t pos = off[i];
    for (int e = noff[b]; e < noff[b + 1]; ++e) {
        const int a = nidx[e];
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

// the first entry of a leaf always starts a segment (its key's leaf bits differ)
__global__ void nm_cols(int n_eval, const int* __restrict__ off, const int* __restrict__ cnt,
                        const int* __restrict__ ex, int* __restrict__ col_first, int* __restrict__ ncol) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_eval) return;
    if (cnt[i] == 0) {
        col_first[i] = 0;
        ncol[i] = 0;
        return;
    }
    const int k0 = off[i], k1 = off[i] + cnt[i];
    col_first[i] = ex[k0];
    ncol[i] = ex[k1] - ex[k0];       // segment starts in [k0, k1)
}

// one CTA per target leaf; thread per (row, column) with the column fastest (coalesced stores)
__global__ void __launch_bounds__(256)
nm_assemble(int n_eval, const int* __restrict__ eval_box, const int* __restrict__ tbeg, const int* __restrict__ tend,
            const int* __restrict__ col_first, const int* __restrict__ ncol, const long long* __restrict__ moff,
            const int* __restrict__ seg_start, const int* __restrict__ col_panel, const int* __restrict__ vals,
            const float* __restrict__ sxyz, const float* __restrict__ snrm, const float* __restrict__ sw,
            const float* __restrict__ txyz, const int32_t* __restrict__ bc, float cU, float cP, float a1, float a,
            float* __restrict__ M) {
    const int i = blockIdx.x;
    if (i >= n_eval) return;
    const int b = eval_box[i];
    const int rows = tend[b] - tbeg[b], nc = ncol[i], ncp = (nc + 3) & ~3;
    if (nc == 0 || rows == 0) return;
    float* base = M + moff[i];
    const int64_t plane = (int64_t)rows * ncp;
    for (int64_t idx = threadIdx.x; idx < plane; idx += blockDim.x) {
        const int r = (int)(idx / ncp), c = (int)(idx - (int64_t)r * ncp);
        if (c >= nc) {                                  // padding columns (x is staged as 0 there)
#pragma unroll
            for (int q = 0; q < 9; ++q) base[q * plane + idx] = 0.f;
            continue;
        }
        const int sg = col_first[i] + c;
        const bool dir = bc[col_panel[sg]] == 0;
        const int t = tbeg[b] + r;
        const float tx = txyz[3 * t], ty = txyz[3 * t + 1], tz = txyz[3 * t + 2];
        float A[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) A[q] = 0.f;
        for (int k = seg_start[sg]; k < seg_start[sg + 1]; ++k) {
            const int s = vals[k];
            const float d[3] = {tx - sxyz[3 * s], ty - sxyz[3 * s + 1], tz - sxyz[3 * s + 2]};
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

constexpr int NM_T = 256, NM_CH = 1024;

// near(t) = N_i x_gathered: one CTA per target leaf, the leaf's panel densities staged in
// shared memory NM_CH columns at a time, a warp per target row, each lane 4 columns per
// step (rows padded to a multiple of 4 columns: nine 16-B streaming loads per lane)
__global__ void __launch_bounds__(NM_T)
nm_apply(int n_eval, const int* __restrict__ eval_box, const int* __restrict__ tbeg, const int* __restrict__ tend,
         const int* __restrict__ col_first, const int* __restrict__ ncol, const long long* __restrict__ moff,
         const int* __restrict__ col_panel, const float* __restrict__ M, const double* __restrict__ x,
         double* __restrict__ near) {
    // fp64 densities and fp64 accumulation of the fp32 operator entries: the near field is
    // then linear in x to fp64 rounding (the kernel is HBM-bound, the FP64 pipe has room)
    __shared__ __align__(16) double xs[3][NM_CH];
    const int i = blockIdx.x;
    if (i >= n_eval) return;
    const int b = eval_box[i];
    const int rows = tend[b] - tbeg[b], nc = ncol[i], ncp = (nc + 3) & ~3, t0 = tbeg[b];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (nc == 0) {
        for (int q = threadIdx.x; q < 3 * rows; q += NM_T) near[3 * (int64_t)t0 + q] = 0.0;
        return;
    }
    const float* base = M + moff[i];
    const int64_t plane = (int64_t)rows * ncp;
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
                double* o = near + 3 * (int64_t)(t0 + r);
                for (int p = 0; p < 3; ++p) o[p] = c0 == 0 ? acc[p] : o[p] + acc[p];
            }
        }
    }
}

__global__ void nm_diff(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n, int* __restrict__ flag) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n && a[k] != b[k]) *flag = 1;
}

}  // namespace

bool near_matrix_enabled() {   // read per solve (tests switch it)
    const char* e = std::getenv("EBEM_BEM_NEARMAT");
    return !(e && std::atoi(e) == 0);
}

bool near_matrix_build(const Tree& t, int nq, int64_t npanels, const int32_t* bc, const Material& m, NearMat& N,
                       cudaStream_t s) {
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
    const int ne = t.n_eval;
    if (ne == 0) return false;
    DBuf<int> cnt(ne + 1), rows(ne), off(ne + 1);
    nm_count<<<ceil_div(ne, 256), 256, 0, s>>>(ne, t.eval_box.p, t.near_off.p, t.near_idx.p, t.sbeg.p, t.send.p,
                                              t.tbeg.p, t.tend.p, cnt.p, rows.p);
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
    const int pbits = bits_for(std::max<int64_t>(npanels, 2)), lbits = bits_for(std::max(ne, 2));
    if (pbits + lbits > 62) return false;
    DBuf<long long> keys(std::max<int64_t>(nent, 1));
    DBuf<int> vals(std::max<int64_t>(nent, 1));
    nm_fill<<<ceil_div((int64_t)ne * 32, 256), 256, 0, s>>>(ne, t.eval_box.p, t.near_off.p, t.near_idx.p, t.sbeg.p,
                                                           t.send.p, off.p, t.src_perm.p, nq, pbits, keys.p, vals.p);
    EB_CHECK_LAUNCH();
    radix_sort_pairs(keys.p, vals.p, nent, pbits + lbits, s);
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
    // per-leaf matrix offsets (int64, host scan of ne values) and the memory check
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
    EB_CUDA(cudaMemGetInfo(&fr, &tt));
    const double frac = std::getenv("EBEM_BEM_NEARMAT_FRAC") ? std::atof(std::getenv("EBEM_BEM_NEARMAT_FRAC")) : 0.6;
    if ((double)tot * 4.0 > frac * (double)fr) {
        N.release();
        return false;
    }
    N.moff.alloc(ne);
    h2d(N.moff.p, mo.data(), ne, s);
    N.M.alloc(std::max<long long>(tot, 1));
    nm_assemble<<<ne, 256, 0, s>>>(ne, t.eval_box.p, t.tbeg.p, t.tend.p, N.col_first.p, N.ncol.p, N.moff.p,
                                   N.seg_start.p, N.col_panel.p, vals.p, t.src_xyz.p, t.src_nrm.p, t.src_w.p,
                                   t.trg_xyz.p, bc, (float)m.cU, (float)m.cP, (float)m.a1, (float)m.a, N.M.p);
    EB_CHECK_LAUNCH();
    N.bc.alloc(npanels);
    EB_CUDA(cudaMemcpyAsync(N.bc.p, bc, sizeof(int32_t) * npanels, cudaMemcpyDeviceToDevice, s));
    N.entries = tot;
    N.ready = true;
    EB_CUDA(cudaStreamSynchronize(s));
    if (std::getenv("EBEM_BUILD_TIMING"))
        std::fprintf(stderr, "[near operator] %d leaves, %lld quadrature entries, %lld columns, %.2f GB\n", ne,
                     (long long)nent, (long long)nseg, tot * 4.0 / 1e9);
    return true;
}

void near_matrix_apply(const Tree& t, const NearMat& N, const double* x, double* near, cudaStream_t s) {
    if (t.n_eval == 0) return;
    static const int pad = beside_translation_pad((const void*)nm_apply);
    nm_apply<<<t.n_eval, NM_T, pad, s>>>(t.n_eval, t.eval_box.p, t.tbeg.p, t.tend.p, N.col_first.p, N.ncol.p,
                                       N.moff.p, N.col_panel.p, N.M.p, x, near);
    EB_CHECK_LAUNCH();
}

}  // namespace ebem
