#include <chrono>
#include <cstdio>
#include <cstdlib>
// Adaptive octree and KIFMM interaction lists on the device (Sec. 2.2,
// "Generation of an octree partitioning of the domain into boxes"; reading R5 in DESIGN.md):
//   bounding cube (min/max reduction) -> 60-bit Morton keys (fp64 quantisation, one IEEE
//   op per step) -> stable LSD radix sort -> level-by-level refinement with prefix scans
//   (a box splits iff max(n_src, n_trg) > max_pts; child ranges by binary search in the
//   sorted keys) -> colleagues -> V, U, W lists (U/W by a per-leaf descent) -> X and the
//   coarse half of U as the duals of W and of the fine half of U.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "fmm.cuh"

namespace ebem {

// ------------------------------------------------------------------ helpers
__host__ __device__ __forceinline__ long long spread3(long long v) {
    // spread the low 20 bits of v so that bit b lands at bit 3b
    v &= 0xFFFFF;
    v = (v | (v << 32)) & 0x1F00000000FFFFLL;
    v = (v | (v << 16)) & 0x1F0000FF0000FFLL;
    v = (v | (v << 8)) & 0x100F00F00F00F00FLL;
    v = (v | (v << 4)) & 0x10C30C30C30C30C3LL;
    v = (v | (v << 2)) & 0x1249249249249249LL;
    return v;
}
__host__ __device__ __forceinline__ long long morton3(long long x, long long y, long long z) {
    return (spread3(x) << 2) | (spread3(y) << 1) | spread3(z);
}

__global__ void bbox_partial(const float* __restrict__ a, int64_t na, const float* __restrict__ b, int64_t nb,
                             float* __restrict__ part) {
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na + nb; i += (int64_t)gridDim.x * blockDim.x) {
        const float* p = i < na ? a + 3 * i : b + 3 * (i - na);
        for (int c = 0; c < 3; ++c) {
            lo[c] = fminf(lo[c], p[c]);
            hi[c] = fmaxf(hi[c], p[c]);
        }
    }
    __shared__ float sh[6][256];
    for (int c = 0; c < 3; ++c) {
        sh[c][threadIdx.x] = lo[c];
        sh[3 + c][threadIdx.x] = hi[c];
    }
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int c = 0; c < 3; ++c) {
                sh[c][threadIdx.x] = fminf(sh[c][threadIdx.x], sh[c][threadIdx.x + o]);
                sh[3 + c][threadIdx.x] = fmaxf(sh[3 + c][threadIdx.x], sh[3 + c][threadIdx.x + o]);
            }
        __syncthreads();
    }
    if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void morton_kernel(const float* __restrict__ src, int64_t nsrc, const float* __restrict__ trg,
                              int64_t ntrg, double ox, double oy, double oz, double scale,
                              long long* __restrict__ keys, int* __restrict__ idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nsrc + ntrg) return;
    const float* p = i < nsrc ? src + 3 * i : trg + 3 * (i - nsrc);
    const double o[3] = {ox, oy, oz};
    long long q[3];
    const double qmax = (double)((1 << MAXLEVEL) - 1);
    for (int c = 0; c < 3; ++c) {
        double t = __dmul_rn(__dsub_rn((double)p[c], o[c]), scale);   // reading R5: no FMA
        t = floor(t);
        t = fmin(fmax(t, 0.0), qmax);
        q[c] = (long long)t;
    }
    keys[i] = morton3(q[0], q[1], q[2]);
    idx[i] = (int)i;
}

__global__ void flags_kernel(const int* __restrict__ perm, int64_t n, int64_t nsrc, int* __restrict__ fs,
                             int* __restrict__ ft) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    int s = 0, t = 0;
    if (i < n) {
        s = perm[i] < nsrc;
        t = !s;
    }
    fs[i] = s;
    ft[i] = t;
}

__global__ void sorted_perms(const int* __restrict__ perm, int64_t n, int64_t nsrc, const int* __restrict__ cs,
                            const int* __restrict__ ct, int* __restrict__ src_perm, int* __restrict__ trg_perm) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int o = perm[i];
    if (o < nsrc) src_perm[cs[i]] = o;
    else trg_perm[ct[i]] = o - (int)nsrc;
}

__global__ void gather3(const float* __restrict__ in, const int* __restrict__ perm, int64_t n, int comp,
                        float* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t o = perm[i];
    for (int c = 0; c < comp; ++c) out[i * comp + c] = in ? in[o * comp + c] : 1.0f;
}

__device__ __forceinline__ int64_t lower_bound_ll(const long long* __restrict__ a, int64_t lo, int64_t hi,
                                                  long long key) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// one level: decide splits and child ranges.  Eight lanes per box, lane c finding where
// child c ends (independent binary searches: the top levels' searches over the whole key
// array were a 7-deep chain of dependent ~20-step searches in one thread).
__global__ void split_count(int nb, int level, const int* __restrict__ beg, const int* __restrict__ end,
                            const long long* __restrict__ bkey, const long long* __restrict__ keys,
                            const int* __restrict__ cs, const int* __restrict__ ct, int max_pts,
                            int* __restrict__ cb, int* __restrict__ nchild) {
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int c = (int)(gid & 7);
    const int64_t b = gid >> 3;
    const bool valid = b < nb;
    const int B = valid ? beg[b] : 0, E = valid ? end[b] : 0;
    const bool split = valid && level < MAXLEVEL && max(cs[E] - cs[B], ct[E] - ct[B]) > max_pts;
    int64_t e = E;
    if (split && c < 7) {
        const int shift = 3 * (MAXLEVEL - level - 1);
        const long long hi = ((bkey[b] << 3) + c + 1) << shift;
        e = lower_bound_ll(keys, B, E, hi);
    }
    // child c spans [end of child c-1, e)
    const unsigned mask = 0xffffffffu;
    int64_t prev = __shfl_up_sync(mask, e, 1, 8);
    if (c == 0) prev = B;
    const unsigned nonempty = __ballot_sync(mask, split && e > prev);
    if (!valid) return;
    if (split) {
        cb[9 * b + c] = (int)prev;
        if (c == 7) cb[9 * b + 8] = E;
    } else {
        cb[9 * b + c] = -1;
        if (c == 7) cb[9 * b + 8] = -1;
    }
    if (c == 0) nchild[b] = __popc((nonempty >> (threadIdx.x & 24)) & 0xffu);
}

__global__ void make_children(int nb, int base_this, int base_next, const int* __restrict__ cb,
                              const int* __restrict__ choff, const long long* __restrict__ bkey,
                              const int* __restrict__ anchor, int* __restrict__ child,
                              int* __restrict__ nbeg, int* __restrict__ nend, int* __restrict__ npar,
                              long long* __restrict__ nkey, int* __restrict__ nanchor) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int k = choff[b];
    for (int c = 0; c < 8; ++c) {
        int id = -1;
        if (cb[9 * b] >= 0) {
            int s = cb[9 * b + c], e = cb[9 * b + c + 1];
            if (e > s) {
                nbeg[k] = s;
                nend[k] = e;
                npar[k] = base_this + b;
                nkey[k] = (bkey[b] << 3) | c;
                nanchor[3 * k] = 2 * anchor[3 * b] + ((c >> 2) & 1);
                nanchor[3 * k + 1] = 2 * anchor[3 * b + 1] + ((c >> 1) & 1);
                nanchor[3 * k + 2] = 2 * anchor[3 * b + 2] + (c & 1);
                id = base_next + k;
                ++k;
            }
        }
        child[8 * b + c] = id;
    }
}

__global__ void box_derived(int nb, const int* __restrict__ beg, const int* __restrict__ end,
                            const int* __restrict__ cs, const int* __restrict__ ct, const int* __restrict__ child,
                            int* sbeg, int* send, int* tbeg, int* tend, int* nsub, int* tsub, int* leaf) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    sbeg[b] = cs[beg[b]];
    send[b] = cs[end[b]];
    tbeg[b] = ct[beg[b]];
    tend[b] = ct[end[b]];
    nsub[b] = send[b] - sbeg[b];
    tsub[b] = tend[b] - tbeg[b];
    int l = 1;
    for (int c = 0; c < 8; ++c) l &= child[8 * b + c] < 0;
    leaf[b] = l;
}

__global__ void colleagues_kernel(int nb, const int* __restrict__ level, const int* __restrict__ anchor,
                                  const long long* __restrict__ bkey, const int* __restrict__ lstart,
                                  int* __restrict__ coll) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int l = level[b];
    const int lim = 1 << l;
    int k = 0;
    for (int dx = -1; dx <= 1; ++dx)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dz = -1; dz <= 1; ++dz, ++k) {
                int x = anchor[3 * b] + dx, y = anchor[3 * b + 1] + dy, z = anchor[3 * b + 2] + dz;
                int id = -1;
                if (x >= 0 && y >= 0 && z >= 0 && x < lim && y < lim && z < lim) {
                    long long key = morton3(x, y, z);
                    int64_t pos = lower_bound_ll(bkey, lstart[l], lstart[l + 1], key);
                    if (pos < lstart[l + 1] && bkey[pos] == key) id = (int)pos;
                }
                coll[27 * b + k] = id;
            }
}

__device__ __forceinline__ bool adjacent_boxes(int la, const int* aa, int lb, const int* ab) {
    // closed cubes intersect and neither contains the other (reading R5)
    const int L = max(la, lb);
    const int sa = 1 << (L - la), sb = 1 << (L - lb);
    bool touch = true, ainb = true, bina = true;
    for (int c = 0; c < 3; ++c) {
        int alo = aa[c] * sa, ahi = alo + sa, blo = ab[c] * sb, bhi = blo + sb;
        touch &= (alo <= bhi) && (blo <= ahi);
        ainb &= (alo >= blo) && (ahi <= bhi);
        bina &= (blo >= alo) && (bhi <= ahi);
    }
    return touch && !ainb && !bina;
}

__device__ void sort_ints(int* a, int n) {
    for (int i = 1; i < n; ++i) {
        int v = a[i], j = i - 1;
        while (j >= 0 && a[j] > v) {
            a[j + 1] = a[j];
            --j;
        }
        a[j + 1] = v;
    }
}

// V(B): children of colleagues of parent(B) not adjacent to B (same level: Chebyshev > 1)
template <bool FILL>
__global__ void vlist_kernel(int nb, const int* __restrict__ level, const int* __restrict__ parent,
                             const int* __restrict__ anchor, const int* __restrict__ child,
                             const int* __restrict__ coll, int* __restrict__ cnt, const int* __restrict__ off,
                             int* __restrict__ out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int par = parent[b];
    int n = 0;
    if (par >= 0) {
        for (int k = 0; k < 27; ++k) {
            int c = coll[27 * par + k];
            if (c < 0) continue;
            for (int q = 0; q < 8; ++q) {
                int a = child[8 * c + q];
                if (a < 0) continue;
                int d = max(abs(anchor[3 * a] - anchor[3 * b]),
                            max(abs(anchor[3 * a + 1] - anchor[3 * b + 1]), abs(anchor[3 * a + 2] - anchor[3 * b + 2])));
                if (d > 1) {
                    if (FILL) out[off[b] + n] = a;
                    ++n;
                }
            }
        }
    }
    if (FILL) sort_ints(out + off[b], n);
    else cnt[b] = n;
}

// U (same level + finer adjacent leaves) and W for every leaf: descent into colleagues
template <bool FILL>
__global__ void uw_kernel(int nb, const int* __restrict__ level, const int* __restrict__ anchor,
                          const int* __restrict__ child, const int* __restrict__ leaf, const int* __restrict__ coll,
                          int* __restrict__ ucnt, int* __restrict__ wcnt, const int* __restrict__ uoff,
                          const int* __restrict__ woff, int* __restrict__ uout, int* __restrict__ wout) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int nu = 0, nw = 0;
    if (leaf[b]) {
        int stack[8 * (MAXLEVEL + 2)];
        int sp = 0;
        for (int k = 0; k < 27; ++k) {
            int c = coll[27 * b + k];
            if (c < 0) continue;
            if (leaf[c]) {
                if (FILL) uout[uoff[b] + nu] = c;
                ++nu;
            } else if (c != b) {
                for (int q = 0; q < 8; ++q)
                    if (child[8 * c + q] >= 0) stack[sp++] = child[8 * c + q];
                while (sp > 0) {
                    int a = stack[--sp];
                    if (adjacent_boxes(level[a], anchor + 3 * a, level[b], anchor + 3 * b)) {
                        if (leaf[a]) {
                            if (FILL) uout[uoff[b] + nu] = a;
                            ++nu;
                        } else {
                            for (int q = 0; q < 8; ++q)
                                if (child[8 * a + q] >= 0) stack[sp++] = child[8 * a + q];
                        }
                    } else {
                        if (FILL) wout[woff[b] + nw] = a;
                        ++nw;
                    }
                }
            }
        }
    }
    if (FILL) {
        sort_ints(uout + uoff[b], nu);
        sort_ints(wout + woff[b], nw);
    } else {
        ucnt[b] = nu;
        wcnt[b] = nw;
    }
}

// duals: coarse-U entries (b in U(a) for finer a) and X (b in X(a) for a in W(b))
__global__ void dual_count(int nb, const int* __restrict__ level, const int* __restrict__ uoff,
                           const int* __restrict__ uidx, const int* __restrict__ woff, const int* __restrict__ widx,
                           int* __restrict__ ucoarse, int* __restrict__ xcnt) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    for (int e = uoff[b]; e < uoff[b + 1]; ++e) {
        int a = uidx[e];
        if (level[a] > level[b]) atomicAdd(&ucoarse[a], 1);
    }
    for (int e = woff[b]; e < woff[b + 1]; ++e) atomicAdd(&xcnt[widx[e]], 1);
}

__global__ void dual_fill(int nb, const int* __restrict__ level, const int* __restrict__ ufoff,
                          const int* __restrict__ ufidx, const int* __restrict__ woff, const int* __restrict__ widx,
                          const int* __restrict__ uoff, int* __restrict__ ucur, int* __restrict__ uidx,
                          const int* __restrict__ xoff, int* __restrict__ xcur, int* __restrict__ xidx) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    for (int e = ufoff[b]; e < ufoff[b + 1]; ++e) {
        int a = ufidx[e];
        if (level[a] > level[b]) uidx[uoff[a] + atomicAdd(&ucur[a], 1)] = b;
    }
    for (int e = woff[b]; e < woff[b + 1]; ++e) {
        int a = widx[e];
        xidx[xoff[a] + atomicAdd(&xcur[a], 1)] = b;
    }
}

__global__ void copy_own_u(int nb, const int* __restrict__ ufoff, const int* __restrict__ ufidx,
                           const int* __restrict__ uoff, int* __restrict__ uidx, int* __restrict__ ucur) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int n = ufoff[b + 1] - ufoff[b];
    for (int e = 0; e < n; ++e) uidx[uoff[b] + e] = ufidx[ufoff[b] + e];
    ucur[b] = n;
}

__global__ void sort_lists(int nb, const int* __restrict__ off, int* __restrict__ idx) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    sort_ints(idx + off[b], off[b + 1] - off[b]);
}

__global__ void add_arrays(int n, const int* a, const int* b, int* c) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) c[i] = a[i] + b[i];
}

// ------------------------------------------------------------------ driver
static void csr_from_counts(DBuf<int>& cnt_then_off, int nb, int64_t& total, cudaStream_t s) {
    // cnt_then_off has nb+1 entries, last = 0; becomes the exclusive scan
    total = exclusive_scan_i32(cnt_then_off.p, cnt_then_off.p, nb + 1, s);
}

void schedule_tree(Tree& t, cudaStream_t s);   // fmm.cu

Tree* build_tree(const float* src, const float* nrm, const float* w, int64_t nsrc, const float* trg,
                 int64_t ntrg, int max_pts, int p, const Material& m, cudaStream_t s, double w_direct) {
    const auto t0_build = std::chrono::steady_clock::now();
    auto T = std::make_unique<Tree>();
    T->w_direct = w_direct;
    Tree& t = *T;
    t.nsrc = nsrc;
    t.ntrg = ntrg;
    t.npts = nsrc + ntrg;
    t.max_pts = max_pts;
    t.p = p;
    t.mat = m;
    t.has_normals = nrm != nullptr;
    t.has_weights = w != nullptr;
    const int64_t n = t.npts;

    // ---- root cube (reading R5): exact fp32 min/max, then fp64 on the host
    {
        const int nbk = 256;
        DBuf<float> part(6 * nbk);
        bbox_partial<<<nbk, 256, 0, s>>>(src, nsrc, trg, ntrg, part.p);
        EB_CHECK_LAUNCH();
        std::vector<float> hp(6 * nbk);
        d2h(hp.data(), part.p, 6 * nbk, s);
        EB_CUDA(cudaStreamSynchronize(s));
        double lo[3], hi[3];
        for (int c = 0; c < 3; ++c) {
            float a = INFINITY, b = -INFINITY;
            for (int k = 0; k < nbk; ++k) {
                a = std::min(a, hp[6 * k + c]);
                b = std::max(b, hp[6 * k + 3 + c]);
            }
            lo[c] = a;
            hi[c] = b;
        }
        double side = 0;
        for (int c = 0; c < 3; ++c) side = std::max(side, hi[c] - lo[c]);
        side = side == 0.0 ? 1.0 : side * (1.0 + std::ldexp(1.0, -10));
        t.side = side;
        for (int c = 0; c < 3; ++c) {
            volatile double mid = (lo[c] + hi[c]) * 0.5;
            volatile double hs = side * 0.5;
            t.origin[c] = mid - hs;
        }
    }
    // ---- Morton keys + stable sort
    t.keys.alloc(n);
    t.perm.alloc(n);
    const double scale = (double)(1 << MAXLEVEL) / t.side;
    morton_kernel<<<ceil_div(n, 256), 256, 0, s>>>(src, nsrc, trg, ntrg, t.origin[0], t.origin[1], t.origin[2],
                                                   scale, t.keys.p, t.perm.p);
    EB_CHECK_LAUNCH();
    radix_sort_pairs(t.keys.p, t.perm.p, n, 3 * MAXLEVEL, s);

    // ---- source / target prefix counts over sorted positions
    DBuf<int> cs(n + 1), ct(n + 1);
    flags_kernel<<<ceil_div(n + 1, 256), 256, 0, s>>>(t.perm.p, n, nsrc, cs.p, ct.p);
    EB_CHECK_LAUNCH();
    exclusive_scan_i32(cs.p, cs.p, n + 1, s);
    exclusive_scan_i32(ct.p, ct.p, n + 1, s);
    t.src_perm.alloc(std::max<int64_t>(nsrc, 1));
    t.trg_perm.alloc(std::max<int64_t>(ntrg, 1));
    sorted_perms<<<ceil_div(n, 256), 256, 0, s>>>(t.perm.p, n, nsrc, cs.p, ct.p, t.src_perm.p, t.trg_perm.p);
    EB_CHECK_LAUNCH();
    t.src_xyz.alloc(std::max<int64_t>(3 * nsrc, 1));
    t.src_nrm.alloc(std::max<int64_t>(3 * nsrc, 1));
    t.src_w.alloc(std::max<int64_t>(nsrc, 1));
    t.trg_xyz.alloc(std::max<int64_t>(3 * ntrg, 1));
    if (nsrc) {
        gather3<<<ceil_div(nsrc, 256), 256, 0, s>>>(src, t.src_perm.p, nsrc, 3, t.src_xyz.p);
        if (nrm) gather3<<<ceil_div(nsrc, 256), 256, 0, s>>>(nrm, t.src_perm.p, nsrc, 3, t.src_nrm.p);
        gather3<<<ceil_div(nsrc, 256), 256, 0, s>>>(w, t.src_perm.p, nsrc, 1, t.src_w.p);
    }
    if (ntrg) gather3<<<ceil_div(ntrg, 256), 256, 0, s>>>(trg, t.trg_perm.p, ntrg, 3, t.trg_xyz.p);
    EB_CHECK_LAUNCH();

    // ---- level-by-level refinement
    struct Lvl {
        DBuf<int> beg, end, par, anchor, child;
        DBuf<long long> key;
        int n = 0;
    };
    std::vector<Lvl> L(1);
    L[0].n = 1;
    L[0].beg.alloc(1);
    L[0].end.alloc(1);
    L[0].par.alloc(1);
    L[0].anchor.alloc(3);
    L[0].key.alloc(1);
    {
        int hb[1] = {0}, he[1] = {(int)n}, hp[1] = {-1}, ha[3] = {0, 0, 0};
        long long hk[1] = {0};
        h2d(L[0].beg.p, hb, 1, s);
        h2d(L[0].end.p, he, 1, s);
        h2d(L[0].par.p, hp, 1, s);
        h2d(L[0].anchor.p, ha, 3, s);
        h2d(L[0].key.p, hk, 1, s);
    }
    int base = 0;
    for (int l = 0;; ++l) {
        Lvl& cur = L[l];
        const int nb = cur.n;
        DBuf<int> cb(9 * nb), nch(nb + 1);
        EB_CUDA(cudaMemsetAsync(nch.p, 0, sizeof(int) * (nb + 1), s));
        split_count<<<ceil_div((int64_t)nb * 8, 128), 128, 0, s>>>(nb, l, cur.beg.p, cur.end.p, cur.key.p, t.keys.p,
                                                                  cs.p, ct.p, max_pts, cb.p, nch.p);
        EB_CHECK_LAUNCH();
        const int nnext = (int)exclusive_scan_i32(nch.p, nch.p, nb + 1, s);
        cur.child.alloc(8 * nb);
        Lvl nx;
        nx.n = nnext;
        nx.beg.alloc(std::max(nnext, 1));
        nx.end.alloc(std::max(nnext, 1));
        nx.par.alloc(std::max(nnext, 1));
        nx.anchor.alloc(3 * std::max(nnext, 1));
        nx.key.alloc(std::max(nnext, 1));
        make_children<<<ceil_div(nb, 128), 128, 0, s>>>(nb, base, base + nb, cb.p, nch.p, cur.key.p, cur.anchor.p,
                                                        cur.child.p, nx.beg.p, nx.end.p, nx.par.p, nx.key.p,
                                                        nx.anchor.p);
        EB_CHECK_LAUNCH();
        base += nb;
        if (nnext == 0) break;
        L.push_back(std::move(nx));
    }
    t.nlevels = (int)L.size();
    t.nboxes = base;
    t.level_start.assign(t.nlevels + 1, 0);
    for (int l = 0; l < t.nlevels; ++l) t.level_start[l + 1] = t.level_start[l] + L[l].n;
    const int nb = t.nboxes;
    t.level.alloc(nb);
    t.anchor.alloc(3 * nb);
    t.parent.alloc(nb);
    t.child.alloc(8 * nb);
    t.pbeg.alloc(nb);
    t.pend.alloc(nb);
    t.bkey.alloc(nb);
    {
        std::vector<int> hl(nb);
        for (int l = 0; l < t.nlevels; ++l) {
            const int o = t.level_start[l], c = L[l].n;
            for (int i = 0; i < c; ++i) hl[o + i] = l;
            d2d(t.anchor.p + 3 * o, L[l].anchor.p, 3 * c, s);
            d2d(t.parent.p + o, L[l].par.p, c, s);
            d2d(t.child.p + 8 * o, L[l].child.p, 8 * c, s);
            d2d(t.pbeg.p + o, L[l].beg.p, c, s);
            d2d(t.pend.p + o, L[l].end.p, c, s);
            d2d(t.bkey.p + o, L[l].key.p, c, s);
        }
        h2d(t.level.p, hl.data(), nb, s);
        EB_CUDA(cudaStreamSynchronize(s));
    }
    L.clear();
    t.sbeg.alloc(nb);
    t.send.alloc(nb);
    t.tbeg.alloc(nb);
    t.tend.alloc(nb);
    t.nsrc_sub.alloc(nb);
    t.ntrg_sub.alloc(nb);
    t.is_leaf.alloc(nb);
    box_derived<<<ceil_div(nb, 256), 256, 0, s>>>(nb, t.pbeg.p, t.pend.p, cs.p, ct.p, t.child.p, t.sbeg.p, t.send.p,
                                                  t.tbeg.p, t.tend.p, t.nsrc_sub.p, t.ntrg_sub.p, t.is_leaf.p);
    EB_CHECK_LAUNCH();

    // ---- colleagues and lists
    DBuf<int> lstart(t.nlevels + 1);
    h2d(lstart.p, t.level_start.data(), t.nlevels + 1, s);
    t.colleague.alloc(27 * nb);
    colleagues_kernel<<<ceil_div(nb, 128), 128, 0, s>>>(nb, t.level.p, t.anchor.p, t.bkey.p, lstart.p, t.colleague.p);
    EB_CHECK_LAUNCH();
    // V
    DBuf<int>& voff = t.lst_off[1];
    voff.alloc(nb + 1);
    EB_CUDA(cudaMemsetAsync(voff.p, 0, sizeof(int) * (nb + 1), s));
    vlist_kernel<false><<<ceil_div(nb, 128), 128, 0, s>>>(nb, t.level.p, t.parent.p, t.anchor.p, t.child.p,
                                                          t.colleague.p, voff.p, nullptr, nullptr);
    EB_CHECK_LAUNCH();
    csr_from_counts(voff, nb, t.lst_n[1], s);
    t.lst_idx[1].alloc(std::max<int64_t>(t.lst_n[1], 1));
    vlist_kernel<true><<<ceil_div(nb, 128), 128, 0, s>>>(nb, t.level.p, t.parent.p, t.anchor.p, t.child.p,
                                                         t.colleague.p, nullptr, voff.p, t.lst_idx[1].p);
    EB_CHECK_LAUNCH();
    // fine U and W
    DBuf<int> ufoff(nb + 1), woff_(nb + 1);
    EB_CUDA(cudaMemsetAsync(ufoff.p, 0, sizeof(int) * (nb + 1), s));
    EB_CUDA(cudaMemsetAsync(woff_.p, 0, sizeof(int) * (nb + 1), s));
    uw_kernel<false><<<ceil_div(nb, 64), 64, 0, s>>>(nb, t.level.p, t.anchor.p, t.child.p, t.is_leaf.p, t.colleague.p,
                                                     ufoff.p, woff_.p, nullptr, nullptr, nullptr, nullptr);
    EB_CHECK_LAUNCH();
    int64_t nuf = 0;
    csr_from_counts(ufoff, nb, nuf, s);
    csr_from_counts(woff_, nb, t.lst_n[2], s);
    DBuf<int> ufidx(std::max<int64_t>(nuf, 1));
    t.lst_idx[2].alloc(std::max<int64_t>(t.lst_n[2], 1));
    uw_kernel<true><<<ceil_div(nb, 64), 64, 0, s>>>(nb, t.level.p, t.anchor.p, t.child.p, t.is_leaf.p, t.colleague.p,
                                                    nullptr, nullptr, ufoff.p, woff_.p, ufidx.p, t.lst_idx[2].p);
    EB_CHECK_LAUNCH();
    t.lst_off[2] = std::move(woff_);
    // duals
    DBuf<int> ucoarse(nb + 1), xcnt(nb + 1);
    EB_CUDA(cudaMemsetAsync(ucoarse.p, 0, sizeof(int) * (nb + 1), s));
    EB_CUDA(cudaMemsetAsync(xcnt.p, 0, sizeof(int) * (nb + 1), s));
    dual_count<<<ceil_div(nb, 128), 128, 0, s>>>(nb, t.level.p, ufoff.p, ufidx.p, t.lst_off[2].p, t.lst_idx[2].p,
                                                 ucoarse.p, xcnt.p);
    EB_CHECK_LAUNCH();
    DBuf<int> ucnt(nb + 1);
    {
        // ucnt = fine count + coarse count
        DBuf<int> fcnt(nb + 1);
        std::vector<int> hoff(nb + 1), hf(nb + 1);
        d2h(hoff.data(), ufoff.p, nb + 1, s);
        EB_CUDA(cudaStreamSynchronize(s));
        for (int b = 0; b < nb; ++b) hf[b] = hoff[b + 1] - hoff[b];
        hf[nb] = 0;
        h2d(fcnt.p, hf.data(), nb + 1, s);
        add_arrays<<<ceil_div(nb + 1, 256), 256, 0, s>>>(nb + 1, fcnt.p, ucoarse.p, ucnt.p);
        EB_CHECK_LAUNCH();
        EB_CUDA(cudaStreamSynchronize(s));
    }
    csr_from_counts(ucnt, nb, t.lst_n[0], s);
    t.lst_off[0] = std::move(ucnt);
    t.lst_idx[0].alloc(std::max<int64_t>(t.lst_n[0], 1));
    csr_from_counts(xcnt, nb, t.lst_n[3], s);
    t.lst_off[3] = std::move(xcnt);
    t.lst_idx[3].alloc(std::max<int64_t>(t.lst_n[3], 1));
    DBuf<int> ucur(nb), xcur(nb);
    EB_CUDA(cudaMemsetAsync(xcur.p, 0, sizeof(int) * nb, s));
    copy_own_u<<<ceil_div(nb, 128), 128, 0, s>>>(nb, ufoff.p, ufidx.p, t.lst_off[0].p, t.lst_idx[0].p, ucur.p);
    dual_fill<<<ceil_div(nb, 128), 128, 0, s>>>(nb, t.level.p, ufoff.p, ufidx.p, t.lst_off[2].p, t.lst_idx[2].p,
                                                t.lst_off[0].p, ucur.p, t.lst_idx[0].p, t.lst_off[3].p, xcur.p,
                                                t.lst_idx[3].p);
    sort_lists<<<ceil_div(nb, 128), 128, 0, s>>>(nb, t.lst_off[0].p, t.lst_idx[0].p);
    sort_lists<<<ceil_div(nb, 128), 128, 0, s>>>(nb, t.lst_off[3].p, t.lst_idx[3].p);
    EB_CHECK_LAUNCH();
    EB_CUDA(cudaStreamSynchronize(s));

    // ---- operators and execution schedule
    const auto tb = std::chrono::steady_clock::now();
    t.plan = get_plan(p, m, s);
    const auto tp = std::chrono::steady_clock::now();
    schedule_tree(t, s);
    if (std::getenv("EBEM_BUILD_TIMING")) {
        const auto te = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        fprintf(stderr, "[ebem build] tree+lists %.2f ms, plan %.2f ms, schedule %.2f ms\n", ms(t0_build, tb),
                ms(tb, tp), ms(tp, te));
    }
    return T.release();
}

void tree_info(const Tree& t, ebem_tree_info* info) {
    std::memset(info, 0, sizeof(*info));
    info->nsrc = t.nsrc;
    info->ntrg = t.ntrg;
    info->nboxes = t.nboxes;
    info->nleaves = t.nleaves;
    info->nlevels = t.nlevels;
    info->p = t.p;
    info->max_pts = t.max_pts;
    info->n_equiv = t.plan ? t.plan->ne : 0;
    info->n_u = t.lst_n[0];
    info->n_v = t.lst_n[1];
    info->n_w = t.lst_n[2];
    info->n_x = t.lst_n[3];
    for (int c = 0; c < 3; ++c) info->origin[c] = t.origin[c];
    info->side = t.side;
    info->device_bytes = t.device_bytes;
}

int64_t tree_export(const Tree& t, int what, void* buf, int64_t cap) {
    const void* src = nullptr;
    int64_t bytes = 0;
    switch (what) {
        case 0: src = t.keys.p; bytes = t.npts * 8; break;
        case 1: src = t.perm.p; bytes = t.npts * 4; break;
        case 2: src = t.level.p; bytes = (int64_t)t.nboxes * 4; break;
        case 3: src = t.anchor.p; bytes = (int64_t)t.nboxes * 12; break;
        case 4: src = t.parent.p; bytes = (int64_t)t.nboxes * 4; break;
        case 5: {
            EB_REQUIRE(cap >= (int64_t)t.nboxes * 8, "export buffer too small");
            std::vector<int> b(t.nboxes), e(t.nboxes), out(2 * t.nboxes);
            EB_CUDA(cudaMemcpy(b.data(), t.pbeg.p, 4 * t.nboxes, cudaMemcpyDeviceToHost));
            EB_CUDA(cudaMemcpy(e.data(), t.pend.p, 4 * t.nboxes, cudaMemcpyDeviceToHost));
            for (int i = 0; i < t.nboxes; ++i) {
                out[2 * i] = b[i];
                out[2 * i + 1] = e[i];
            }
            std::memcpy(buf, out.data(), 8 * t.nboxes);
            return (int64_t)t.nboxes * 8;
        }
        case 6: case 7: case 8: case 9:
            src = t.lst_off[what - 6].p; bytes = ((int64_t)t.nboxes + 1) * 4; break;
        case 10: case 11: case 12: case 13:
            src = t.lst_idx[what - 10].p; bytes = t.lst_n[what - 10] * 4; break;
        default: throw Error("fmm_tree_export: unknown array id");
    }
    EB_REQUIRE(cap >= bytes, "export buffer too small");
    if (bytes) EB_CUDA(cudaMemcpy(buf, src, bytes, cudaMemcpyDeviceToHost));
    return bytes;
}

}  // namespace ebem
