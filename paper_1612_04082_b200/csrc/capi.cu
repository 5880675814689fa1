// extern "C" boundary of the library (include/elastobem.h).  Argument checking, host
// staging of host-pointer calls, exception -> error-code translation.  No compute here.
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <map>
#include <mutex>

#include "../../include/elastobem.h"
#include "fmm.cuh"
#include "p2p.cuh"

namespace ebem {

static thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ------------------------------------------------------------------ block cache (DBuf)
namespace {
struct BlockCache {
    std::mutex mu;
    std::multimap<size_t, void*> free_blocks;   // rounded size -> block
    size_t cached = 0, cap = 0;
    BlockCache() {
        const char* e = std::getenv("EBEM_CACHE_MB");
        cap = (size_t)(e ? std::atoll(e) : 16384) << 20;
    }
};
BlockCache& block_cache() {
    static BlockCache* c = new BlockCache;      // never destroyed: DBufs may outlive statics
    return *c;
}
constexpr size_t CACHE_MIN = 1 << 20, CACHE_GRAIN = 2 << 20;
size_t cache_round(size_t b) { return (b + CACHE_GRAIN - 1) / CACHE_GRAIN * CACHE_GRAIN; }
}  // namespace

void* cache_alloc(size_t bytes) {
    void* p = nullptr;
    if (bytes >= CACHE_MIN) {
        BlockCache& c = block_cache();
        const size_t r = cache_round(bytes);
        {
            std::lock_guard<std::mutex> g(c.mu);
            auto it = c.free_blocks.find(r);
            if (it != c.free_blocks.end()) {
                p = it->second;
                c.free_blocks.erase(it);
                c.cached -= r;
                return p;
            }
        }
        if (cudaMalloc(&p, r) != cudaSuccess) {   // out of memory: return the cache, retry once
            cudaGetLastError();
            cache_trim();
            EB_CUDA(cudaMalloc(&p, r));
        }
        return p;
    }
    EB_CUDA(cudaMalloc(&p, bytes));
    return p;
}

void cache_free(void* p, size_t bytes) {
    if (!p) return;
    if (bytes >= CACHE_MIN) {
        BlockCache& c = block_cache();
        const size_t r = cache_round(bytes);
        std::lock_guard<std::mutex> g(c.mu);
        if (c.cached + r <= c.cap) {
            c.free_blocks.emplace(r, p);
            c.cached += r;
            return;
        }
    }
    cudaFree(p);
}

int64_t cache_trim() {
    BlockCache& c = block_cache();
    std::lock_guard<std::mutex> g(c.mu);
    for (auto& kv : c.free_blocks) cudaFree(kv.second);
    c.free_blocks.clear();
    const int64_t freed = (int64_t)c.cached;
    c.cached = 0;
    return freed;
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        EB_CUDA(cudaGetDevice(&dev));
        EB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

void direct_sum_device(int kernel, const Material& m, const float* trg, int64_t ntrg,
                       const float* src, const float* nrm, const float* w, const float* f,
                       const float* g, int64_t nsrc, float* out, cudaStream_t s);

// Copies host arrays to scratch device memory (nullptr passes through).
// The stream-ordered scratch allocations (host-pointer staging, direct-sum records and
// partial sums) come from the device's default memory pool; by default it hands memory back
// at every synchronisation, so each call re-mapped its buffers (measured: +4 ms per 1M-point
// host-pointer matvec).  Keep the freed memory in the pool instead.
void keep_pool_memory() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    EB_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    EB_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = UINT64_MAX;
    EB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    done = true;
}

struct Staged {
    std::vector<void*> bufs;
    cudaStream_t s;
    explicit Staged(cudaStream_t s_) : s(s_) {}
    template <class T>
    const T* in(const T* h, size_t n) {
        if (!h || n == 0) return h;
        T* d = nullptr;
        EB_CUDA(cudaMallocAsync(&d, n * sizeof(T), s));
        bufs.push_back(d);
        h2d(d, h, n, s);
        return d;
    }
    template <class T>
    T* out(size_t n) {
        T* d = nullptr;
        EB_CUDA(cudaMallocAsync(&d, std::max<size_t>(n, 1) * sizeof(T), s));
        bufs.push_back(d);
        return d;
    }
    ~Staged() {
        for (void* p : bufs) cudaFreeAsync(p, s);
    }
};

// Every non-NULL array argument of one call must be of one kind (include/elastobem.h,
// "Memory"): a host pointer handed to a kernel would fault and poison the CUDA context, so a
// mix is rejected up front.  Returns true for device pointers.
static bool device_args(std::initializer_list<const void*> ptrs) {
    int ndev = 0, nhost = 0;
    for (const void* p : ptrs)
        if (p) ++(is_device_ptr(p) ? ndev : nhost);
    EB_REQUIRE(ndev == 0 || nhost == 0, "array arguments mix host and device pointers");
    return ndev > 0;
}

static void check_material(double K, double G) {
    EB_REQUIRE(K > 0 && G > 0, "material: K and G must be positive");
}

static void check_kernel_args(int kernel, const float* nrm, const float* f, const float* g,
                              int64_t nsrc) {
    EB_REQUIRE(kernel >= K_U && kernel <= K_DS, "unknown kernel id");
    if (nsrc == 0) return;
    if (kernel_sl(kernel)) EB_REQUIRE(f != nullptr, "kernel needs the single-layer density f");
    if (kernel_dl(kernel)) {
        EB_REQUIRE(g != nullptr, "kernel needs the double-layer density g");
        EB_REQUIRE(nrm != nullptr, "kernel needs source normals");
    }
}

}  // namespace ebem

using namespace ebem;

#define EB_API_BEGIN \
    try {                \
        keep_pool_memory();
#define EB_API_END                                    \
    }                                                 \
    catch (const Error& e) {                          \
        set_last_error(e.what());                     \
        return std::strstr(e.what(), "cuda") || std::strstr(e.what(), "CUDA") ? EBEM_ERR_CUDA \
                                                                              : EBEM_ERR_ARG; \
    }                                                 \
    catch (const std::exception& e) {                 \
        set_last_error(e.what());                     \
        return EBEM_ERR_ARG;                          \
    }

extern "C" const char* ebem_last_error(void) { return g_last_error.c_str(); }

extern "C" int bem_kernel_direct(int kernel, const float* trg, int64_t ntrg, const float* src,
                                 const float* nrm, const float* w, const float* f, const float* g,
                                 int64_t nsrc, double K, double G, float* out, void* stream) {
    EB_API_BEGIN
    set_last_error("");
    EB_REQUIRE(ntrg >= 0 && nsrc >= 0, "negative sizes");
    EB_REQUIRE(ntrg == 0 || (trg && out), "trg/out required");
    EB_REQUIRE(nsrc == 0 || src, "src required");
    check_kernel_args(kernel, nrm, f, g, nsrc);
    check_material(K, G);
    cudaStream_t s = (cudaStream_t)stream;
    Material m = make_material(K, G);
    const int nc = kernel_ncomp(kernel);
    const bool dev = device_args({trg, src, nrm, w, f, g, out});
    if (ntrg == 0) return EBEM_OK;
    if (dev) {
        direct_sum_device(kernel, m, trg, ntrg, src, nrm, w, f, g, nsrc, out, s);
    } else {
        Staged st(s);
        const float* dtrg = st.in(trg, ntrg * 3);
        const float* dsrc = st.in(src, nsrc * 3);
        const float* dnrm = st.in(kernel_dl(kernel) ? nrm : nullptr, nsrc * 3);
        const float* dw = st.in(w, nsrc);
        const float* df = st.in(kernel_sl(kernel) ? f : nullptr, nsrc * 3);
        const float* dg = st.in(kernel_dl(kernel) ? g : nullptr, nsrc * 3);
        float* dout = st.out<float>(ntrg * nc);
        direct_sum_device(kernel, m, dtrg, ntrg, dsrc, dnrm, dw, df, dg, nsrc, dout, s);
        d2h(out, dout, ntrg * nc, s);
        EB_CUDA(cudaStreamSynchronize(s));
    }
    return EBEM_OK;
    EB_API_END
}

extern "C" int fmm_build_tree(const float* src, const float* nrm, const float* w, int64_t nsrc,
                              const float* trg, int64_t ntrg, int max_pts, int p, double K,
                              double G, ebem_tree** tree, void* stream) {
    EB_API_BEGIN
    set_last_error("");
    EB_REQUIRE(tree != nullptr, "tree out-pointer is NULL");
    *tree = nullptr;
    EB_REQUIRE(nsrc >= 0 && ntrg >= 0 && nsrc + ntrg > 0, "need at least one point");
    EB_REQUIRE(nsrc + ntrg < (int64_t)1 << 31, "at most 2^31-1 points");
    EB_REQUIRE(max_pts >= 1, "max_pts must be >= 1");
    EB_REQUIRE(p >= 3 && p <= 12, "p must be in [3, 12]");
    check_material(K, G);
    cudaStream_t s = (cudaStream_t)stream;
    const bool dev = device_args({src, nrm, w, trg});
    Staged st(s);
    const float* dsrc = dev ? src : st.in(src, nsrc * 3);
    const float* dnrm = dev ? nrm : st.in(nrm, nsrc * 3);
    const float* dw = dev ? w : st.in(w, nsrc);
    const float* dtrg = dev ? trg : st.in(trg, ntrg * 3);
    *tree = reinterpret_cast<ebem_tree*>(
        build_tree(dsrc, dnrm, dw, nsrc, dtrg, ntrg, max_pts, p, make_material(K, G), s));
    return EBEM_OK;
    EB_API_END
}

static int fmm_eval_common(ebem_tree* tree, int kernel, const float* f, const float* g, float* out,
                           void* stream, bool stress) {
    EB_API_BEGIN
    set_last_error("");
    EB_REQUIRE(tree != nullptr, "NULL tree");
    Tree* t = reinterpret_cast<Tree*>(tree);
    if (stress)
        EB_REQUIRE(kernel == K_D || kernel == K_S || kernel == K_DS, "stress needs kernel D, S or DS");
    else
        EB_REQUIRE(kernel == K_U || kernel == K_P || kernel == K_UP, "matvec needs kernel U, P or UP");
    check_kernel_args(kernel, t->has_normals ? (const float*)1 : nullptr, f, g, t->nsrc);
    EB_REQUIRE(out != nullptr || t->ntrg == 0, "out required");
    cudaStream_t s = (cudaStream_t)stream;
    const int nc = kernel_ncomp(kernel);
    if (device_args({f, g, out})) {
        fmm_evaluate(*t, kernel, f, g, out, s);
    } else {
        Staged st(s);
        const float* df = st.in(kernel_sl(kernel) ? f : nullptr, t->nsrc * 3);
        const float* dg = st.in(kernel_dl(kernel) ? g : nullptr, t->nsrc * 3);
        float* dout = st.out<float>(t->ntrg * nc);
        fmm_evaluate(*t, kernel, df, dg, dout, s);
        d2h(out, dout, t->ntrg * nc, s);
        EB_CUDA(cudaStreamSynchronize(s));
    }
    return EBEM_OK;
    EB_API_END
}

extern "C" int fmm_matvec(ebem_tree* tree, int kernel, const float* f, const float* g, float* out,
                          void* stream) {
    return fmm_eval_common(tree, kernel, f, g, out, stream, false);
}

extern "C" int fmm_eval_stress(ebem_tree* tree, int kernel, const float* f, const float* g,
                               float* out, void* stream) {
    return fmm_eval_common(tree, kernel, f, g, out, stream, true);
}

extern "C" int fmm_tree_free(ebem_tree* tree) {
    EB_API_BEGIN
    delete reinterpret_cast<Tree*>(tree);
    return EBEM_OK;
    EB_API_END
}

extern "C" int64_t ebem_launch_count(void) { return launch_count(); }

extern "C" int64_t ebem_trim_cache(void) { return cache_trim(); }

extern "C" int fmm_set_profiling(ebem_tree* tree, int on) {
    EB_API_BEGIN
    EB_REQUIRE(tree, "NULL tree");
    set_profiling(*reinterpret_cast<Tree*>(tree), on);
    return EBEM_OK;
    EB_API_END
}

extern "C" int fmm_phase_stats(ebem_tree* tree, int kernel, ebem_phase_stat* out, int cap) {
    EB_API_BEGIN
    EB_REQUIRE(tree && out && cap >= 0, "bad argument");
    EB_REQUIRE(kernel >= K_U && kernel <= K_DS, "unknown kernel id");
    return phase_stats(*reinterpret_cast<Tree*>(tree), kernel, out, cap);
    EB_API_END
}

extern "C" int fmm_tree_info(const ebem_tree* tree, ebem_tree_info* info) {
    EB_API_BEGIN
    EB_REQUIRE(tree && info, "NULL argument");
    const Tree* t = reinterpret_cast<const Tree*>(tree);
    tree_info(*t, info);
    return EBEM_OK;
    EB_API_END
}

extern "C" int64_t fmm_tree_export(const ebem_tree* tree, int what, void* buf, int64_t cap) {
    EB_API_BEGIN
    EB_REQUIRE(tree && buf, "NULL argument");
    return tree_export(*reinterpret_cast<const Tree*>(tree), what, buf, cap);
    EB_API_END
}

extern "C" int bem_create(const float* vertices, int64_t npanels, int nq, int max_pts, int p, double K, double G,
                          ebem_bem** bem, void* stream) {
    EB_API_BEGIN
    set_last_error("");
    EB_REQUIRE(bem && vertices && npanels > 0, "bad argument");
    EB_REQUIRE(max_pts >= 1 && p >= 3 && p <= 12, "bad FMM parameters");
    check_material(K, G);
    cudaStream_t s = (cudaStream_t)stream;
    Staged st(s);
    const float* dv = is_device_ptr(vertices) ? vertices : st.in(vertices, npanels * 9);
    *bem = reinterpret_cast<ebem_bem*>(ebem::bem_create(dv, npanels, nq, max_pts, p, make_material(K, G), s));
    return EBEM_OK;
    EB_API_END
}

extern "C" int bem_apply(ebem_bem* bem, const int32_t* bc_type, const float* x, float* y, void* stream) {
    EB_API_BEGIN
    EB_REQUIRE(bem && bc_type && x && y, "NULL argument");
    EB_REQUIRE(device_args({bc_type, x, y}), "bem_apply needs device pointers");
    ebem::bem_apply(*reinterpret_cast<Bem*>(bem), bc_type, x, y, (cudaStream_t)stream);
    return EBEM_OK;
    EB_API_END
}

extern "C" int bem_rhs(ebem_bem* bem, const int32_t* bc_type, const float* bc_val, float* b, void* stream) {
    EB_API_BEGIN
    EB_REQUIRE(bem && bc_type && bc_val && b, "NULL argument");
    EB_REQUIRE(device_args({bc_type, bc_val, b}), "bem_rhs needs device pointers");
    ebem::bem_rhs(*reinterpret_cast<Bem*>(bem), bc_type, bc_val, b, (cudaStream_t)stream);
    return EBEM_OK;
    EB_API_END
}

extern "C" int bem_gmres_solve(ebem_bem* bem, const int32_t* bc_type, const float* bc_val, float* x, int restart,
                               int max_iter, double tol, int precond, int32_t* iters_out, double* resid_out,
                               void* stream) {
    EB_API_BEGIN
    set_last_error("");
    EB_REQUIRE(bem && bc_type && bc_val && x, "NULL argument");
    EB_REQUIRE(restart >= 1 && restart <= 63 && max_iter >= 1 && tol > 0, "bad GMRES parameters");
    EB_REQUIRE(precond >= 0 && precond <= 2, "precond must be 0, 1 or 2");
    EB_REQUIRE(device_args({bc_type, bc_val, x}), "bem_gmres_solve needs device pointers");
    const int rc = ebem::bem_gmres(*reinterpret_cast<Bem*>(bem), bc_type, bc_val, x, restart, max_iter, tol, iters_out,
                                   resid_out, precond, (cudaStream_t)stream);
    if (rc != EBEM_OK) set_last_error("GMRES did not reach the tolerance");
    return rc;
    EB_API_END
}

extern "C" int bem_gmres_history(const ebem_bem* bem, int what, double* buf, int cap) {
    EB_API_BEGIN
    EB_REQUIRE(bem && (buf || cap == 0) && cap >= 0 && (what == 0 || what == 1), "bad argument");
    return bem_history(*reinterpret_cast<const Bem*>(bem), what, buf, cap);
    EB_API_END
}

extern "C" int bem_free(ebem_bem* bem) {
    EB_API_BEGIN
    ebem::bem_free(reinterpret_cast<Bem*>(bem));
    return EBEM_OK;
    EB_API_END
}
