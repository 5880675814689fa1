// Shared host/device plumbing for the elastostatic BEM/KIFMM library (sm_100a).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace ebem {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
    explicit Error(const std::string& s) : std::runtime_error(s) {}
};

void set_last_error(const std::string& s);

#define EB_CUDA(call)                                                                       \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            throw ::ebem::Error(std::string(#call) + ": " + cudaGetErrorString(e_) + " at " \
                                + __FILE__ + ":" + std::to_string(__LINE__));               \
    } while (0)

// every kernel launch of the library is followed by EB_CHECK_LAUNCH(), which also counts it
// (ebem_launch_count(): the bench's evidence of how many of our kernels ran)
void count_launch();
#define EB_CHECK_LAUNCH()          \
    do {                           \
        ::ebem::count_launch();    \
        EB_CUDA(cudaGetLastError()); \
    } while (0)

#define EB_REQUIRE(cond, msg)                                  \
    do {                                                       \
        if (!(cond)) throw ::ebem::Error(std::string(msg));    \
    } while (0)

// ------------------------------------------------------------------ device buffers
// Block cache behind DBuf: released blocks of >= 1 MB are kept (up to a total of
// EBEM_CACHE_MB, default 16 GB) and handed out again to an allocation of the same rounded
// size, so rebuilding a tree of the same problem allocates nothing (cudaMalloc + cudaFree of
// the ~1 GB workspace cost 4-5 ms of a 1M-point build).  cache_trim() returns everything to
// the driver (before free-memory queries).
void* cache_alloc(size_t bytes);
void cache_free(void* p, size_t bytes);
int64_t cache_trim();        // returns the bytes handed back to the driver

// Owning device allocation (the block cache above; the library's only allocator for
// long-lived state, stream-ordered cudaMallocAsync for per-call scratch).
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t n_) { alloc(n_); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t n_) {
        release();
        n = n_;
        if (n) p = (T*)cache_alloc(n * sizeof(T));
    }
    void release() {
        if (p) cache_free(p, n * sizeof(T));
        p = nullptr;
        n = 0;
    }
    void zero(cudaStream_t s) {
        if (n) EB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
    size_t bytes() const { return n * sizeof(T); }
};

template <class T>
inline void h2d(T* dst, const T* src, size_t n, cudaStream_t s) {
    if (n) EB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <class T>
inline void d2h(T* dst, const T* src, size_t n, cudaStream_t s) {
    if (n) EB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}
template <class T>
inline void d2d(T* dst, const T* src, size_t n, cudaStream_t s) {
    if (n) EB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
}

// true if p is a device (or managed) pointer; host pageable/pinned -> false
bool is_device_ptr(const void* p);

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

int num_sms();

// ------------------------------------------------------------------ material
// Constants of the four kernels for isotropic material (K, G) -> (G, nu), PAPER.md
// Eq. (elast) and Eqs. disp_1, disp_2, stress_2, stress_3 (readings R1-R3).
struct Material {
    double K, G, nu;
    double cU;   // 1 / (16 pi (1-nu) G)          U
    double a1;   // 3 - 4 nu                      U
    double cP;   // 1 / (8 pi (1-nu))             P
    double a;    // 1 - 2 nu                      P, D, S
    double cD;   // -1 / (8 pi (1-nu))            D (reading R2)
    double cS;   // G / (4 pi (1-nu))             S (reading R3)
    double b4;   // 1 - 4 nu                      S
};

inline Material make_material(double K, double G) {
    const double PI = 3.14159265358979323846;
    Material m;
    m.K = K;
    m.G = G;
    m.nu = (3.0 * K - 2.0 * G) / (2.0 * (3.0 * K + G));
    m.cU = 1.0 / (16.0 * PI * (1.0 - m.nu) * G);
    m.a1 = 3.0 - 4.0 * m.nu;
    m.cP = 1.0 / (8.0 * PI * (1.0 - m.nu));
    m.a = 1.0 - 2.0 * m.nu;
    m.cD = -1.0 / (8.0 * PI * (1.0 - m.nu));
    m.cS = G / (4.0 * PI * (1.0 - m.nu));
    m.b4 = 1.0 - 4.0 * m.nu;
    return m;
}

}  // namespace ebem
