// Microbenchmark: how fast can one B200 add 310 M fp64 values into random 456-element rows of a
// 153 MB accumulator (the M2L epilogue's traffic, 1M-point matvec at p = 6)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_rates tools/ubench/red_rates.cu && ./red_rates
// Variants (each thread block = 128 threads = 128 operator rows, loops over "columns" whose
// target row is pseudo-random, like a translation tile's pairs):
//   0  red.global.add.f64, one per lane (the kernel's epilogue)
//   1  red.global.add.f32, one per lane
//   2  red.global.add.v2.f32 (lane owns 2 consecutive rows)
//   3  red.global.add.v4.f32 (lane owns 4 consecutive rows)
//   6  red.global.add.u64 (fixed-point accumulation), one per lane
//   7  red.global.add.u32, one per lane
//   4  cp.reduce.async.bulk .add.f64 from shared memory, one 1 KB row slice (128 rows) per op
//   5  the same, one 256 B slice (32 rows) per op, issued by each warp's lane 0
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int LD = 456;
__constant__ int NROWS_D = 41913;   // rows of the accumulator (argv[1]); 41913 rows = 153 MB in fp64
static int NROWS = 41913;
static int CTAS_PER_SM = 4;            // argv[2]: 128-thread CTAs per SM issuing the adds

__device__ __forceinline__ unsigned hash(unsigned x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(128) k(double* Y, float* Yf, int cols_per_cta) {
    __shared__ __align__(128) double stage[2][128];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int m0 = (blockIdx.x % 3) * 128;            // row slice 0, 128, 256 (rows < 384 + 72)
    for (int c = 0; c < cols_per_cta; ++c) {
        const unsigned tr = hash(blockIdx.x * 7919u + c) % NROWS_D;
        const float v = 1.0f + lane;
        if (MODE == 0) {
            atomicAdd(Y + (size_t)tr * LD + m0 + t, (double)v);
        } else if (MODE == 1) {
            atomicAdd(Yf + (size_t)tr * LD + m0 + t, v);
        } else if (MODE == 2) {
            if (t < 64)
                asm volatile("red.global.v2.f32.add [%0], {%1, %2};" ::"l"(Yf + (size_t)tr * LD + m0 + 2 * t), "f"(v), "f"(v) : "memory");
            else
                asm volatile("red.global.v2.f32.add [%0], {%1, %2};" ::"l"(Yf + (size_t)(tr ^ 1) * LD + m0 + 2 * (t - 64)), "f"(v), "f"(v) : "memory");
        } else if (MODE == 3) {
            // 128 threads cover 4 columns' 128 rows: thread -> (column t / 32, rows 4 (t % 32))
            const unsigned tr4 = (tr + (t >> 5)) % NROWS_D;
            asm volatile("red.global.v4.f32.add [%0], {%1, %2, %3, %4};" ::"l"(Yf + (size_t)tr4 * LD + m0 + 4 * (t & 31)), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
        } else if (MODE == 6) {
            atomicAdd(reinterpret_cast<unsigned long long*>(Y) + (size_t)tr * LD + m0 + t, (unsigned long long)(long long)(v * 1024.f));
        } else if (MODE == 7) {
            atomicAdd(reinterpret_cast<unsigned*>(Yf) + (size_t)tr * LD + m0 + t, (unsigned)(int)(v * 1024.f));
        } else if (MODE == 4) {
            double* st = stage[c & 1];
            if (c >= 2) {   // the bulk op that read this buffer two columns ago must have read it
                if (t == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncthreads();
            }
            st[t] = (double)v;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (t == 0) {
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(Y + (size_t)tr * LD + m0),
                             "r"((unsigned)__cvta_generic_to_shared(st)), "r"(1024) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else if (MODE == 5) {
            double* st = stage[c & 1] + 32 * warp;
            if (c >= 2) {
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
            }
            st[lane] = (double)v;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(Y + (size_t)tr * LD + m0 + 32 * warp),
                             "r"((unsigned)__cvta_generic_to_shared(st)), "r"(256) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    if (MODE >= 4) {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

template <int MODE>
void run(const char* what, double* Y, float* Yf, double values_per_thread_col) {
    // total values = 310 M in every variant
    const int grid = 148 * CTAS_PER_SM;
    const double total = 310e6;
    const int cols = (int)(total / (grid * 128.0 * values_per_thread_col));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    k<MODE><<<grid, 128>>>(Y, Yf, cols);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    k<MODE><<<grid, 128>>>(Y, Yf, cols);
    CK(cudaEventRecord(b));
    CK(cudaDeviceSynchronize());
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double vals = (double)grid * 128 * cols * values_per_thread_col;
    printf("%-58s %7.3f ms for %.0f M values = %6.1f G values/s\n", what, ms, vals / 1e6, vals / ms / 1e6);
}

int main(int argc, char** argv) {
    if (argc > 1) NROWS = atoi(argv[1]);
    if (argc > 2) CTAS_PER_SM = atoi(argv[2]);
    printf("%d CTAs of 128 threads per SM\n", CTAS_PER_SM);
    CK(cudaMemcpyToSymbol(NROWS_D, &NROWS, sizeof(int)));
    printf("accumulator: %d rows x 456 = %.0f MB (fp64), %.0f MB (fp32)\n", NROWS, NROWS * 456 * 8e-6, NROWS * 456 * 4e-6);
    double* Y; float* Yf;
    CK(cudaMalloc(&Y, (size_t)NROWS * LD * 8));
    CK(cudaMalloc(&Yf, (size_t)NROWS * LD * 4));
    CK(cudaMemset(Y, 0, (size_t)NROWS * LD * 8));
    CK(cudaMemset(Yf, 0, (size_t)NROWS * LD * 4));
    run<0>("red.f64, one per lane (256 B per warp)", Y, Yf, 1);
    run<1>("red.f32, one per lane (128 B per warp)", Y, Yf, 1);
    run<2>("red.v2.f32 (8 B per lane)", Y, Yf, 2);
    run<3>("red.v4.f32 (16 B per lane)", Y, Yf, 4);
    run<6>("red.u64, one per lane (256 B per warp)", Y, Yf, 1);
    run<7>("red.u32, one per lane (128 B per warp)", Y, Yf, 1);
    run<4>("cp.reduce.async.bulk add.f64, 1 KB per op (via smem)", Y, Yf, 1);
    run<5>("cp.reduce.async.bulk add.f64, 256 B per op (via smem)", Y, Yf, 1);
    return 0;
}
