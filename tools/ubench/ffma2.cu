// Microbenchmark: FP32 FMA throughput of scalar FFMA vs packed FFMA2 (sm_100a).
// Each thread runs 8 independent chains; grid = 148 x 8 CTAs of 256 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2 ffma2.cu && ./ffma2
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fmaf(x[c], a, b);
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, int iters, float a, float b) {
    float2 x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = __ffma2_rn(x[c], a2, b2);
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c].x + x[c].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed: 3-register FFMA with distinct registers (no immediates)
__global__ void k_ffma_reg(float* out, int iters, const float* ab) {
    float x[8], y[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { x[c] = threadIdx.x * 1e-3f + c; y[c] = ab[c]; }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fmaf(x[c], y[c], y[(c + 1) & 7]);
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2_reg(float* out, int iters, const float* ab) {
    float2 x[8], y[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { x[c] = make_float2(threadIdx.x * 1e-3f + c, c); y[c] = make_float2(ab[c], ab[c + 1]); }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = __ffma2_rn(x[c], y[c], y[(c + 1) & 7]);
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c].x + x[c].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int blocks = sms * 8, threads = 256, iters = 20000;
    float* out;
    float* ab;
    cudaMalloc(&out, blocks * threads * sizeof(float));
    cudaMalloc(&ab, 16 * sizeof(float));
    cudaMemset(ab, 0, 16 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch, double lanes_per_thread_iter) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 5.0 * blocks * threads * (double)iters * lanes_per_thread_iter * 2;
        printf("{\"kernel\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %d}\n", name,
               flops / (ms * 1e-3) / 1e12, ms / 5, sms, clk / 1000);
    };
    run("FFMA (imm/const operands)", [&] { k_ffma<<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f); }, 8);
    run("FFMA2 (uniform operands)", [&] { k_ffma2<<<blocks, threads>>>(out, iters, 1.0001f, 1e-7f); }, 16);
    run("FFMA (3 registers)", [&] { k_ffma_reg<<<blocks, threads>>>(out, iters, ab); }, 8);
    run("FFMA2 (3 registers)", [&] { k_ffma2_reg<<<blocks, threads>>>(out, iters, ab); }, 16);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
