// FFMA2 operand forms (sm_100a): throughput of packed FP32 FMA by operand kind.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_forms ffma2_forms.cu
#include <cstdio>
#include <cuda_runtime.h>

// A: acc_c = fma(v_c, s (per-thread scalar, broadcast), acc_c)
__global__ void kA(float* out, int iters, const float* in) {
    const int t = threadIdx.x;
    float s = in[t & 15];
    float2 v[8], acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { v[c] = make_float2(in[c], in[c + 1]); acc[c] = make_float2(t, c); }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = __ffma2_rn(v[c], make_float2(s, s), acc[c]);
        s += 1e-7f;   // keep s a live per-thread register
    }
    float r = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) r += acc[c].x + acc[c].y;
    out[blockIdx.x * blockDim.x + t] = r;
}
// B: acc_c = fma(v_c, w_c, acc_c), all operands packed registers
__global__ void kB(float* out, int iters, const float* in) {
    const int t = threadIdx.x;
    float2 v[8], w[8], acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { v[c] = make_float2(in[c], in[c + 1]); w[c] = make_float2(in[c + 2], in[c + 3]); acc[c] = make_float2(t, c); }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = __ffma2_rn(v[c], w[c], acc[c]);
    float r = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) r += acc[c].x + acc[c].y;
    out[blockIdx.x * blockDim.x + t] = r;
}
// C: scalar FFMA with three registers: acc_c = fma(v_c, w_c, acc_c)
__global__ void kC(float* out, int iters, const float* in) {
    const int t = threadIdx.x;
    float v[16], w[16], acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) { v[c] = in[c]; w[c] = in[c + 2]; acc[c] = t + c; }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[c] = fmaf(v[c], w[c], acc[c]);
    float r = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) r += acc[c];
    out[blockIdx.x * blockDim.x + t] = r;
}
// D: FMUL2 chains: acc_c = acc_c * v_c
__global__ void kD(float* out, int iters, const float* in) {
    const int t = threadIdx.x;
    float2 v[8], acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) { v[c] = make_float2(in[c], in[c + 1]); acc[c] = make_float2(t, c); }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = __fmul2_rn(acc[c], v[c]);
    float r = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) r += acc[c].x + acc[c].y;
    out[blockIdx.x * blockDim.x + t] = r;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 20000;
    float *out, *in;
    cudaMalloc(&out, blocks * threads * sizeof(float));
    cudaMalloc(&in, 32 * sizeof(float));
    float h[32];
    for (int i = 0; i < 32; ++i) h[i] = 1.0f + 1e-7f * i;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch, double lanes) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"form\": \"%s\", \"lane_ops_per_s_T\": %.2f}\n", name, 5.0 * blocks * threads * (double)iters * lanes / (ms * 1e-3) / 1e12);
    };
    run("A FFMA2 v, bcast-reg, acc", [&] { kA<<<blocks, threads>>>(out, iters, in); }, 16);
    run("B FFMA2 v, w, acc", [&] { kB<<<blocks, threads>>>(out, iters, in); }, 16);
    run("C FFMA v, w, acc (scalar)", [&] { kC<<<blocks, threads>>>(out, iters, in); }, 16);
    run("D FMUL2 acc, v", [&] { kD<<<blocks, threads>>>(out, iters, in); }, 16);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
