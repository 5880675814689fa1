// Packed FP32 pairs for the pair loops (sm_100a FFMA2 / FMUL2 / FADD2).
//
// Every P2P-like loop here is issue bound, not FMA bound: one pair of U+P costs ~37 FP32
// instructions plus the rsqrt and the shared-memory reads, and ncu showed ~80% issue with the
// FMA pipe ~60% busy.  sm_100a executes two fp32 lanes per instruction (FFMA2 & co., measured
// at the same 72-73 TFLOP/s as scalar FFMA), so evaluating TWO targets per instruction against
// the same source (the source operand a broadcast `.F32` register) halves the FP32 issue slots
// per pair while the arithmetic per target is unchanged (the same operations in the same
// order; only where the scalar build contracted a separate multiply and add into one FFMA can
// the last bit differ).
//
// F2 is a float2 with the arithmetic operators the kernel templates of elastic.cuh use, so
// acc_U / acc_P / acc_UP / acc_D / acc_S / acc_DS instantiate for it unchanged.
#pragma once
#include <cuda_runtime.h>

namespace ebem {

struct F2 {
    float2 v;
    F2() = default;
    __device__ __forceinline__ F2(float2 x) : v(x) {}
    __device__ __forceinline__ explicit F2(float s) : v(make_float2(s, s)) {}   // broadcast
    __device__ __forceinline__ F2(float a, float b) : v(make_float2(a, b)) {}
};

__device__ __forceinline__ F2 operator+(F2 a, F2 b) { return F2(__fadd2_rn(a.v, b.v)); }
__device__ __forceinline__ F2 operator-(F2 a) { return F2(make_float2(-a.v.x, -a.v.y)); }
__device__ __forceinline__ F2 operator-(F2 a, F2 b) { return F2(__fadd2_rn(a.v, make_float2(-b.v.x, -b.v.y))); }
__device__ __forceinline__ F2 operator*(F2 a, F2 b) { return F2(__fmul2_rn(a.v, b.v)); }
__device__ __forceinline__ F2& operator+=(F2& a, F2 b) { return a = a + b; }
__device__ __forceinline__ F2 fmat(F2 a, F2 b, F2 c) { return F2(__ffma2_rn(a.v, b.v, c.v)); }

// rsqrt per lane (MUFU is scalar)
__device__ __forceinline__ F2 rsqrt2(F2 x) { return F2(rsqrtf(x.v.x), rsqrtf(x.v.y)); }
// r = 0 excluded (reading R8): the own panel belongs to the local pass
__device__ __forceinline__ F2 safe_rinv2(F2 r2) {
    const float a = rsqrtf(r2.v.x), b = rsqrtf(r2.v.y);
    return F2(r2.v.x > 0.f ? a : 0.f, r2.v.y > 0.f ? b : 0.f);
}

}  // namespace ebem
