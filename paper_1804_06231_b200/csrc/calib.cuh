// calib.cuh -- FP32 roofline calibration and the idealised
// full-mask interaction rate (the GPU analogue of PAPER.md Table 2, P:222-241:
// "one particle directly interacting with 2560 other particles without any
// distance checks").  Not on the hot path; exported via include/sph_calib.h.
#pragma once

#include "common.cuh"
#include "density.cuh"

namespace pvsph {

__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c)
{
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

constexpr int CALIB_CHAINS = 8;

// mode 0: FFMA, 8 independent chains per thread; 2 flops per FFMA.
__global__ void k_calib_ffma(float *out, int iters)
{
    float a[CALIB_CHAINS];
    float b = 0.999f + 1e-7f * threadIdx.x, c = 1e-3f;
#pragma unroll
    for (int k = 0; k < CALIB_CHAINS; ++k) a[k] = 0.5f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < CALIB_CHAINS; ++k) a[k] = fmaf(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < CALIB_CHAINS; ++k) s += a[k];
    if (s == 123.456f) out[0] = s;
}

// mode 1: FFMA2 (fma.rn.f32x2), 8 independent chains; 4 flops per FFMA2.
__global__ void k_calib_ffma2(float *out, int iters)
{
    unsigned long long a[CALIB_CHAINS];
    float2 bb = make_float2(0.999f + 1e-7f * threadIdx.x, 0.998f), cc = make_float2(1e-3f, 2e-3f);
    unsigned long long b = *reinterpret_cast<unsigned long long *>(&bb);
    unsigned long long c = *reinterpret_cast<unsigned long long *>(&cc);
#pragma unroll
    for (int k = 0; k < CALIB_CHAINS; ++k) {
        float2 t = make_float2(0.5f + k, 0.25f + k);
        a[k] = *reinterpret_cast<unsigned long long *>(&t);
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < CALIB_CHAINS; ++k) a[k] = f2_fma(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < CALIB_CHAINS; ++k) {
        float2 t = *reinterpret_cast<float2 *>(&a[k]);
        s += t.x + t.y;
    }
    if (s == 123.456f) out[0] = s;
}

// mode 2: full-mask interaction (Table 2 analogue): each thread is one i that
// interacts with CALIB_NJ shared-memory neighbours per pass, no distance check.
constexpr int CALIB_NJ = 256;

__global__ void k_calib_interact(float *out, int iters)
{
    __shared__ float4 sx[CALIB_NJ], sv[CALIB_NJ];
    for (int k = threadIdx.x; k < CALIB_NJ; k += blockDim.x) {
        float t = (float)k / CALIB_NJ;
        sx[k] = make_float4(0.01f * t, 0.02f * (1.f - t), 0.005f * t, 0.f);
        sv[k] = make_float4(t, -t, 0.5f * t, 1e-3f);
    }
    __syncthreads();
    IPart p;
    p.x = 0.0101f; p.y = 0.0102f; p.z = 0.0053f; p.h = 0.02f;
    p.vx = 0.3f; p.vy = -0.2f; p.vz = 0.1f; p.m = 1e-3f;
    p.Hinv = 1.0f / 0.05f; p.H2 = 0.0025f; p.Hd = 0.05f; p.slot = 0;
    p.u0 = p.u1 = p.u2 = 0.0;
    Acc a;
    acc_zero(a);
    for (int i = 0; i < iters; ++i)
        for (int k = 0; k < CALIB_NJ; ++k) {
            float4 q = sx[k];
            float dx = p.x - q.x, dy = p.y - q.y, dz = p.z - q.z;
            float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            interact(p, dx, dy, dz, r2, sv[k], a);
        }
    float s = a.rho + a.wc + a.srt + a.st + a.D + a.Rx + a.Ry + a.Rz + (float)a.nngb;
    if (s == 123.456f) out[0] = s;
}

}  // namespace pvsph
