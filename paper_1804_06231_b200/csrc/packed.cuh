// packed.cuh -- two fp32 lanes in one 64-bit register pair, computed with the
// sm_100 packed instructions FFMA2 / FADD2 / FMUL2 (PTX add/sub/mul/fma .f32x2).
// One packed instruction issues once and does the work of two scalar ones.
#pragma once

namespace pvsph {

typedef unsigned long long f2;

__device__ __forceinline__ f2 pk(float a, float b)
{
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk(f2 v, float &a, float &b)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2 as_f2(float2 v) { return pk(v.x, v.y); }
__device__ __forceinline__ f2 bc2(float a) { return pk(a, a); }
__device__ __forceinline__ f2 add2(f2 a, f2 b)
{
    f2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b)
{
    f2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b)
{
    f2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c)
{
    f2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// acc += a * b and acc += a, updating the accumulator register pair in place
__device__ __forceinline__ void acc_fma2(f2 &acc, f2 a, f2 b)
{
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ void acc_add2(f2 &acc, f2 a)
{
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(a));
}
// 1/sqrt(x) for normal x > 0 (MUFU.RSQ, no denormal fix-up; callers clamp x >= 1e-30)
__device__ __forceinline__ float rsqrt_fast(float x)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sum2(f2 v)
{
    float a, b;
    upk(v, a, b);
    return a + b;
}

}  // namespace pvsph
