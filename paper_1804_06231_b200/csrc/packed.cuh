// packed.cuh -- two fp32 lanes in one 64-bit register pair, computed with the
// sm_100 packed instructions FFMA2 / FADD2 / FMUL2 (PTX add/sub/mul/fma .f32x2).
// One packed instruction issues once and does the work of two scalar ones.
#pragma once

namespace pvsph {

// Packed pair of fp32 lanes: float2 with the sm_100 FFMA2/FADD2/FMUL2 intrinsics, so that
// the register allocator sees real pairs (no 64-bit inline-asm copies).
typedef float2 f2;

__device__ __forceinline__ f2 pk(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ void upk(f2 v, float &a, float &b)
{
    a = v.x;
    b = v.y;
}
__device__ __forceinline__ f2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ f2 add2(f2 a, f2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ f2 sub2(f2 a, f2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { return __ffma2_rn(a, b, c); }
// acc += a * b and acc += a
__device__ __forceinline__ void acc_fma2(f2 &acc, f2 a, f2 b) { acc = __ffma2_rn(a, b, acc); }
__device__ __forceinline__ void acc_add2(f2 &acc, f2 a) { acc = __fadd2_rn(acc, a); }
// 1/sqrt(x) for normal x > 0 (MUFU.RSQ, no denormal fix-up; callers clamp x >= 1e-30)
__device__ __forceinline__ float rsqrt_fast(float x)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// rsqrt refined by one Newton step, y (3/2 - x y^2 / 2): ~1 ulp instead of MUFU.RSQ's ~2
// (R14: near the cut-off w' amplifies the rounding of x = r/H)
__device__ __forceinline__ float rsqrt_nr(float x)
{
    const float y = rsqrt_fast(x);
    return y * fmaf(-0.5f * x * y, y, 1.5f);
}
__device__ __forceinline__ f2 rsqrt_nr2(f2 x)
{
    const f2 y = make_float2(rsqrt_fast(x.x), rsqrt_fast(x.y));
    const f2 t = __ffma2_rn(__fmul2_rn(x, make_float2(-0.5f, -0.5f)), __fmul2_rn(y, y), make_float2(1.5f, 1.5f));
    return __fmul2_rn(y, t);
}
__device__ __forceinline__ float sum2(f2 v) { return v.x + v.y; }
__device__ __forceinline__ f2 zero2() { return make_float2(0.0f, 0.0f); }

}  // namespace pvsph

namespace pvsph {

// 32-bit shared-memory addressing (avoids generic-pointer window arithmetic in hot loops).
__device__ __forceinline__ unsigned smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float4 lds_f4(unsigned a)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned lds_u16(unsigned a)
{
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
// Loads of shared data that is read-only while the warp computes (no volatile: the
// compiler may schedule them early; their addresses derive from values loaded after
// the staging barrier, which anchors them after it).
__device__ __forceinline__ float4 ldsr_f4(unsigned a)
{
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
// the same with a constant byte offset folded into the instruction ([reg + imm])
template <unsigned OFF>
__device__ __forceinline__ float4 ldsr_f4_at(unsigned a)
{
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a), "n"(OFF));
    return v;
}
__device__ __forceinline__ unsigned ldsr_u16(unsigned a)
{
    unsigned short v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned lds_u32(unsigned a)
{
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
// mbarrier + bulk copy (the TMA engine's 1-D form): global -> shared without registers.
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned a, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void *src, unsigned bytes, unsigned mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void sts_u16(unsigned a, unsigned v)
{
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
// push onto a hit stack: volatile (ordered against the volatile pops), but no memory clobber,
// so the read-only staged loads around it can still be scheduled freely
__device__ __forceinline__ void sts_u16_push(unsigned a, unsigned v)
{
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v));
}
__device__ __forceinline__ void sts_u32(unsigned a, unsigned v)
{
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

}  // namespace pvsph
