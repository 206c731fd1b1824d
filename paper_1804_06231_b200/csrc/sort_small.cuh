// sort_small.cuh -- the small-cell tier of sph_sort_cells (P:92 sorted projections, P:102 the
// 13 directions), shared by k_sort_small (sort.cuh) and the fused build (k_stable_small<true>,
// build.cuh, sph_build_sort_cells).
#pragma once

#include "common.cuh"

namespace pvsph {

constexpr int SORT_SMALL = 32;

// r += (a < b) as a compare and a predicated add (the compiler's select form costs three
// instructions per comparison in the rank loops below)
__device__ __forceinline__ void count_lt(unsigned &r, unsigned a, unsigned b)
{
    asm("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}" : "+r"(r) : "r"(a), "r"(b));
}

// The same for a, b < 2^31 as the sign bit of a - b (IMAD.IADD on the FMA pipe + LEA.HI):
// mixing both forms spreads a rank loop over the FMA and ALU pipes (each takes one warp
// instruction every two cycles), where compare + predicated add alone keep the ALU pipe full.
__device__ __forceinline__ void count_lt_sign(unsigned &r, unsigned a, unsigned b)
{
    r += (a - b) >> 31;
}

#ifndef SORT_CNT_MODE
#define SORT_CNT_MODE 1          // 0: compare + add only; 1: alternate with the sign form; 2: sign form only
#endif
__device__ __forceinline__ void count_lt_k(int k, unsigned &r, unsigned a, unsigned b)
{
    if (SORT_CNT_MODE == 2 || (SORT_CNT_MODE == 1 && (k & 1))) count_lt_sign(r, a, b);
    else count_lt(r, a, b);
}

__device__ __forceinline__ void cell_corner(const DevGrid &g, long long cell, double corner[3])
{
    long long plane = (long long)g.ny * g.nz;
    int ixl = (int)(cell / plane);
    int iy = (int)((cell / g.nz) % g.ny);
    int iz = (int)(cell % g.nz);
    int ixg = wrap_i(ixl - g.ghost_x + g.x_lo, g.nc[0]);
    corner[0] = (double)ixg * g.cl[0];
    corner[1] = (double)iy * g.cl[1];
    corner[2] = (double)iz * g.cl[2];
}


// The ranking composite of one particle along direction d: quantised key (25 bits) << 5 |
// in-cell index; (u0, u1, u2) = position - fp32 cell corner.
__device__ __forceinline__ unsigned small_composite(float u0, float u1, float u2, int d, int idx, float scale,
                                                    float cmax_s)
{
    const int a0 = dir_component(d, 0), a1 = dir_component(d, 1), a2 = dir_component(d, 2);
    const int kd = (a0 != 0) + (a1 != 0) + (a2 != 0);
    const float inv = kd == 1 ? 1.0f : (kd == 2 ? 0.70710678118654752f : 0.57735026918962576f);
    const float key = ((float)a0 * u0 + (float)a1 * u1 + (float)a2 * u2) * inv;
    // quantised key: floor((key + cmax) scale) as one FFMA and a rounding conversion
    const int qk = min(max(__float2int_rd(fmaf(key, scale, cmax_s)), 0), 33554431);
    return ((unsigned)qk << 5) | (unsigned)idx;     // < 2^30 (count_lt_sign)
}

// The 13 lists of one cell of n <= 32 particles, one particle per lane (sph_sort_cells' small
// tier, also run inside the fused build, sph_build_sort_cells).  Lane l holds a particle p whose
// in-cell index is idx (l itself in k_sort_small; the stable rank in the fused build); fc: the
// fp32 corner of the cell.  All 13 directions are ranked in one pass over the cell:
// composite = quantised key (25 bits) << 5 | in-cell index (the slot order is the input order,
// so equal keys keep input order).  The fp32 key error (< 1e-6 C_l) and the quantum
// 2 sqrt(3) C_l / 2^25 (~1e-7 C_l) are far below the window margin delta = 2^-16 C_l (DESIGN.md
// §4.2); the density sweeps tolerate that much disorder.  S: the warp's 32 x 16 composites.
__device__ __forceinline__ void sort_small_lists(unsigned *S, uint16_t *ord, long long cap, int s0, int n, bool mine,
                                                 float4 p, int idx, const float fc[3], float scale, float cmax_s)
{
    const int lane = threadIdx.x & 31;
    // cell-local coordinates in fp32: x - fp32(corner) is exact (Sterbenz) unless both are
    // within a cell of 0, where the error is below ulp(C_l)
    const float u0 = p.x - fc[0], u1 = p.y - fc[1], u2 = p.z - fc[2];
    unsigned comp[SPH_NDIR];
#pragma unroll
    for (int d = 0; d < SPH_NDIR; ++d) {
        comp[d] = small_composite(u0, u1, u2, d, idx, scale, cmax_s);
        if (mine) S[lane * 16 + d] = comp[d];
    }
    __syncwarp();
    unsigned r[SPH_NDIR];
#pragma unroll
    for (int d = 0; d < SPH_NDIR; ++d) r[d] = 0;
    for (int m = 0; m < n; ++m) {
        const uint4 c0 = *reinterpret_cast<const uint4 *>(&S[m * 16 + 0]);
        const uint4 c1 = *reinterpret_cast<const uint4 *>(&S[m * 16 + 4]);
        const uint4 c2 = *reinterpret_cast<const uint4 *>(&S[m * 16 + 8]);
        const unsigned c12 = S[m * 16 + 12];
        count_lt_k(0, r[0], c0.x, comp[0]); count_lt_k(1, r[1], c0.y, comp[1]);
        count_lt_k(2, r[2], c0.z, comp[2]); count_lt_k(3, r[3], c0.w, comp[3]);
        count_lt_k(4, r[4], c1.x, comp[4]); count_lt_k(5, r[5], c1.y, comp[5]);
        count_lt_k(6, r[6], c1.z, comp[6]); count_lt_k(7, r[7], c1.w, comp[7]);
        count_lt_k(8, r[8], c2.x, comp[8]); count_lt_k(9, r[9], c2.y, comp[9]);
        count_lt_k(10, r[10], c2.z, comp[10]); count_lt_k(11, r[11], c2.w, comp[11]);
        count_lt_k(12, r[12], c12, comp[12]);
    }
    if (mine) {
#pragma unroll
        for (int d = 0; d < SPH_NDIR; ++d) ord[(long long)d * cap + s0 + r[d]] = (uint16_t)idx;
    }
    __syncwarp();
}

}  // namespace pvsph
