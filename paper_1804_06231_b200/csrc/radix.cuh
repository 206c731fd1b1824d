// radix.cuh -- block-wide helpers of the shared-memory LSD radix sorts (k_sort_radix in
// sort.cuh, k_stable_radix in build.cuh).
#pragma once

namespace pvsph {

// Exclusive prefix sum over the T threads of a CTA (T / 32 <= 32 warps); wsum: 64 words of
// shared memory ([0, 32) warp totals, [32, 64) warp offsets).  Two barriers.
template <int T>
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned *wsum, int lane, int w)
{
    constexpr int NW = T / 32;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned s = lane < NW ? wsum[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < NW) wsum[32 + lane] = s - wsum[lane];      // exclusive warp offsets
    }
    __syncthreads();
    return wsum[32 + w] + x - v;
}

}  // namespace pvsph
