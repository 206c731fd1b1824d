// bitonic.cuh -- register-resident bitonic stages shared by the sort tiers (sort.cuh) and the
// build's stable in-cell reorder of large cells (build.cuh).  A warp holds a 256-element chunk
// of 64-bit composites, 8 per lane (element i = base + 8 lane + q).
#pragma once

namespace pvsph {

constexpr int BT_CHUNK = 256;
constexpr int BT_E = BT_CHUNK / 32;

// Bitonic stages j = J0, J0/2, ..., 1 of merge size k on the warp's chunk in registers
// (element index i = base + 8 lane + q).
template <int J0>
__device__ __forceinline__ void bt_reg_stages(unsigned long long (&v)[BT_E], int base, int lane, int k)
{
#pragma unroll
    for (int j = J0; j > 0; j >>= 1) {
        if (j >= BT_E) {
#pragma unroll
            for (int q = 0; q < BT_E; ++q) {
                const int i = base + lane * BT_E + q, l = i ^ j;
                const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[q], j / BT_E);
                const bool lo = ((i & k) == 0) == (i < l);
                v[q] = lo ? (o < v[q] ? o : v[q]) : (o > v[q] ? o : v[q]);
            }
        } else {
#pragma unroll
            for (int q = 0; q < BT_E; ++q) {
                if (q & j) continue;
                const int i = base + lane * BT_E + q;
                const unsigned long long a = v[q], b = v[q + j];
                const bool sw = ((i & k) == 0) ? (a > b) : (a < b);
                v[q] = sw ? b : a;
                v[q + j] = sw ? a : b;
            }
        }
    }
}

// The chunk sorted whole (merge sizes k = 2 .. 256), directions from the global index.
__device__ __forceinline__ void bt_sort_chunk(unsigned long long (&v)[BT_E], int base, int lane)
{
    bt_reg_stages<1>(v, base, lane, 2);
    bt_reg_stages<2>(v, base, lane, 4);
    bt_reg_stages<4>(v, base, lane, 8);
    bt_reg_stages<8>(v, base, lane, 16);
    bt_reg_stages<16>(v, base, lane, 32);
    bt_reg_stages<32>(v, base, lane, 64);
    bt_reg_stages<64>(v, base, lane, 128);
    bt_reg_stages<128>(v, base, lane, 256);
}

// Merge sizes k = 512 .. P of a CTA-wide bitonic sort of hs[0, P) (P a power of two >= 512,
// every chunk already sorted by bt_sort_chunk and stored): distances j >= 256 through shared
// memory (a barrier each), the last eight in registers.  Ends with a barrier.
template <int T>
__device__ __forceinline__ void bt_cta_merge(unsigned long long *hs, int P, int lane, int w)
{
    constexpr int NW = T / 32;
    for (int k = 2 * BT_CHUNK; k <= P; k <<= 1) {
        for (int j = k >> 1; j >= BT_CHUNK; j >>= 1) {
            __syncthreads();
            for (int pi = threadIdx.x; pi < P / 2; pi += T) {
                const int i = (pi / j) * 2 * j + (pi % j), l = i + j;
                const unsigned long long a = hs[i], b = hs[l];
                const bool sw = ((i & k) == 0) ? (a > b) : (a < b);
                if (sw) {
                    hs[i] = b;
                    hs[l] = a;
                }
            }
        }
        __syncthreads();
        for (int ch = w; ch < P / BT_CHUNK; ch += NW) {
            const int base = ch * BT_CHUNK;
            unsigned long long v[BT_E];
#pragma unroll
            for (int q = 0; q < BT_E; ++q) v[q] = hs[base + lane * BT_E + q];
            bt_reg_stages<128>(v, base, lane, k);
#pragma unroll
            for (int q = 0; q < BT_E; ++q) hs[base + lane * BT_E + q] = v[q];
        }
    }
    __syncthreads();
}

}  // namespace pvsph
