// sort.cuh -- sph_sort_cells: per-cell sorted projections along the 13
// directions ("projecting the particle positions ... sorted with respect
// to their position along this axis"; "13 distinct directions").
//
// Key of particle k in cell c along d: fp32( (x_k - corner_c) . d/|d| ),
// the difference and dot product in fp64.  Order: ascending
// key, ties by input index perm[k] -- deterministic whatever the slot order.
// Each list entry is the particle's in-cell index (uint16, include/sph.h).
//
// Small cells (n <= SORT_SMALL = 32): one warp per cell, one particle per lane,
// 32-bit composites (quantised fp32 key, in-cell index) ranked by counting.
// Cells of up to SORT_MED = 128: k_sort_mid, one warp per cell, same composites.
// Cells of up to SORT_W256 = 256: k_sort_warp256, a register bitonic sort per warp.
// Medium/huge cells: stable LSD radix sorts in shared memory (k_sort_radix).  Cells above
// SORT_HUGE_MAX: the same radix sort with its key/index buffers in global scratch (L2).
#pragma once

#include "common.cuh"
#include "radix.cuh"
#include "sort_small.cuh"

namespace pvsph {

constexpr int SORT_MED = 128;           // cells above: k_sort_warp256 (bitonic), k_sort_radix
constexpr int SORT_W256 = 256;          //   up to here: one warp per cell, in registers (k_sort_warp256)
constexpr int SORT_MED_MAX = 2048;      //   medium tier (k_sort_radix): 128 threads, 33 KB shared memory
#ifndef SORT_MED_THREADS
#define SORT_MED_THREADS 128
#endif
constexpr int SORT_MED_T = SORT_MED_THREADS;
constexpr int SORT_HUGE_MAX = 16384;    //   huge tier: 512 threads, 225 KB; above it chunked ranking again
#ifndef SORT_HUGE_THREADS
#define SORT_HUGE_THREADS 512
#endif
constexpr int SORT_HUGE_T = SORT_HUGE_THREADS;
constexpr int SORT_WARPS = 8;
constexpr int SORT_GIANT_T = 1024;
constexpr int SORT_DIR_GROUPS = 5;     // direction groups of the huge and giant tiers (k_sort_radix)      // cells above SORT_HUGE_MAX (k_sort_radix<GLOBAL>)

// Level passes: the list of cell j along direction d is read only when the
// neighbour of j at offset +d or -d holds home particles of this grid, and a cell with home
// particles reads its own list along DENSE_SELF_DIR (k_density_dense); need[j] collects those
// directions as a 13-bit mask.
__global__ void k_mark_needed(DevGrid g, const int *__restrict__ cell_nhome, int *__restrict__ need)
{
    const long long plane = (long long)g.ny * g.nz;
    for (long long cell = blockIdx.x * (long long)blockDim.x + threadIdx.x; cell < g.ncell;
         cell += (long long)gridDim.x * blockDim.x) {
        if (cell_nhome[cell] == 0) continue;
        atomicOr(&need[cell], 1 << DENSE_SELF_DIR);     // k_density_dense's self-cell sweep
        const int ixl = (int)(cell / plane), iy = (int)((cell / g.nz) % g.ny), iz = (int)(cell % g.nz);
        for (int ox = -1; ox <= 1; ++ox) {
            int jx = ixl + ox;
            if (g.ghost_x) {
                if (jx < 0 || jx >= g.nxl) continue;
            } else {
                jx = wrap_i(jx, g.nc[0]);
            }
            for (int oy = -1; oy <= 1; ++oy)
                for (int oz = -1; oz <= 1; ++oz) {
                    if (!(ox | oy | oz)) continue;
                    int sg;
                    const int d = canon_dir(ox, oy, oz, sg);
                    atomicOr(&need[((long long)jx * g.ny + wrap_i(iy + oy, g.ny)) * g.nz + wrap_i(iz + oz, g.nz)],
                             1 << d);
                }
        }
    }
}

__global__ void __launch_bounds__(SORT_WARPS * 32, 4) k_sort_small(DevGrid g, DevCells c, uint16_t *ord,
                                                                    long long cbeg, long long cend, int2 *big_items,
                                                                    int *big_count, int *huge_items, int *huge_count,
                                                                    int huge_cap, int *mid_items, int *mid_count,
                                                                    int *w256_items, int *w256_count,
                                                                    const int *__restrict__ need, bool small_done,
                                                                    int huge_ngrp)
{
    __shared__ unsigned sh[SORT_WARPS][32 * 16];          // [lane][16] composites per warp
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const float cmax = 1.7320508075688772f * (float)fmax(g.cl[0], fmax(g.cl[1], g.cl[2]));
    const float scale = 33554432.0f / (2.0f * cmax);         // 2^25 over the key range
    const float cmax_s = cmax * scale;
    // 32 cells per warp step: lane l reads cell base + l, then the warp walks the non-empty
    // ones (sparse fine grids of level passes are mostly empty cells)
    for (long long base = cbeg + ((long long)blockIdx.x * SORT_WARPS + w) * 32; base < cend;
         base += (long long)gridDim.x * SORT_WARPS * 32) {
        const long long mycell = base + lane;
        const int my_s0 = mycell < cend ? c.cell_start[mycell] : 0;
        int my_n = mycell < cend ? c.cell_start[mycell + 1] - my_s0 : 0;
        if (need && my_n > 0 && !need[mycell]) my_n = 0;     // lists never read on this level grid
        if (small_done && my_n <= SORT_SMALL) my_n = 0;     // sph_build_sort_cells: written by the build
        // each lane the fp32 corner of ITS cell, once per 32 cells (the cell -> (x, y, z)
        // divisions cost ~10 % of the warp's instructions when done per cell by every lane)
        float my_corner[3] = {0.f, 0.f, 0.f};
        if (my_n > 0 && my_n <= SORT_SMALL) {
            double cd[3];
            cell_corner(g, mycell, cd);
            my_corner[0] = (float)cd[0]; my_corner[1] = (float)cd[1]; my_corner[2] = (float)cd[2];
        }
        unsigned todo = __ballot_sync(0xffffffffu, my_n > 0);
      while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        const long long cell = base + j;
        const int s0 = __shfl_sync(0xffffffffu, my_s0, j);
        const int n = __shfl_sync(0xffffffffu, my_n, j);
        if (n > SORT_MED && n <= SORT_W256) {              // k_sort_warp256
            if (lane == 0) w256_items[atomicAdd(w256_count, 1)] = (int)cell;
            continue;
        }
        if (n > SORT_MED && n <= SORT_HUGE_MAX) {
            // medium cells from the front of the list, huge ones from the back (k_sort_radix)
            if (lane == 0) {
                if (n <= SORT_MED_MAX) {
                    huge_items[atomicAdd(&huge_count[0], 1)] = (int)cell;
                } else {
                    const int pos = atomicAdd(&huge_count[1], huge_ngrp);
                    for (int gi = 0; gi < huge_ngrp; ++gi) huge_items[huge_cap - 1 - (pos + gi)] = (int)cell | (gi << 28);
                }
            }
            continue;
        }
        if (n > SORT_SMALL && n <= SORT_MED) {             // k_sort_mid: one warp per cell
            if (lane == 0) mid_items[atomicAdd(mid_count, 1)] = (int)cell;
            continue;
        }
        if (n > SORT_SMALL) {                              // above SORT_HUGE_MAX: k_sort_radix<GLOBAL>
            if (lane == 0) {
                const int pos = atomicAdd(big_count, SORT_DIR_GROUPS);
                for (int gi = 0; gi < SORT_DIR_GROUPS; ++gi) big_items[pos + gi] = make_int2((int)cell, gi);
            }
            continue;
        }
        const float fc[3] = {__shfl_sync(0xffffffffu, my_corner[0], j), __shfl_sync(0xffffffffu, my_corner[1], j),
                             __shfl_sync(0xffffffffu, my_corner[2], j)};
        const bool mine = lane < n;
        const float4 p = mine ? c.xyzh[s0 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
        sort_small_lists(sh[w], ord, c.cap, s0, n, mine, p, lane, fc, scale, cmax_s);
        __syncwarp();
      }
    }
}

// One CTA per cell of SORT_W256 < n <= MAXN particles: for each direction a stable LSD radix
// sort in shared memory.  The key is the fp64-projected fp32 key (pv_key) quantised to 24 bits
// over the cell's key range [-sqrt(3) C_max, +sqrt(3) C_max] (quantum 2 sqrt(3) C_max / 2^24,
// ~2e-7 C_l: the disorder the density sweeps tolerate, DESIGN.md §4.2 R5, as the 25-bit keys
// of k_sort_small); equal keys keep the in-cell (input) order.  Three 8-bit passes.  Warp w
// owns the contiguous segment [w S, (w+1) S) of the current buffer; the counters are per
// (digit, warp), so one exclusive scan gives every warp its output offset per digit; the warp
// walks its segment 32 elements at a time, ranking each lane among its digit peers
// (__match_any_sync; RU batches in flight), so the scatter is stable.  The counters of the
// next pass are filled during this pass's scatter (the destination's segment is known there)
// and those of the first pass while the keys are computed: one sweep per pass.  Shared
// memory: keys and indices double-buffered (12 B per element) plus 2 x 256 x NW counters.
constexpr int radix_smem(int maxn, int t) { return maxn * 12 + 2 * 256 * (t / 32) * 4 + 64 * 4; }

// GLOBAL (cells above SORT_HUGE_MAX): the key and index buffers live in global scratch -- 12 B
// per particle at the cell's own slots of the build's record region, free once the build is
// done, so no allocation and no overlap between cells; they stay in L2 for a cell of up to
// 65535 -- and only the counters in shared memory.  Items: every ISTRIDE-th int.
constexpr int radix_smem_global(int t) { return 2 * 256 * (t / 32) * 4 + 64 * 4; }

// Direction groups: a cell's 13 directions may be split into ngrp groups sorted by different
// CTAs (the huge and giant tiers: a few big cells would otherwise leave most SMs idle while one
// CTA walks all 13 directions).  Group gi holds directions [13 gi / ngrp, 13 (gi + 1) / ngrp).
// Items: huge tier cell | gi << 28 (ngrp > 1 needs ncell < 2^28); giant tier (GLOBAL) int2
// (cell, gi), whose scratch is the gi-th 12-byte-per-slot stripe of the record region (ngrp <= 5:
// 5 x 12 B fit the 64-byte records).
template <int MAXN, int T, bool FROM_BACK, bool GLOBAL = false, int ISTRIDE = 1>
__global__ void __launch_bounds__(T) k_sort_radix(DevGrid g, DevCells c, uint16_t *ord, const int *items,
                                                 const int *count, int cap, const int *__restrict__ need,
                                                 unsigned *gscratch = nullptr, int ngrp = 1)
{
    constexpr int NW = T / 32;
    constexpr int NH = 256 * NW;                       // counters, [digit][warp]
    constexpr int HPT = NH / T;                        // per thread in the scan
    constexpr int RU = 4;                              // batches of 32 in flight per warp
    static_assert(NH % T == 0, "radix: 256 x warps must be a multiple of the threads");
    extern __shared__ unsigned rs[];
    unsigned *keyA = rs, *keyB = rs + MAXN;
    uint16_t *idxA = reinterpret_cast<uint16_t *>(rs + 2 * MAXN), *idxB = idxA + MAXN;
    unsigned *histA = GLOBAL ? rs : rs + 3 * MAXN;     // after the two u16 index arrays
    unsigned *histB = histA + NH;
    unsigned *wsum = histB + NH;                       // [0, 32) warp totals, [32, 64) offsets
    const int nitems = *count;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    const float cmax = 1.7320508075688772f * (float)fmax(g.cl[0], fmax(g.cl[1], g.cl[2]));
    const float scale = 16777216.0f / (2.0f * cmax);   // 2^24 over the key range
    const float cmax_s = cmax * scale;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const long long ii = (long long)ISTRIDE * (FROM_BACK ? cap - 1 - it : it);
        const int item = items[ii];
        const long long cell = GLOBAL || ngrp == 1 ? item : (item & 0x0fffffff);
        const int gi = GLOBAL ? items[ii + 1] : (ngrp == 1 ? 0 : (int)((unsigned)item >> 28));
        const int d_lo = SPH_NDIR * gi / ngrp, d_hi = SPH_NDIR * (gi + 1) / ngrp;
        const int s0 = c.cell_start[cell];
        const int n = c.cell_start[cell + 1] - s0;
        if (GLOBAL) {
            unsigned *base = gscratch + 3ll * s0 + 3ll * gi * c.cap;
            keyA = base;
            keyB = base + n;
            idxA = reinterpret_cast<uint16_t *>(base + 2 * n);
            idxB = idxA + n;
        }
        const int S = (n + NW - 1) / NW;
        const float invS = 1.0f / (float)S;            // segment of slot e: floor((e + 0.5) / S), exact here
        const int lo = min(n, w * S), hi = min(n, lo + S);
        double corner[3];
        cell_corner(g, cell, corner);
        const int mask = need ? need[cell] : 0x1fff;
        for (int d = d_lo; d < d_hi; ++d) {
            if (!((mask >> d) & 1)) continue;          // CTA-uniform
#pragma unroll
            for (int q = 0; q < HPT; ++q) histA[threadIdx.x * HPT + q] = 0u;
            __syncthreads();
            for (int e = threadIdx.x; e < n; e += T) {
                const float4 p = c.xyzh[s0 + e];
                const float key = pv_key((double)p.x - corner[0], (double)p.y - corner[1],
                                         (double)p.z - corner[2], d);
                const unsigned k = (unsigned)min(max(__float2int_rd(fmaf(key, scale, cmax_s)), 0), 16777215);
                keyA[e] = k;
                idxA[e] = (uint16_t)e;
                atomicAdd(&histA[(k & 255u) * NW + (int)(((float)e + 0.5f) * invS)], 1u);
            }
            unsigned *ks = keyA, *kd = keyB, *hc = histA, *hn = histB;
            uint16_t *is = idxA, *id = idxB;
#pragma unroll 1
            for (int shift = 0; shift < 24; shift += 8) {
                const bool more = shift < 16;
                __syncthreads();                        // counters of this pass complete, last scatter done
                unsigned loc[HPT], sum = 0u;
#pragma unroll
                for (int q = 0; q < HPT; ++q) { loc[q] = hc[threadIdx.x * HPT + q]; sum += loc[q]; }
                unsigned run = block_excl_scan<T>(sum, wsum, lane, w);
#pragma unroll
                for (int q = 0; q < HPT; ++q) {
                    hc[threadIdx.x * HPT + q] = run;
                    run += loc[q];
                    if (more) hn[threadIdx.x * HPT + q] = 0u;   // the last pass's offsets, free now
                }
                __syncthreads();
                for (int b = lo; b < hi; b += 32 * RU) {
                    unsigned k[RU], dg[RU], peers[RU];
                    uint16_t ix[RU];
#pragma unroll
                    for (int u = 0; u < RU; ++u) {
                        const int i = b + 32 * u + lane;
                        k[u] = i < hi ? ks[i] : 0u;
                        ix[u] = i < hi ? is[i] : (uint16_t)0;
                        dg[u] = i < hi ? (k[u] >> shift) & 255u : 256u;   // 256: past the segment
                    }
#pragma unroll
                    for (int u = 0; u < RU; ++u) peers[u] = __match_any_sync(0xffffffffu, dg[u]);
#pragma unroll
                    for (int u = 0; u < RU; ++u) {
                        // batches in order: each reads its digit's running offset, scatters, and
                        // the digit's lowest lane advances the offset before the next batch reads
                        const unsigned r = __popc(peers[u] & lt_mask);
                        const unsigned hx = min(dg[u], 255u) * NW + w;
                        const unsigned base = hc[hx];
                        if (dg[u] < 256u) {
                            const unsigned pos = base + r;
                            kd[pos] = k[u];
                            id[pos] = ix[u];
                            if (more)
                                atomicAdd(&hn[((k[u] >> (shift + 8)) & 255u) * NW + (int)(((float)pos + 0.5f) * invS)], 1u);
                        }
                        __syncwarp();
                        if (dg[u] < 256u && r == 0) hc[hx] = base + __popc(peers[u]);
                        __syncwarp();
                    }
                }
                unsigned *tk = ks; ks = kd; kd = tk;
                uint16_t *ti = is; is = id; id = ti;
                unsigned *th = hc; hc = hn; hn = th;
            }
            __syncthreads();
            for (int k = threadIdx.x; k < n; k += T) ord[(long long)d * c.cap + s0 + k] = is[k];
            __syncthreads();
        }
    }
}

// Cells of SORT_MED < n <= SORT_W256 particles: one warp per cell, bitonic sort of 64-bit
// composites (orderable fp32 key << 32 | in-cell index) over P = 256 elements held in registers (lane l holds elements
// 8 l .. 8 l + 7): exchanges at distance j < 8 inside the lane, j >= 8 by warp shuffles; no
// shared memory, no barrier, eight cells per CTA at a time.
__global__ void __launch_bounds__(SORT_WARPS * 32) k_sort_warp256(DevGrid g, DevCells c, uint16_t *ord,
                                                                   const int *__restrict__ items,
                                                                   const int *__restrict__ count,
                                                                   const int *__restrict__ need)
{
    constexpr int E = SORT_W256 / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nitems = *count;
    for (int it = blockIdx.x * SORT_WARPS + w; it < nitems; it += gridDim.x * SORT_WARPS) {
        const long long cell = items[it];
        const int s0 = c.cell_start[cell];
        const int n = c.cell_start[cell + 1] - s0;
        double corner[3];
        cell_corner(g, cell, corner);
        const int mask = need ? need[cell] : 0x1fff;
        float4 p[E];
#pragma unroll
        for (int q = 0; q < E; ++q) {
            const int e = lane * E + q;
            p[q] = e < n ? c.xyzh[s0 + e] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll 1
        for (int d = 0; d < SPH_NDIR; ++d) {
            if (!((mask >> d) & 1)) continue;              // warp-uniform
            unsigned long long v[E];
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int e = lane * E + q;
                const float key = pv_key((double)p[q].x - corner[0], (double)p[q].y - corner[1],
                                         (double)p[q].z - corner[2], d);
                v[q] = e < n ? ((unsigned long long)float_order(key) << 32) | (unsigned)e : ~0ull;
            }
#pragma unroll
            for (int k = 2; k <= SORT_W256; k <<= 1) {
#pragma unroll
                for (int j = k >> 1; j > 0; j >>= 1) {
                    if (j >= E) {
#pragma unroll
                        for (int q = 0; q < E; ++q) {
                            const int i = lane * E + q, l = i ^ j;
                            const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[q], j / E);
                            const bool lo = ((i & k) == 0) == (i < l);
                            v[q] = lo ? (o < v[q] ? o : v[q]) : (o > v[q] ? o : v[q]);
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < E; ++q) {
                            if (q & j) continue;
                            const int i = lane * E + q;
                            const unsigned long long a = v[q], b = v[q + j];
                            const bool sw = ((i & k) == 0) ? (a > b) : (a < b);
                            v[q] = sw ? b : a;
                            v[q + j] = sw ? a : b;
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < E; ++q) {
                const int e = lane * E + q;
                if (e < n) ord[(long long)d * c.cap + s0 + e] = (uint16_t)(v[q] & 0xffffffffull);
            }
        }
    }
}

// Cells of SORT_SMALL < n <= SORT_MED particles: one warp per cell, up to four particles per
// lane, 31-bit composites (24-bit quantised key << 7 | in-cell index, n <= 128) of one
// direction at a time in shared memory, ranked by counting.
constexpr int SORT_MID_PER = SORT_MED / 32;

__global__ void __launch_bounds__(SORT_WARPS * 32) k_sort_mid(DevGrid g, DevCells c, uint16_t *ord,
                                                               const int *__restrict__ mid_items,
                                                               const int *__restrict__ mid_count,
                                                               const int *__restrict__ need)
{
    __shared__ unsigned sh[SORT_WARPS][SORT_MED];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned *S = sh[w];
    const int nitems = *mid_count;
    const float cmax = 1.7320508075688772f * (float)fmax(g.cl[0], fmax(g.cl[1], g.cl[2]));
    const float scale = 16777216.0f / (2.0f * cmax);   // 24-bit keys: composites < 2^31 (count_lt_sign)
    const float cmax_s = cmax * scale;
    for (int it = blockIdx.x * SORT_WARPS + w; it < nitems; it += gridDim.x * SORT_WARPS) {
        const long long cell = mid_items[it];
        const int s0 = c.cell_start[cell];
        const int n = c.cell_start[cell + 1] - s0;
        const int mask = need ? need[cell] : 0x1fff;
        double corner[3];
        cell_corner(g, cell, corner);
        float u[SORT_MID_PER][3];
#pragma unroll
        for (int k = 0; k < SORT_MID_PER; ++k) {
            const int e = lane + 32 * k;
            const float4 p = e < n ? c.xyzh[s0 + e] : make_float4(0.f, 0.f, 0.f, 0.f);
            // as k_sort_small: x - fp32(corner) in fp32
            u[k][0] = p.x - (float)corner[0];
            u[k][1] = p.y - (float)corner[1];
            u[k][2] = p.z - (float)corner[2];
        }
#pragma unroll 1
        for (int d = 0; d < SPH_NDIR; ++d) {
            if (!((mask >> d) & 1)) continue;              // warp-uniform
            const int a0 = dir_component(d, 0), a1 = dir_component(d, 1), a2 = dir_component(d, 2);
            const int kd = (a0 != 0) + (a1 != 0) + (a2 != 0);
            const float inv = kd == 1 ? 1.0f : (kd == 2 ? 0.70710678118654752f : 0.57735026918962576f);
            unsigned comp[SORT_MID_PER];
#pragma unroll
            for (int k = 0; k < SORT_MID_PER; ++k) {
                const int e = lane + 32 * k;
                const float key = ((float)a0 * u[k][0] + (float)a1 * u[k][1] + (float)a2 * u[k][2]) * inv;
                const int qk = min(max(__float2int_rd(fmaf(key, scale, cmax_s)), 0), 16777215);
                comp[k] = ((unsigned)qk << 7) | (unsigned)e;
                if (e < n) S[e] = comp[k];
            }
            __syncwarp();
            unsigned r[SORT_MID_PER] = {0, 0, 0, 0};
            for (int m = 0; m < n; ++m) {
                const unsigned v = S[m];
#pragma unroll
                for (int k = 0; k < SORT_MID_PER; ++k) count_lt_k(k, r[k], v, comp[k]);
            }
#pragma unroll
            for (int k = 0; k < SORT_MID_PER; ++k) {
                const int e = lane + 32 * k;
                if (e < n) ord[(long long)d * c.cap + s0 + r[k]] = (uint16_t)e;
            }
            __syncwarp();
        }
    }
}

}  // namespace pvsph
