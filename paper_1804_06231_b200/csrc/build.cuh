// build.cuh -- sph_build_cells: cell binning as a counting sort.
//
//   k_bin          : validate, fp64 bin, atomic slot rank within the cell
//   k_scan_*       : exclusive scan of the per-cell counts -> cell_start
//   k_scatter_rec  : the particle's 64-byte record (x, y, z, h, vx, vy, vz, m,
//                    input index) to slot cell_start[cell] + rank (two full
//                    sectors per particle: no read-modify-write at random slots)
//   k_stable_*     : per cell, sort the records by input index (the atomic ranks
//                    arrive in any order) -> xyzh, vm, perm, slot_cell with the
//                    in-cell order = input order, all reads/writes coalesced
//
// Stable in-cell order makes everything downstream deterministic and, with
// slab ghosts received in the sender's cell order, identical across GPU
// counts.  HBM traffic per particle ~ 32 (read) + 8
// (cell/rank) + 40 (re-read) + 64 (scattered 64-byte record: two full sectors) +
// 64 (stable read) + 40 (write) ~ 250 B (random-access granularity).
#pragma once

#include "common.cuh"
#include "radix.cuh"
#include "sort_small.cuh"

namespace pvsph {

// The binning rule of one particle: its local cell, or -1 (rejected: status set, or a ghost
// outside this grid's ghost planes).
__device__ __forceinline__ int bin_cell(const DevGrid &g, long long n_own, long long p, float4 a, float4 b,
                                        double clmin, unsigned *status)
{
    bool finite = isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w) && isfinite(b.x) &&
                  isfinite(b.y) && isfinite(b.z) && isfinite(b.w);
    if (!finite) {
        set_status(status, ST_EDOMAIN);
        return -1;
    }
    if (!(a.w > 0.0f) || !(b.w > 0.0f) ||
        (is_home(g.h_home_min, g.h_home_max, a.w) && (double)g.gamma * (double)a.w + 2.0 * (double)g.skin > clmin)) {
        // (a neighbour-only particle of a level pass may have gamma h > C_l)
        set_status(status, ST_EH_RANGE);
        return -1;
    }
    double x[3] = {a.x, a.y, a.z};
    int ic[3];
    bool inside = true;
    for (int k = 0; k < 3; ++k) {
        if (!(x[k] >= 0.0 && x[k] < g.box[k])) inside = false;
        int c = (int)floor(x[k] * (double)g.nc[k] / g.box[k]);
        ic[k] = c < 0 ? 0 : (c > g.nc[k] - 1 ? g.nc[k] - 1 : c);
    }
    int ixl = -1;
    if (inside) {
        if (p < n_own) {
            if (ic[0] >= g.x_lo && ic[0] < g.x_hi) ixl = ic[0] - g.x_lo + g.ghost_x;
        } else if (g.ghost_x) {
            if (ic[0] == wrap_i(g.x_lo - 1, g.nc[0])) ixl = 0;
            else if (ic[0] == wrap_i(g.x_hi, g.nc[0])) ixl = g.nxl - 1;
        }
    }
    if (ixl < 0) {
        // a ghost outside the ghost planes is not needed on this grid (a finer level
        // grid keeps only its own thinner ghost planes): dropped; anything else is an error
        if (!(inside && p >= n_own && g.ghost_x)) set_status(status, ST_EDOMAIN);
        return -1;
    }
    return (ixl * g.ny + ic[1]) * g.nz + ic[2];
}

#ifndef BIN_U
#define BIN_U 2        // particles per thread and step: loads, then atomics, then stores (A/B c5: 1 / 2 / 4 -> build + sort 18.29 / 18.22 / 18.22 ms)
#endif
__global__ void k_bin(DevGrid g, long long n_own, long long n_total, const float4 *__restrict__ xyzh_in,
                      const float4 *__restrict__ vm_in, int *__restrict__ cell_of, int *__restrict__ rank,
                      int *__restrict__ count, unsigned *status)
{
    const double clmin = fmin(g.cl[0], fmin(g.cl[1], g.cl[2]));
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; p0 < n_total; p0 += BIN_U * stride) {
        float4 a[BIN_U], b[BIN_U];
        int cell[BIN_U], rk[BIN_U];
#pragma unroll
        for (int u = 0; u < BIN_U; ++u) {
            const long long p = p0 + u * stride;
            a[u] = p < n_total ? xyzh_in[p] : make_float4(0.f, 0.f, 0.f, 0.f);
            b[u] = p < n_total ? vm_in[p] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < BIN_U; ++u) {
            const long long p = p0 + u * stride;
            cell[u] = p < n_total ? bin_cell(g, n_own, p, a[u], b[u], clmin, status) : -1;
        }
#pragma unroll
        for (int u = 0; u < BIN_U; ++u) rk[u] = cell[u] >= 0 ? atomicAdd(&count[cell[u]], 1) : 0;
#pragma unroll
        for (int u = 0; u < BIN_U; ++u) {
            const long long p = p0 + u * stride;
            if (p >= n_total) continue;
            if (cell[u] >= 0) rank[p] = rk[u];
            cell_of[p] = cell[u];
        }
    }
}

// ---- three-phase exclusive scan of count[ncell] into start[ncell + 1] ------
constexpr int SCAN_T = 1024;          // threads per block
constexpr int SCAN_V = 4;             // values per thread
constexpr int SCAN_TILE = SCAN_T * SCAN_V;

__device__ __forceinline__ int block_exclusive_scan(int v, int *sh, int &total)
{
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        sh[lane] = s;
    }
    __syncthreads();
    int off = w ? sh[w - 1] : 0;
    total = sh[(blockDim.x >> 5) - 1];
    __syncthreads();
    return off + x - v;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_tiles(const int *count, long long n, int *start,
                                                        int *__restrict__ tile_sum, unsigned *status,
                                                        int vmax = SPH_MAX_CELL)
{
    __shared__ int sh[32];
    long long base = (long long)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_V;
    int v[SCAN_V];
    int s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_V; ++k) {
        v[k] = base + k < n ? count[base + k] : 0;
        if (v[k] > vmax) set_status(status, ST_ECAPACITY);
        s += v[k];
    }
    int total;
    int off = block_exclusive_scan(s, sh, total);
#pragma unroll
    for (int k = 0; k < SCAN_V; ++k) {
        if (base + k < n) start[base + k] = off;
        off += v[k];
    }
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

// Single block: exclusive scan of the tile sums in place; writes start[n] = total.
__global__ void __launch_bounds__(SCAN_T) k_scan_sums(int *__restrict__ tile_sum, long long ntiles,
                                                       int *__restrict__ start, long long n)
{
    __shared__ int sh[32];
    int carry = 0;
    for (long long b = 0; b < ntiles; b += SCAN_T) {
        long long i = b + threadIdx.x;
        int v = i < ntiles ? tile_sum[i] : 0;
        int total;
        int e = block_exclusive_scan(v, sh, total);
        if (i < ntiles) tile_sum[i] = carry + e;
        carry += total;
    }
    if (threadIdx.x == 0) start[n] = carry;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_add(int *__restrict__ start, long long n,
                                                      const int *__restrict__ tile_sum)
{
    int add = tile_sum[blockIdx.x];
    long long base = (long long)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_V;
#pragma unroll
    for (int k = 0; k < SCAN_V; ++k)
        if (base + k < n) start[base + k] += add;
}

// ---- ghost exchange helper (sph_select_planes) ----------------------------
// The owned particles of global plane x_lo (list 0) and x_hi - 1 (list 1), in input order.
// k_sel_count: per block of SEL_B particles, how many fall in each list (blk[list * nblk + b]);
// the three scan kernels turn that into offsets; k_sel_write recomputes the flags, ranks them
// inside the block (warp ballots + a block scan) and copies the particles.
constexpr int SEL_B = 1024;

__device__ __forceinline__ int sel_list(const DevGrid &g, float x)
{
    int c = (int)floor((double)x * (double)g.nc[0] / g.box[0]);   // the binning rule of k_bin
    c = c < 0 ? 0 : (c > g.nc[0] - 1 ? g.nc[0] - 1 : c);
    return c == g.x_lo ? 0 : (c == g.x_hi - 1 ? 1 : -1);
}

__global__ void __launch_bounds__(SEL_B) k_sel_count(DevGrid g, long long n, const float4 *__restrict__ xyzh,
                                                      int *__restrict__ blk, long long nblk)
{
    const long long p = blockIdx.x * (long long)SEL_B + threadIdx.x;
    const int l = p < n ? sel_list(g, xyzh[p].x) : -1;
    const int c0 = __syncthreads_count(l == 0), c1 = __syncthreads_count(l == 1);
    if (threadIdx.x == 0) {
        blk[blockIdx.x] = c0;
        blk[nblk + blockIdx.x] = c1;
    }
}

__global__ void __launch_bounds__(SEL_B) k_sel_write(DevGrid g, long long n, const float4 *__restrict__ xyzh,
                                                      const float4 *__restrict__ vm, const int *__restrict__ off,
                                                      long long nblk, float4 *sel_x, float4 *sel_v, long long cap,
                                                      long long *counts, unsigned *status)
{
    __shared__ int wsum[2][SEL_B / 32];
    const long long p = blockIdx.x * (long long)SEL_B + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int l = p < n ? sel_list(g, xyzh[p].x) : -1;
    const unsigned b0 = __ballot_sync(0xffffffffu, l == 0), b1 = __ballot_sync(0xffffffffu, l == 1);
    if (lane == 0) {
        wsum[0][w] = __popc(b0);
        wsum[1][w] = __popc(b1);
    }
    __syncthreads();
    if (l >= 0) {
        int before = 0;
        for (int k = 0; k < w; ++k) before += wsum[l][k];
        const unsigned mine = l == 0 ? b0 : b1;
        const long long total0 = off[nblk];                            // particles of list 0
        const long long base = l == 0 ? off[blockIdx.x] : (long long)off[nblk + blockIdx.x] - total0;
        const long long r = base + before + __popc(mine & ((1u << lane) - 1u));
        if (r < cap) {
            sel_x[l * cap + r] = xyzh[p];
            sel_v[l * cap + r] = vm[p];
        } else {
            set_status(status, ST_ECAPACITY);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        counts[0] = off[nblk];
        counts[1] = (long long)off[2 * nblk] - off[nblk];
    }
}

// ---- slab migration on a reuse rebuild (sph_partition_migrants / sph_merge_by_id) --------
// List 0: the owned particles whose (wrapped) x plane is the left neighbour's last plane
// x_lo - 1, list 1: the right neighbour's first plane x_hi, list 2: the rest; each in input
// order (a stable three-way partition, the scheme of k_sel_count / k_sel_write).
__device__ __forceinline__ int mig_list(const DevGrid &g, float x)
{
    int c = (int)floor((double)x * (double)g.nc[0] / g.box[0]);   // the binning rule of k_bin
    c = c < 0 ? 0 : (c > g.nc[0] - 1 ? g.nc[0] - 1 : c);
    const int lo = (g.x_lo - 1 + g.nc[0]) % g.nc[0], hi = g.x_hi % g.nc[0];
    return c == lo ? 0 : (c == hi ? 1 : 2);
}

__global__ void __launch_bounds__(SEL_B) k_mig_count(DevGrid g, long long n, const float4 *__restrict__ xyzh,
                                                      int *__restrict__ blk, long long nblk)
{
    const long long p = blockIdx.x * (long long)SEL_B + threadIdx.x;
    const int l = p < n ? mig_list(g, xyzh[p].x) : -1;
    const int c0 = __syncthreads_count(l == 0), c1 = __syncthreads_count(l == 1), c2 = __syncthreads_count(l == 2);
    if (threadIdx.x == 0) {
        blk[blockIdx.x] = c0;
        blk[nblk + blockIdx.x] = c1;
        blk[2 * nblk + blockIdx.x] = c2;
    }
}

struct MigOut {
    float4 *x[3], *v[3];
    long long *g[3];
    long long cap[3];
};

__global__ void __launch_bounds__(SEL_B) k_mig_write(DevGrid g, long long n, const float4 *__restrict__ xyzh,
                                                      const float4 *__restrict__ vm, const long long *__restrict__ gid,
                                                      const int *__restrict__ off, long long nblk, MigOut o,
                                                      long long *counts, unsigned *status)
{
    __shared__ int wsum[3][SEL_B / 32];
    const long long p = blockIdx.x * (long long)SEL_B + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int l = p < n ? mig_list(g, xyzh[p].x) : -1;
    unsigned b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) b[k] = __ballot_sync(0xffffffffu, l == k);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) wsum[k][w] = __popc(b[k]);
    }
    __syncthreads();
    if (l >= 0) {
        int before = 0;
        for (int k = 0; k < w; ++k) before += wsum[l][k];
        const unsigned mine = l == 0 ? b[0] : (l == 1 ? b[1] : b[2]);
        const long long base = (long long)off[l * nblk + blockIdx.x] - (l > 0 ? (long long)off[l * nblk] : 0ll);
        const long long r = base + before + __popc(mine & ((1u << lane) - 1u));
        if (r < o.cap[l]) {
            o.x[l][r] = xyzh[p];
            o.v[l][r] = vm[p];
            o.g[l][r] = gid[p];
        } else {
            set_status(status, ST_ECAPACITY);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        counts[0] = off[nblk];
        counts[1] = (long long)off[2 * nblk] - off[nblk];
        counts[2] = (long long)off[3 * nblk] - off[2 * nblk];
    }
}

// Merge of three lists, each ascending in id, ids distinct across them: element i of list L
// goes to i + (elements of the other two lists with a smaller id), found by binary search.
__device__ __forceinline__ long long lower_bound_id(const long long *a, long long n, long long key)
{
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long m = (lo + hi) >> 1;
        if (a[m] < key) lo = m + 1;
        else hi = m;
    }
    return lo;
}

struct MergeIn {
    const float4 *x[3], *v[3];
    const long long *g[3];
    long long n[3];
};

__global__ void k_merge_by_id(MergeIn in, float4 *__restrict__ ox, float4 *__restrict__ ov, long long *__restrict__ og)
{
    const long long total = in.n[0] + in.n[1] + in.n[2];
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int l = t < in.n[0] ? 0 : (t < in.n[0] + in.n[1] ? 1 : 2);
        const long long i = t - (l > 0 ? in.n[0] : 0) - (l > 1 ? in.n[1] : 0);
        const long long key = in.g[l][i];
        long long pos = i;
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (k != l) pos += lower_bound_id(in.g[k], in.n[k], key);
        ox[pos] = in.x[l][i];
        ov[pos] = in.v[l][i];
        og[pos] = key;
    }
}

// 64-byte scatter record: the particle's 8 floats and its input index, written as two full
// 32-byte sectors (two 256-bit stores) so a random slot costs no read-modify-write.
struct alignas(64) ParticleRec {
    float4 xyzh, vm;
    int idx, pad[7];
};

#ifndef SCATTER_U
#define SCATTER_U 2    // particles per thread and step, loads issued before the stores (A/B c5: 1 / 2 / 4 -> build + sort 18.43 / 18.27 / 18.39 ms)
#endif
__global__ void k_scatter_rec(DevGrid g, long long n_total, const int *__restrict__ cell_of, const int *__restrict__ rank,
                              const int *__restrict__ start, const float4 *__restrict__ xyzh_in,
                              const float4 *__restrict__ vm_in, ParticleRec *__restrict__ rec)
{
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; p0 < n_total; p0 += SCATTER_U * stride) {
        int c[SCATTER_U], slot[SCATTER_U];
        float4 a[SCATTER_U], b[SCATTER_U];
#pragma unroll
        for (int u = 0; u < SCATTER_U; ++u) {
            const long long p = p0 + u * stride;
            c[u] = p < n_total ? __ldcs(cell_of + p) : -1;      // c < 0: rejected input, no slot
        }
#pragma unroll
        for (int u = 0; u < SCATTER_U; ++u) {
            const long long p = p0 + u * stride;
            if (c[u] >= 0) {
                slot[u] = start[c[u]] + __ldcs(rank + p);
                a[u] = __ldcs(xyzh_in + p);
                b[u] = __ldcs(vm_in + p);
            }
        }
#pragma unroll
        for (int u = 0; u < SCATTER_U; ++u) {
            if (c[u] < 0) continue;
            const long long p = p0 + u * stride;
            // one 256-bit store (STG.256): the whole 32-byte sector at once, no read-modify-write
            // (evict-first: the scattered stream must not push cell_start out of L2)
            asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(rec + slot[u]),
                         "f"(a[u].x), "f"(a[u].y), "f"(a[u].z), "f"(a[u].w), "f"(b[u].x), "f"(b[u].y), "f"(b[u].z),
                         "f"(b[u].w)
                         : "memory");
            // key of the in-cell order: home particles first, each group in input order
            const unsigned key = (unsigned)p | (is_home(g.h_home_min, g.h_home_max, a[u].w) ? 0u : 0x80000000u);
            asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %2, %2, %2, %2, %2, %2};" ::"l"(&rec[slot[u]].idx),
                         "r"(key), "r"(0)
                         : "memory");
        }
    }
}

// sph_drift: x <- fp32(x + fp32(v dt)) per component for every stored particle (list reuse,
// P:102).  Per particle the exact stored increment x_new - x_old (fp32 subtraction
// of nearby values: exact) is accumulated in disp[s] (its norm rounded up by 1e-6 relative, so
// disp bounds |x - x_build| by the triangle inequality); per cell the paper's max_dx = the
// largest disp of its particles (cell_dx, atomic max on the float bits: all values >= 0);
// *max_disp (optional) = the largest of all.
// n_stored: cell_start[ncell] (rejected inputs -- e.g. dead ghost rows -- have no slot, so the
// stored count can be below the build's n).
__global__ void k_drift(float4 *__restrict__ xyzh, const float4 *__restrict__ vm, const int *__restrict__ n_stored,
                        float dt, float *__restrict__ disp, const int *__restrict__ slot_cell,
                        float *__restrict__ cell_dx, float *max_disp)
{
    const long long n = *n_stored;
    float mx = 0.0f;
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n;
         s += (long long)gridDim.x * blockDim.x) {
        float4 p = xyzh[s];
        const float4 v = vm[s];
        const float nx = __fadd_rn(p.x, __fmul_rn(v.x, dt)), ny = __fadd_rn(p.y, __fmul_rn(v.y, dt)),
                    nz = __fadd_rn(p.z, __fmul_rn(v.z, dt));
        const float ax = nx - p.x, ay = ny - p.y, az = nz - p.z;   // the stored increment
        p.x = nx;
        p.y = ny;
        p.z = nz;
        xyzh[s] = p;
        const float d = disp[s] + sqrtf(fmaf(ax, ax, fmaf(ay, ay, az * az))) * 1.000001f;
        disp[s] = d;
        atomicMax(reinterpret_cast<int *>(cell_dx) + slot_cell[s], __float_as_int(d));
        mx = fmaxf(mx, d);
    }
    if (max_disp) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int *>(max_disp), __float_as_int(mx));
    }
}

// sph_gather_positions: the stored (drifted) positions back in input order, each coordinate
// wrapped into [0, L) (x < 0 -> x + L, x >= L -> x - L; a sum that rounds to L becomes 0):
// the input of the next sph_build_cells when a reuse loop rebuilds.
__global__ void k_gather_positions(const float4 *__restrict__ xyzh, const int *__restrict__ perm,
                                   const int *__restrict__ n_stored, long long n_out, float bx, float by, float bz,
                                   float4 *__restrict__ out)
{
    const long long n = *n_stored;       // cell_start[ncell]: slots past it were never written
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n;
         s += (long long)gridDim.x * blockDim.x) {
        const int q = perm[s];
        if (q < 0 || q >= n_out) continue;                 // ghosts / other ranks' particles
        float4 p = xyzh[s];
        const float b[3] = {bx, by, bz};
        float c[3] = {p.x, p.y, p.z};
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            float v = c[k];
            if (v < 0.0f) v += b[k];
            else if (v >= b[k]) v -= b[k];
            if (v >= b[k]) v = 0.0f;
            c[k] = v;
        }
        out[q] = make_float4(c[0], c[1], c[2], p.w);
    }
}

constexpr int STABLE_SMALL = 128;
constexpr int STABLE_WARPS = 8;
constexpr int STABLE_LANE = 4;          // cells up to this size: one lane (k_stable_small)
constexpr int STABLE_BIG_CHUNK = 256;
constexpr int STABLE_BIG_TILE = 4096;
constexpr int STABLE_BT_MAX = 16384;     // cells of STABLE_SMALL < n <= this: k_stable_radix
constexpr int STABLE_BT_T = 512;
constexpr int STABLE_MED_MAX = 2048;     //   of which <= this: 128-thread CTAs
constexpr int STABLE_MED_T = 128;

// One warp per cell of <= STABLE_SMALL particles: rank each input index among the
// cell's (all distinct) and move its record there.  Larger cells are queued as
// (cell, chunk).  slot_cell is written for every slot.
__device__ __forceinline__ void stable_place(int s0, int e, int r, const ParticleRec *__restrict__ rec,
                                             float4 *__restrict__ xyzh,
                                             float4 *__restrict__ vm, int *__restrict__ perm)
{
    const float4 qx = rec[s0 + e].xyzh, qv = rec[s0 + e].vm;
    const unsigned key = (unsigned)rec[s0 + e].idx;
    xyzh[s0 + r] = qx;
    vm[s0 + r] = qv;
    perm[s0 + r] = (int)(key & 0x7fffffffu);
}

// SORT (sph_build_sort_cells): a cell of <= SORT_SMALL particles also gets its 13 sorted lists
// here, from the records the warp already holds (sort_small_lists, the small tier of
// sph_sort_cells; identical lists): the memory-bound placement and the issue-bound ranking
// overlap in one kernel, and the sort does not re-read the cell.
template <bool SORT>
__global__ void __launch_bounds__(STABLE_WARPS * 32) k_stable_small(long long ncell, const int *__restrict__ start,
                                                                    const ParticleRec *__restrict__ rec,
                                                                    float4 *__restrict__ xyzh, float4 *__restrict__ vm,
                                                                    int *__restrict__ perm, int *__restrict__ slot_cell,
                                                                    int *__restrict__ cell_nhome,
                                                                    float *__restrict__ cell_hmax,
                                                                    int *__restrict__ row_home, int nz,
                                                                    int2 *big_items, int *big_count, int *bt_items,
                                                                    int *bt_count, int bt_cap, DevGrid g,
                                                                    uint16_t *ord, long long cap)
{
    __shared__ unsigned sh[STABLE_WARPS][STABLE_SMALL];
    __shared__ unsigned ss[SORT ? STABLE_WARPS : 1][32 * 16];   // SORT: composites per warp
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int PER = STABLE_SMALL / 32;
    const float cmax = 1.7320508075688772f * (float)fmax(g.cl[0], fmax(g.cl[1], g.cl[2]));
    const float scale = 33554432.0f / (2.0f * cmax);         // as k_sort_small
    const float cmax_s = cmax * scale;
    // 32 cells per warp step (empty cells cost one lane each: sparse fine grids)
    for (long long base = ((long long)blockIdx.x * STABLE_WARPS + w) * 32; base < ncell;
         base += (long long)gridDim.x * STABLE_WARPS * 32) {
        const long long mycell = base + lane;
        const int my_s0 = mycell < ncell ? start[mycell] : 0;
        const int my_n = mycell < ncell ? start[mycell + 1] - my_s0 : 0;
        if (mycell < ncell && my_n == 0) {
            cell_nhome[mycell] = 0;
            cell_hmax[mycell] = 0.0f;
        }
        float my_corner[3] = {0.f, 0.f, 0.f};              // SORT: the lane's own cell, once per 32 cells
        if (SORT && my_n > 0 && my_n <= SORT_SMALL) {
            double cd[3];
            cell_corner(g, mycell, cd);
            my_corner[0] = (float)cd[0]; my_corner[1] = (float)cd[1]; my_corner[2] = (float)cd[2];
        }
        bool tiny = false;
        if (!SORT && my_n > 0 && my_n <= STABLE_LANE) {
            // a cell of up to STABLE_LANE particles (most non-empty cells of sparse level grids):
            // the lane places it itself -- same order (key: home first, input order) and outputs
            tiny = true;
            unsigned k[STABLE_LANE];
#pragma unroll
            for (int e = 0; e < STABLE_LANE; ++e) k[e] = e < my_n ? (unsigned)rec[my_s0 + e].idx : 0xffffffffu;
            float hm = 0.0f;
            int nh = 0;
#pragma unroll
            for (int e = 0; e < STABLE_LANE; ++e) {
                if (e >= my_n) break;
                int r = 0;
#pragma unroll
                for (int m = 0; m < STABLE_LANE; ++m) r += k[m] < k[e] ? 1 : 0;   // keys distinct
                const float4 qx = rec[my_s0 + e].xyzh;
                xyzh[my_s0 + r] = qx;
                vm[my_s0 + r] = rec[my_s0 + e].vm;
                perm[my_s0 + r] = (int)(k[e] & 0x7fffffffu);
                slot_cell[my_s0 + e] = (int)mycell;
                nh += k[e] < 0x80000000u ? 1 : 0;
                hm = fmaxf(hm, qx.w);
            }
            cell_nhome[mycell] = nh;
            cell_hmax[mycell] = hm;
            if (nh > 0) row_home[mycell / nz] = 1;
        }
        unsigned todo = __ballot_sync(0xffffffffu, my_n > 0 && !tiny);
      while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        const long long cell = base + j;
        const int s0 = __shfl_sync(0xffffffffu, my_s0, j);
        const int n = __shfl_sync(0xffffffffu, my_n, j);
        int nh = 0;
        float hm = 0.0f;
        for (int e = lane; e < n; e += 32) {
            slot_cell[s0 + e] = (int)cell;
            nh += (unsigned)rec[s0 + e].idx < 0x80000000u;
            hm = fmaxf(hm, rec[s0 + e].xyzh.w);
        }
        nh = __reduce_add_sync(0xffffffffu, nh);
        hm = __int_as_float(__reduce_max_sync(0xffffffffu, (unsigned)__float_as_int(hm)));   // h > 0
        if (lane == 0) {
            cell_nhome[cell] = nh;
            cell_hmax[cell] = hm;
            if (nh > 0) row_home[cell / nz] = 1;         // k_v4_tiles skips rows without home particles
        }
        if (n > STABLE_SMALL && n <= STABLE_BT_MAX) {      // k_stable_radix: medium from the front, huge from the back
            if (lane == 0) {
                if (n <= STABLE_MED_MAX) bt_items[atomicAdd(&bt_count[0], 1)] = (int)cell;
                else bt_items[bt_cap - 1 - atomicAdd(&bt_count[1], 1)] = (int)cell;
            }
            continue;
        }
        if (n > STABLE_SMALL) {
            if (lane == 0) {
                int nch = (n + STABLE_BIG_CHUNK - 1) / STABLE_BIG_CHUNK;
                int pos = atomicAdd(big_count, nch);
                for (int k = 0; k < nch; ++k) big_items[pos + k] = make_int2((int)cell, k);
            }
            continue;
        }
        unsigned v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = lane + 32 * k;
            v[k] = e < n ? (unsigned)rec[s0 + e].idx : 0u;
            if (e < n) sh[w][e] = v[k];
        }
        __syncwarp();
        int r0 = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int e = lane + 32 * k;
            if (e < n) {
                int r = 0;
                for (int m = 0; m < n; ++m) r += sh[w][m] < v[k];
                stable_place(s0, e, r, rec, xyzh, vm, perm);
                if (k == 0) r0 = r;
            }
        }
        __syncwarp();
        if (SORT && n <= SORT_SMALL) {
            // lane e holds record e, placed at in-cell index r0
            const float fc[3] = {__shfl_sync(0xffffffffu, my_corner[0], j), __shfl_sync(0xffffffffu, my_corner[1], j),
                                 __shfl_sync(0xffffffffu, my_corner[2], j)};
            const bool mine = lane < n;
            const float4 p = mine ? rec[s0 + lane].xyzh : make_float4(0.f, 0.f, 0.f, 0.f);
            sort_small_lists(ss[SORT ? w : 0], ord, cap, s0, n, mine, p, r0, fc, scale, cmax_s);
        }
      }
    }
}

// One CTA per cell of STABLE_SMALL < n <= STABLE_BT_MAX particles: a stable LSD radix sort of
// the records' keys (input index | not-home bit << 31, all distinct) in shared memory, then
// every record moved to its rank: 8-bit digits, only the bytes in which the cell's keys differ (OR ^ AND over the cell; random input order: three of four), per
// pass a count sweep, one exclusive scan over (digit, warp) and a stable MATCH-ranked
// scatter of (key, in-cell position) -- the scheme of k_sort_radix (sort.cuh).
// Two tiers as in sph_sort_cells: cells of <= STABLE_MED_MAX on 128-thread CTAs (33 KB, several
// per SM; queued from the front of the item list), larger ones on 512 threads (212 KB; from
// the back).
constexpr int stable_radix_smem(int maxn, int t) { return maxn * 12 + 256 * (t / 32) * 4 + 64 * 4; }

template <int MAXN, int T, bool FROM_BACK>
__global__ void __launch_bounds__(T) k_stable_radix(const int *__restrict__ start,
                                                   const ParticleRec *__restrict__ rec,
                                                   float4 *__restrict__ xyzh, float4 *__restrict__ vm,
                                                   int *__restrict__ perm, const int *__restrict__ items,
                                                   const int *__restrict__ count, int cap)
{
    constexpr int NW = T / 32, NH = 256 * NW, HPT = NH / T, RU = 4;
    static_assert(NH % T == 0, "radix: 256 x warps must be a multiple of the threads");
    extern __shared__ unsigned rs[];
    unsigned *keyA = rs, *keyB = rs + MAXN;
    uint16_t *idxA = reinterpret_cast<uint16_t *>(rs + 2 * MAXN), *idxB = idxA + MAXN;
    unsigned *hist = rs + 3 * MAXN, *wsum = hist + NH;
    __shared__ unsigned s_or, s_and;
    const int nitems = *count;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const long long cell = items[FROM_BACK ? cap - 1 - it : it];
        const int s0 = start[cell], n = start[cell + 1] - s0;
        const int S = (n + NW - 1) / NW;
        const int lo = min(n, w * S), hi = min(n, lo + S);
        if (threadIdx.x == 0) { s_or = 0u; s_and = ~0u; }
        __syncthreads();
        unsigned o = 0u, a = ~0u;
        for (int e = threadIdx.x; e < n; e += T) {
            const unsigned k = (unsigned)rec[s0 + e].idx;
            keyA[e] = k;
            idxA[e] = (uint16_t)e;
            o |= k;
            a &= k;
        }
        o = __reduce_or_sync(0xffffffffu, o);
        a = __reduce_and_sync(0xffffffffu, a);
        if (lane == 0) { atomicOr(&s_or, o); atomicAnd(&s_and, a); }
        __syncthreads();
        const unsigned diff = s_or ^ s_and;
        unsigned *ks = keyA, *kd = keyB;
        uint16_t *is = idxA, *id = idxB;
        for (int shift = 0; shift < 32; shift += 8) {
            if (!((diff >> shift) & 255u)) continue;   // CTA-uniform: every key has this byte
#pragma unroll
            for (int q = 0; q < HPT; ++q) hist[threadIdx.x * HPT + q] = 0u;
            __syncthreads();
            for (int b = lo; b < hi; b += 32 * RU) {
                unsigned dg[RU], peers[RU];
#pragma unroll
                for (int u = 0; u < RU; ++u) {
                    const int i = b + 32 * u + lane;
                    dg[u] = i < hi ? (ks[i] >> shift) & 255u : 256u;
                }
#pragma unroll
                for (int u = 0; u < RU; ++u) peers[u] = __match_any_sync(0xffffffffu, dg[u]);
#pragma unroll
                for (int u = 0; u < RU; ++u)
                    if (dg[u] < 256u && !(peers[u] & lt_mask)) atomicAdd(&hist[dg[u] * NW + w], __popc(peers[u]));
            }
            __syncthreads();
            unsigned loc[HPT], sum = 0u;
#pragma unroll
            for (int q = 0; q < HPT; ++q) { loc[q] = hist[threadIdx.x * HPT + q]; sum += loc[q]; }
            unsigned run = block_excl_scan<T>(sum, wsum, lane, w);
#pragma unroll
            for (int q = 0; q < HPT; ++q) { hist[threadIdx.x * HPT + q] = run; run += loc[q]; }
            __syncthreads();
            for (int b = lo; b < hi; b += 32 * RU) {
                unsigned k[RU], dg[RU], peers[RU];
                uint16_t ix[RU];
#pragma unroll
                for (int u = 0; u < RU; ++u) {
                    const int i = b + 32 * u + lane;
                    k[u] = i < hi ? ks[i] : 0u;
                    ix[u] = i < hi ? is[i] : (uint16_t)0;
                    dg[u] = i < hi ? (k[u] >> shift) & 255u : 256u;
                }
#pragma unroll
                for (int u = 0; u < RU; ++u) peers[u] = __match_any_sync(0xffffffffu, dg[u]);
#pragma unroll
                for (int u = 0; u < RU; ++u) {
                    const unsigned r = __popc(peers[u] & lt_mask);
                    const unsigned hx = min(dg[u], 255u) * NW + w;
                    const unsigned base = hist[hx];
                    if (dg[u] < 256u) {
                        kd[base + r] = k[u];
                        id[base + r] = ix[u];
                    }
                    __syncwarp();
                    if (dg[u] < 256u && r == 0) hist[hx] = base + __popc(peers[u]);
                    __syncwarp();
                }
            }
            __syncthreads();
            unsigned *tk = ks; ks = kd; kd = tk;
            uint16_t *ti = is; is = id; id = ti;
        }
        for (int r = threadIdx.x; r < n; r += T) stable_place(s0, is[r], r, rec, xyzh, vm, perm);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(STABLE_BIG_CHUNK) k_stable_big(const int *__restrict__ start,
                                                                  const ParticleRec *__restrict__ rec,
                                                                  float4 *__restrict__ xyzh, float4 *__restrict__ vm,
                                                                  int *__restrict__ perm,
                                                                  const int2 *big_items, const int *big_count)
{
    __shared__ unsigned tile[STABLE_BIG_TILE];
    const int nitems = *big_count;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        int2 item = big_items[it];
        int s0 = start[item.x];
        int n = start[item.x + 1] - s0;
        int e = item.y * STABLE_BIG_CHUNK + threadIdx.x;
        bool mine = e < n;
        unsigned v = mine ? (unsigned)rec[s0 + e].idx : 0u;
        int r = 0;
        for (int t0 = 0; t0 < n; t0 += STABLE_BIG_TILE) {
            int tn = min(STABLE_BIG_TILE, n - t0);
            __syncthreads();
            for (int m = threadIdx.x; m < tn; m += blockDim.x) tile[m] = (unsigned)rec[s0 + t0 + m].idx;
            __syncthreads();
            if (mine)
                for (int m = 0; m < tn; ++m) r += tile[m] < v;
        }
        if (mine) stable_place(s0, e, r, rec, xyzh, vm, perm);
        __syncthreads();
    }
}


}  // namespace pvsph
