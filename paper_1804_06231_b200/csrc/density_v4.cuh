// density_v4.cuh -- the production sph_density_all engine.
//
// Method (unchanged from the reference engine in density.cuh): every owned
// particle i gathers from its own cell and the 26 neighbour cells; in a
// neighbour cell only the window of its list sorted along the pair axis whose
// projected separation is below H_i + delta is tested (Code 2; the
// per-particle bound of P:151-165), in-range pairs are interacted
// and the sums are written once per particle.
//
// Mapping onto the B200 SM:
//
//  * Tiles.  A tile is a z-range of cells in a PAIR of adjacent rows (x, y),
//    (x, y+1) holding at most V4_TP = 256 particles (k_v4_tiles cuts the rows
//    greedily; the cut depends only on the row pair's own counts, so tiles are
//    identical on any number of GPUs).  Row pairs are enumerated in 4 x 4
//    blocks so that CTAs running at the same time share neighbourhoods in L2.
//  * Staging (the particle cache of P:136).  A CTA copies the tile's
//    neighbourhood -- 4 x 3 rows times (z-range + 2) cells -- into shared
//    memory: positions as SoA X, Y, Z (periodic images beyond a low face
//    pre-shifted by -L, exact by Sterbenz: DESIGN.md §4.3) and (v, m) as
//    float4.  Particles beyond a high face are left in place and the home
//    coordinate is shifted instead (also exact).  ~1.8k particles at c5.
//  * Lanes.  One lane per home particle (register accumulators, one writer).
//    The self cell and the 13 direction pairs are swept in a fixed order; for
//    direction d the lane's window in the +d neighbour (a prefix of its list)
//    and in the -d neighbour (a suffix of the same-direction list) are found
//    exactly by bisection on the staged positions and swept back to back (their
//    lengths are anti-correlated, which evens the lanes out).
//  * Hits (the left-packing of P:185) go to a per-lane queue of staged indices
//    in shared memory ([slot][lane], conflict-free); when most lanes hold two
//    the warp pops one pair per lane and evaluates both interactions with
//    FFMA2/FADD2/FMUL2.  Every particle sums its hits in sweep order, so the
//    result does not depend on the tile or the warp (deterministic, identical
//    on any number of GPUs).
//  * Tiles that do not fit (a slice of more than V4_TP particles, or a
//    neighbourhood above the staging capacity: clustered data) are processed by
//    the same CTA with the reference per-particle sweep reading global memory
//    (identical arithmetic per pair).
#pragma once

#include "common.cuh"
#include "density.cuh"
#include "packed.cuh"

#include <type_traits>

namespace pvsph {

// tile geometry (overridable at compile time for experiments: -DTILE_WARPS=4 ...)
#ifndef TILE_WARPS
#define TILE_WARPS 8
#define TILE_MAXZ 21
#define TILE_MS 2336
#define TILE_ML 8192
#endif
constexpr int V4_WARPS = TILE_WARPS;
constexpr int V4_CTAS = 2;               // resident CTAs per SM (launch bounds; smem below fits 2)
constexpr int V4_TP = V4_WARPS * 32;     // home particles per tile: exactly V4_TP except where a limit cuts
constexpr int V4_Q = 24;                 // hit stack depth per lane, 2-byte entries
constexpr int V4_ROWS = 12;              // staged rows: ox in -1..1, oy in -1..2 (relative to the tile's first row)
constexpr int V4_MAXZ = TILE_MAXZ;       // staged cells per row (tiles span <= 19 slices)
constexpr int V4_MAXCELLS = V4_ROWS * V4_MAXZ;
constexpr int V4_MAXH = 2 * (V4_MAXZ - 2);   // home cells per tile
constexpr int V4_MS = TILE_MS;           // staged particles (< 4096: 12-bit queue entries)
constexpr int V4_ML = TILE_ML;           // staged list entries (27 segments per home cell)
constexpr int V4_HOFF = (V4_MAXH + 4 + 3) / 4 * 4;      // ints, keeps the following arrays 16-byte aligned
constexpr size_t V4_SMEM = (size_t)V4_MS * 32 + (size_t)V4_MAXCELLS * 16 + (size_t)V4_ML * 2 + (size_t)V4_HOFF * 4 +
                           (size_t)V4_WARPS * V4_Q * 32 * 2 + (size_t)V4_MAXZ * 16;
static_assert(V4_ML % 8 == 0 && (V4_WARPS * V4_Q * 32 * 2) % 16 == 0, "16-byte aligned shared arrays");


// Results of one particle at its INPUT index: rho, wcount, rho_dh, wcount_dh, div_v, curl_v (3)
// in the first 32-byte sector; nngb, the input index and the call's generation (tag) in the
// second.  Each sector is written whole by one 256-bit store (no read-modify-write), scattered
// while the compute-bound density kernel runs; the input-order transpose (k_unpermute) then
// reads the records sequentially and keeps those tagged by this call (home particles).
struct alignas(32) OutRec {
    float4 a, b;
    int nngb, idx;
    unsigned gen, pad[5];
};

// generation of the running sph_density_all call (ws word, bumped by k_v4_tiles<false>)
__shared__ unsigned s_gen;

__device__ __forceinline__ void store_rec(OutRec *orec, int idx, float rho, float wc, float rho_dh, float wc_dh,
                                          float div, float cx, float cy, float cz, int nngb)
{
    // evict-first: the scattered records must not push the staged neighbourhoods out of L2
    asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(orec + idx), "f"(rho),
                 "f"(wc), "f"(rho_dh), "f"(wc_dh), "f"(div), "f"(cx), "f"(cy), "f"(cz)
                 : "memory");
    asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %4, %4, %4, %4};" ::"l"(&orec[idx].nngb), "r"(nngb),
                 "r"(idx), "r"(s_gen), "r"(0)
                 : "memory");
}

// out[p] = record p for the first n_out input indices whose record this call wrote (home on
// this grid, not rejected): sequential 64-byte reads, coalesced SoA writes.
__global__ void __launch_bounds__(256) k_unpermute(DevOut o, const OutRec *__restrict__ orec,
                                                    const unsigned *__restrict__ genp)
{
    const unsigned gen = *genp;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < o.n_out; p += stride) {
        const float4 *q = reinterpret_cast<const float4 *>(orec + p);
        const int4 t = __ldcs(reinterpret_cast<const int4 *>(q + 2));   // nngb, idx, gen, -
        if (t.y != (int)p || (unsigned)t.z != gen) continue;            // not written by this call
        const float4 a = __ldcs(q), b = __ldcs(q + 1);
        __stcs(o.rho + p, a.x);
        __stcs(o.wcount + p, a.y);
        __stcs(o.rho_dh + p, a.z);
        __stcs(o.wcount_dh + p, a.w);
        __stcs(o.div_v + p, b.x);
        __stcs(o.curl_v + p, b.y);
        __stcs(o.curl_v + o.n_out + p, b.z);
        __stcs(o.curl_v + 2 * o.n_out + p, b.w);
        __stcs(o.nngb + p, t.x);
    }
}

// ---- optional phase timing (compile with -DPVSPH_PHASE_TIMING; profiling only) --------
#ifdef PVSPH_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[12];   // 0 stage, 1 search, 2 sweep, 3 drain, 4 final drain, 5 barrier
#define PH_T0(v) long long v = clock64();
#define PH_ADD(k, v) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase_cycles[k], (unsigned long long)(clock64() - (v))); } while (0)
#else
#define PH_T0(v)
#define PH_ADD(k, v) do { } while (0)
#endif

// ---- tile list ------------------------------------------------------------------
// row_home[(x, y) row] = 1 iff some cell of the row holds a home particle (cell_nhome > 0):
// k_v4_tiles skips the other rows (fine level grids are mostly empty).  Computed by
// sph_density_all itself from the cells, so it depends on no other call's workspace state.
__global__ void k_row_home(long long nrows, int nz, const int *__restrict__ cell_nhome, int *__restrict__ row_home)
{
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long row = warp; row < nrows; row += nwarps) {
        int any = 0;
        for (int z = lane; z < nz; z += 32) any |= cell_nhome[row * nz + z] > 0;
        any = __any_sync(0xffffffffu, any);
        if (lane == 0) row_home[row] = any;
    }
}

struct RowPairs {
    int nxo, nyp, nby;
    long long nkeys;
};

#ifndef RP_BX
#define RP_BX 4        // row-pair blocks: RP_BX x-planes by RP_BY row pairs
#endif
#ifndef RP_BY
#define RP_BY 4
#endif
__host__ __device__ __forceinline__ RowPairs row_pairs(const DevGrid &g)
{
    RowPairs r;
    r.nxo = g.x_hi - g.x_lo;
    r.nyp = (g.ny + 1) / 2;
    r.nby = (r.nyp + RP_BY - 1) / RP_BY;
    r.nkeys = (long long)((r.nxo + RP_BX - 1) / RP_BX) * r.nby * (RP_BX * RP_BY);
    return r;
}

__host__ __device__ __forceinline__ void key_rowpair(const RowPairs &r, long long key, int &xo, int &yp)
{
    const long long blk = key / (RP_BX * RP_BY);
    const int w = (int)(key % (RP_BX * RP_BY));
    xo = (int)(blk / r.nby) * RP_BX + w / RP_BY;
    yp = (int)(blk % r.nby) * RP_BY + w % RP_BY;
}

__host__ __device__ __forceinline__ long long v4_tile_capacity(const DevGrid &g, long long n)
{
    // every tile holds a non-empty z-slice, and a slice yields at most ceil(n_slice / V4_TP) tiles
    return n / V4_TP + g.n_owned_cells + 64;
}

// Local cell of staged row k (ox = k/4 - 1, oy = k%4 - 1 relative to the tile's first
// row y0 of owned plane xo) at unwrapped z; also the periodic flags of DESIGN.md §4.3.
struct StagedRow {
    long long base;   // local cell id of (row, z = 0)
    int gx, uy;       // unwrapped global x plane and y row
};

__device__ __forceinline__ StagedRow staged_row(const DevGrid &g, int xo, int y0, int k)
{
    const int ox = k / 4 - 1, oy = k % 4 - 1;
    const int xl = xo + g.ghost_x;
    const int jx = g.ghost_x ? xl + ox : wrap_i(xl + ox, g.nc[0]);
    StagedRow r;
    r.gx = g.x_lo + xo + ox;
    r.uy = y0 + oy;
    r.base = ((long long)jx * g.ny + wrap_i(r.uy, g.ny)) * g.nz;
    return r;
}

// Per z: particles of the home slice, of the 12 staged rows, and of the 9 rows around
// each home row (the 27-cell list sizes are sums of three consecutive z).
struct ZCols {
    int slice, c12, c9a, c9b;
};

__device__ __forceinline__ ZCols zcols(const DevGrid &g, const int *__restrict__ cs, const int *__restrict__ nhome,
                                       const long long rb[V4_ROWS], bool hasB, int z)
{
    const int wz = wrap_i(z, g.nz);
    int n[V4_ROWS];
#pragma unroll
    for (int k = 0; k < V4_ROWS; ++k) n[k] = cs[rb[k] + wz + 1] - cs[rb[k] + wz];
    ZCols c;
    // home particles of the slice (rows 5, 6 = the tile's two rows); the rest counts all particles
    c.slice = (z >= 0 && z < g.nz) ? nhome[rb[5] + wz] + (hasB ? nhome[rb[6] + wz] : 0) : 0;
    c.c12 = c.c9a = c.c9b = 0;
#pragma unroll
    for (int k = 0; k < V4_ROWS; ++k) {
        c.c12 += n[k];
        if (k % 4 <= 2) c.c9a += n[k];
        if (k % 4 >= 1) c.c9b += n[k];
    }
    if (!hasB) c.c9b = 0;
    return c;
}

// Cut of one row pair into tiles.  The particles of a row pair are taken in the
// sequence z = 0, 1, ..., each z-slice listing its row-A cell then its row-B cell.
// A staged tile is a run of V4_TP consecutive particles of that sequence (fewer
// where a limit cuts it): at most V4_MS staged neighbours, V4_ML list entries and
// V4_MAXZ - 2 slices, so every warp of the CTA is full.  Its first and last cells
// may be shared with the neighbouring tiles.  A slice whose neighbourhood cannot be
// staged becomes global-memory tiles of <= V4_TP particles.  Descriptor:
// {key, z_a | z_b << 16, first particle in slice z_a, count (< 0: global-memory)}.
// The cut depends only on the row pair's own counts (identical on any GPU count).
template <bool WRITE>
__global__ void k_v4_tiles(DevGrid g, const int *__restrict__ cell_start, const int *__restrict__ nhome,
                           int *__restrict__ off, int4 *tiles, long long tile_cap, unsigned *status, unsigned *gen,
                           int *gtiles, int *gcount, const int *__restrict__ row_home)
{
    // the counting launch opens a new sph_density_all call: its records carry the new tag
    if (!WRITE && blockIdx.x == 0 && threadIdx.x == 0) *gen += 1u;
    const RowPairs r = row_pairs(g);
    for (long long key = blockIdx.x * (long long)blockDim.x + threadIdx.x; key < r.nkeys;
         key += (long long)gridDim.x * blockDim.x) {
        int xo, yp;
        key_rowpair(r, key, xo, yp);
        int nt = 0;
        // row pairs without a home particle (most rows of a fine level grid) emit nothing
        const long long ra = (long long)(xo + g.ghost_x) * g.ny + 2 * yp;
        const bool any_home = xo < r.nxo && yp < r.nyp && (row_home[ra] || (2 * yp + 1 < g.ny && row_home[ra + 1]));
        if (any_home) {
            const int y0 = 2 * yp;
            const bool hasB = y0 + 1 < g.ny;
            long long rb[V4_ROWS];
#pragma unroll
            for (int k = 0; k < V4_ROWS; ++k) rb[k] = staged_row(g, xo, y0, k).base;
            int pos = WRITE ? off[key] : 0;
            auto emit = [&](int za, int zb, int first, int cnt) {
                if (WRITE) {
                    if (pos < tile_cap) {
                        tiles[pos] = make_int4((int)key, za | (zb << 16), first, cnt);
                        if (cnt < 0) gtiles[atomicAdd(gcount, 1)] = pos;   // k_density_dense's work list
                    } else {
                        set_status(status, ST_ECAPACITY);
                    }
                    ++pos;
                }
                ++nt;
            };
            ZCols cm = zcols(g, cell_start, nhome, rb, hasB, -1), c0 = zcols(g, cell_start, nhome, rb, hasB, 0),
                  cp = zcols(g, cell_start, nhome, rb, hasB, 1);
            bool open = false;
            int tz = 0, tfirst = 0, home = 0, stg = 0, lst = 0;
            int z = 0, o = 0;                      // next particle: o-th of slice z
            while (z < g.nz) {
                const int nb = cm.c9a + c0.c9a + cp.c9a + cm.c9b + c0.c9b + cp.c9b;
                bool take = true;
                if (!open) {
                    if (cm.c12 + c0.c12 + cp.c12 > V4_MS || nb > V4_ML) {
                        for (int k = o; k < c0.slice; k += V4_TP) emit(z, z, k, -min(V4_TP, c0.slice - k));
                        take = false;              // whole slice done
                        o = c0.slice;
                    } else {
                        open = true;
                        tz = z;
                        tfirst = o;
                        home = 0;
                        stg = cm.c12 + c0.c12 + cp.c12;
                        lst = nb;
                    }
                } else if (o == 0) {               // the open tile would extend to slice z
                    if (stg + cp.c12 > V4_MS || lst + nb > V4_ML || z - tz + 1 > V4_MAXZ - 2) {
                        if (home > 0) emit(tz, z - 1, tfirst, home);
                        open = false;
                        continue;                  // start a new tile at slice z
                    }
                    stg += cp.c12;
                    lst += nb;
                }
                if (take) {
                    const int n = min(c0.slice - o, V4_TP - home);
                    home += n;
                    o += n;
                    if (home == V4_TP) {
                        emit(tz, z, tfirst, home);
                        open = false;
                    }
                }
                if (o >= c0.slice) {
                    ++z;
                    o = 0;
                    cm = c0;
                    c0 = cp;
                    cp = zcols(g, cell_start, nhome, rb, hasB, z + 1);
                }
            }
            if (open && home > 0) emit(tz, g.nz - 1, tfirst, home);
        }
        if (!WRITE) off[key] = nt;
    }
}

// ---- the engine ------------------------------------------------------------------
// Block-wide exclusive scan of one int per thread (blockDim.x == V4_TP).
__device__ __forceinline__ int block_exscan(int v, int *wsum, int &total)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int pre = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < V4_WARPS; ++k) {
        const int s = wsum[k];
        pre += k < w ? s : 0;
        tot += s;
    }
    __syncthreads();
    total = tot;
    return pre + x - v;
}

// Reference per-particle sweep (global memory) for tiles that are not staged.
template <bool COUNT>
__device__ __forceinline__ void v4_particle_global(const DevGrid &g, const DevCells &c, OutRec *orec, int i,
                                                   unsigned cand[4], unsigned hits[4])
{
    const int home = c.slot_cell[i];
    HomeCell hc = home_cell(g, home);
    IPart p = load_i(g, c, i, hc.corner);
    Acc a;
    acc_zero(a);
    sweep_self<COUNT>(c, p, c.cell_start[home], c.cell_start[home + 1], a, cand[0], hits[0]);
    for (int ox = -1; ox <= 1; ++ox)
        for (int oy = -1; oy <= 1; ++oy)
            for (int oz = -1; oz <= 1; ++oz) {
                if (!(ox | oy | oz)) continue;
                int cj, sh[3];
                if (!neighbour(g, hc, ox, oy, oz, cj, sh)) continue;
                const int k = kind_of(ox, oy, oz);
                sweep_pair<COUNT>(g, c, p, cj, ox, oy, oz, sh, a, cand[k], hits[k]);
            }
    Final f = finalise(g, p, a, true);
    const float rinv = 1.0f / f.rho;
    store_rec(orec, c.perm[i], f.rho, f.wc, f.rho_dh, f.wc_dh, f.div * rinv, f.cx * rinv, f.cy * rinv, f.cz * rinv, a.nngb);
}

// Packed accumulators; D and curl use v_j - v_i (= -v_ij) so the cross products
// need no negation: Dn = -sum fac (v_ij . x_ij); R = P - N.
struct Acc2 {
    f2 rho, wc, srt, st, Dn, Px, Nx, Py, Ny, Pz, Nz;
};

// Two interactions (MASK: the odd half may be empty, mk = (1, 0)).
// M4 in branch-free form: w(x) = u^3 - v^3/2, w'(x) = -3 (u - v)(u + v),
// u = max(0, 1 - x), v = max(0, 1 - 2x)  (equal to the two-branch form of R1);
// u - v = min(x, u) is formed without cancellation.
template <bool MASK>
__device__ __forceinline__ void interact_pair(f2 Hinv2, f2 dx, f2 dy, f2 dz, f2 m, f2 nvx, f2 nvy, f2 nvz, f2 mk,
                                              Acc2 &A)
{
    f2 r2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    float r2a, r2b;
    upk(r2, r2a, r2b);
    // r^2 = 0 (coincident particles): rinv stays finite, x = 0 and w'(0) = 0 make every gradient term 0
    f2 rinv = rsqrt_nr2(pk(fmaxf(r2a, 1e-30f), fmaxf(r2b, 1e-30f)));
    f2 x = mul2(mul2(r2, rinv), Hinv2);
    f2 u = sub2(bc2(1.0f), x);
    f2 v = fma2(bc2(-2.0f), x, bc2(1.0f));
    float va, vb, xa, xb, ua, ub;
    upk(v, va, vb);
    upk(x, xa, xb);
    upk(u, ua, ub);
    v = pk(fmaxf(va, 0.0f), fmaxf(vb, 0.0f));
    const f2 mn = pk(fminf(xa, ua), fminf(xb, ub));
    f2 uu = mul2(u, u), vv = mul2(v, v);
    f2 w = fma2(uu, u, mul2(bc2(-0.5f), mul2(vv, v)));
    f2 dw = mul2(bc2(-3.0f), mul2(mn, add2(u, v)));
    if (MASK) {
        w = mul2(w, mk);
        dw = mul2(dw, mk);
        m = mul2(m, mk);
    }
    acc_fma2(A.rho, m, w);
    acc_add2(A.wc, w);
    f2 t = fma2(x, dw, mul2(bc2(3.0f), w));
    acc_fma2(A.srt, m, t);
    acc_add2(A.st, t);
    f2 nvdx = fma2(nvx, dx, fma2(nvy, dy, mul2(nvz, dz)));
    f2 fac = mul2(mul2(m, dw), rinv);
    acc_fma2(A.Dn, fac, nvdx);
    f2 fx = mul2(fac, nvx), fy = mul2(fac, nvy), fz = mul2(fac, nvz);
    acc_fma2(A.Px, fz, dy);
    acc_fma2(A.Nx, fy, dz);
    acc_fma2(A.Py, fx, dz);
    acc_fma2(A.Ny, fz, dx);
    acc_fma2(A.Pz, fy, dx);
    acc_fma2(A.Nz, fx, dy);
}

__device__ __forceinline__ int v4_kind(int d)
{
    // faces (0,0,1) (0,1,0) (1,0,0); corners (1,+-1,+-1); the rest edges
    return (d == 0 || d == 2 || d == 8) ? 1 : ((d == 4 || d == 6 || d == 10 || d == 12) ? 3 : 2);
}

// Shared-memory view of a staged tile (32-bit shared addresses).
struct V4Stage {
    unsigned P;               // float4 x, y, z (low-face images pre-shifted by -L), 0
    unsigned V;               // float4 vx, vy, vz, m
    unsigned L;               // uint16 staged indices: 27 segments per home cell
    const int4 *tab;          // {base, count, gstart, flags}: flags bits 0-2 home shift (+L image), 3-5 pre-shifted
    int nzs;
};

// Window lengths: the number of leading entries of two staged segments whose
// projected separation is below Hk; the separation grows along each segment.
// Segment 0 (+d neighbour, reversed list) is read backwards from storage index f0
// with sep = (x_j - h0) . d, segment 1 (-d neighbour, reversed list) forwards from
// f1 with sep = (h1 - x_j) . d.  Branch-free bisection with `top` = the largest
// power of two <= the warp's longest segment, so every lane runs the same steps:
// the exact per-particle bound of P:151-165; the two searches are interleaved.
template <int D>
__device__ __forceinline__ float v4_dot(float dx, float dy, float dz)
{
    // d . (dx, dy, dz) with the canonical direction's components (+1, -1 or 0) folded in
    constexpr int a0 = D == 0 ? 0 : (D <= 3 ? 0 : 1);
    constexpr int a1 = D == 0 ? 0 : (D <= 3 ? 1 : (D - 4) / 3 - 1);
    constexpr int a2 = D == 0 ? 1 : (D <= 3 ? D - 2 : (D - 4) % 3 - 1);
    float s = 0.0f;
    bool any = false;
    if (a0 != 0) { s = a0 > 0 ? dx : -dx; any = true; }
    if (a1 != 0) { s = any ? (a1 > 0 ? s + dy : s - dy) : (a1 > 0 ? dy : -dy); any = true; }
    if (a2 != 0) { s = any ? (a2 > 0 ? s + dz : s - dz) : (a2 > 0 ? dz : -dz); }
    return s;
}

template <int D>
__device__ __forceinline__ void v4_windows_d(const V4Stage &S, int top, int f0, int n0, int f1, int n1, float h0x,
                                             float h0y, float h0z, float h1x, float h1y, float h1z, float Hk,
                                             int &len0, int &len1)
{
    int lo0 = 0, lo1 = 0;
    for (int st = top; st > 0; st >>= 1) {
        const int k0 = lo0 + st, k1 = lo1 + st;           // is entry k - 1 inside the window?
        const bool v0 = k0 <= n0, v1 = k1 <= n1;
        const unsigned i0 = v0 ? ldsr_u16(S.L + 2u * (unsigned)(f0 - k0 + 1)) : 0u;
        const unsigned i1 = v1 ? ldsr_u16(S.L + 2u * (unsigned)(f1 + k1 - 1)) : 0u;
        const float4 p0 = ldsr_f4(S.P + 16u * i0), p1 = ldsr_f4(S.P + 16u * i1);
        const float s0 = v4_dot<D>(p0.x - h0x, p0.y - h0y, p0.z - h0z);
        const float s1 = v4_dot<D>(h1x - p1.x, h1y - p1.y, h1z - p1.z);
        if (v0 && s0 < Hk) lo0 = k0;
        if (v1 && s1 < Hk) lo1 = k1;
    }
    len0 = lo0;
    len1 = lo1;
}

// Windows of two directions D0, D1 at once: four independent bisections in lockstep.
template <int D0, int D1>
__device__ __forceinline__ void v4_windows2_d(const V4Stage &S, int top, const int f[4], const int n[4],
                                              const float h[4][3], const float Hk[2], int len[4])
{
    int lo[4] = {0, 0, 0, 0};
    for (int st = top; st > 0; st >>= 1) {
        unsigned idx[4];
        bool v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int kk = lo[k] + st;
            v[k] = kk <= n[k];
            // segments 0, 2 (+d) read backwards from f, segments 1, 3 (-d) forwards
            idx[k] = v[k] ? ldsr_u16(S.L + 2u * (unsigned)((k & 1) ? f[k] + kk - 1 : f[k] - kk + 1)) : 0u;
        }
        float4 p[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) p[k] = ldsr_f4(S.P + 16u * idx[k]);
        const float s0 = v4_dot<D0>(p[0].x - h[0][0], p[0].y - h[0][1], p[0].z - h[0][2]);
        const float s1 = v4_dot<D0>(h[1][0] - p[1].x, h[1][1] - p[1].y, h[1][2] - p[1].z);
        const float s2 = v4_dot<D1>(p[2].x - h[2][0], p[2].y - h[2][1], p[2].z - h[2][2]);
        const float s3 = v4_dot<D1>(h[3][0] - p[3].x, h[3][1] - p[3].y, h[3][2] - p[3].z);
        if (v[0] && s0 < Hk[0]) lo[0] += st;
        if (v[1] && s1 < Hk[0]) lo[1] += st;
        if (v[2] && s2 < Hk[1]) lo[2] += st;
        if (v[3] && s3 < Hk[1]) lo[3] += st;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) len[k] = lo[k];
}

__device__ __forceinline__ void v4_windows2(const V4Stage &S, int dpair, int top, const int f[4], const int n[4],
                                            const float h[4][3], const float Hk[2], int len[4])
{
#define V4W2(P) case P: v4_windows2_d<2 * P, 2 * P + 1>(S, top, f, n, h, Hk, len); break;
    switch (dpair) {
        V4W2(0) V4W2(1) V4W2(2) V4W2(3) V4W2(4) V4W2(5)
    default: len[0] = len[1] = len[2] = len[3] = 0;
    }
#undef V4W2
}

__device__ __forceinline__ void v4_windows(const V4Stage &S, int d, int top, int f0, int n0, int f1, int n1,
                                           float h0x, float h0y, float h0z, float h1x, float h1y, float h1z, float Hk,
                                           int &len0, int &len1)
{
#define V4W(D) case D: v4_windows_d<D>(S, top, f0, n0, f1, n1, h0x, h0y, h0z, h1x, h1y, h1z, Hk, len0, len1); break;
    switch (d) {
        V4W(0) V4W(1) V4W(2) V4W(3) V4W(4) V4W(5) V4W(6) V4W(7) V4W(8) V4W(9) V4W(10) V4W(11) V4W(12)
    default: len0 = len1 = 0;
    }
#undef V4W
}

// One lane = one home particle of a staged tile.  lpos: first list entry of its home
// cell, qh: its staged column, yoff: its row in the tile (0/1).  FRAMES: the tile
// touches a high box face (some home coordinate must be shifted by -L).
// Hits are pushed on a per-lane stack of staged indices in shared memory (slot k of
// lane l at qbase + 64 k + 2 l: conflict-free); every particle sums its hits in a
// fixed order, so the result does not depend on the tile or the warp.
template <bool COUNT, bool FRAMES>
__device__ __forceinline__ void v4_particle_staged(const DevGrid &g, const DevCells &c, OutRec *orec,
                                                   const V4Stage &S, unsigned qbase, bool active, int i, int yoff,
                                                   int qh, int lpos, unsigned cand[4], unsigned hits[4])
{
    const unsigned sQ = qbase + 2u * (threadIdx.x & 31);
    float x = 0.f, y = 0.f, z = 0.f, vx = 0.f, vy = 0.f, vz = 0.f, m = 0.f, H2 = -1.f, Hinv = 0.f, Hd = 0.f;
    if (active) {
        const float4 a = c.xyzh[i];
        const float4 b = c.vm[i];
        x = a.x; y = a.y; z = a.z;
        vx = b.x; vy = b.y; vz = b.z; m = b.w;
        const double H = (double)g.gamma * (double)a.w;   // exact product; H^2, 1/H rounded once
        H2 = (float)(H * H);
        Hinv = (float)(1.0 / H);
        Hd = (float)H + g.delta;
    }
    const float xs = x - g.boxf[0], ys = y - g.boxf[1], zs = z - g.boxf[2];   // exact where used (x >= L/2)
    const float Hd2 = Hd * 1.41421356237309505f, Hd3 = Hd * 1.73205080756887729f;   // (H + delta) sqrt(kind)
    const f2 Hinv2 = bc2(Hinv);
    auto scell = [&](int ox, int oy, int oz) { return ((ox + 1) * 4 + oy + yoff + 1) * S.nzs + qh + oz; };
    const int4 eh = S.tab[scell(0, 0, 0)];
    const int kh = active ? i - eh.z : -1;                // in-cell index of i

    Acc2 A;
    A.rho = A.wc = A.srt = A.st = A.Dn = A.Px = A.Nx = A.Py = A.Ny = A.Pz = A.Nz = zero2();
    unsigned qp = sQ;                                     // stack top (next free slot)
    int nngb = 0;

    auto home_of = [&](unsigned fl, float &hx, float &hy, float &hz) {
        hx = (fl & 1u) ? xs : x;
        hy = (fl & 2u) ? ys : y;
        hz = (fl & 4u) ? zs : z;
    };
    // pop two hits per lane (FINAL: also a single one)
    auto drain = [&](auto final_tag) {
        constexpr bool FINAL = decltype(final_tag)::value;
        const unsigned n = (qp - sQ) >> 6;
        if (n >= 2 || (FINAL && n == 1)) {
            const bool two = !FINAL || n >= 2;
            const unsigned e0 = lds_u16(qp - 64u);
            const unsigned e1 = two ? lds_u16(qp - 128u) : e0;
            qp -= two ? 128u : 64u;
            nngb += two ? 2 : 1;
            const unsigned s0 = FRAMES ? (e0 & 0xfffu) : e0, s1 = FRAMES ? (e1 & 0xfffu) : e1;
            float hx0 = x, hy0 = y, hz0 = z, hx1 = x, hy1 = y, hz1 = z;
            if (FRAMES) {
                home_of(e0 >> 12, hx0, hy0, hz0);
                home_of(e1 >> 12, hx1, hy1, hz1);
            }
            const float4 p0 = ldsr_f4(S.P + 16u * s0), p1 = ldsr_f4(S.P + 16u * s1);
            const float4 v0 = ldsr_f4(S.V + 16u * s0), v1 = ldsr_f4(S.V + 16u * s1);
            const f2 mk = pk(1.0f, two ? 1.0f : 0.0f);
            interact_pair<FINAL>(Hinv2, pk(hx0 - p0.x, hx1 - p1.x), pk(hy0 - p0.y, hy1 - p1.y),
                                 pk(hz0 - p0.z, hz1 - p1.z), pk(v0.w, v1.w), pk(v0.x - vx, v1.x - vx),
                                 pk(v0.y - vy, v1.y - vy), pk(v0.z - vz, v1.z - vz), mk, A);
        }
    };
    // keep every stack at <= V4_Q - 9 entries (8 pushes follow before the next check)
    auto drain_check = [&]() {
        for (;;) {
            const unsigned n = (qp - sQ) >> 6;
            if (!(__popc(__ballot_sync(0xffffffffu, n >= 2)) >= 24 || __any_sync(0xffffffffu, n >= V4_Q - 8)))
                break;
            PH_T0(td0)
            drain(std::false_type{});
            PH_ADD(3, td0);
        }
    };
    // candidates t .. t+3 of the window L[lb + ...] (SELF: the home cell, staged index base + t, minus i)
    auto step4 = [&](auto self_tag, unsigned lb, int base, int t, int total, int len0, unsigned fl0, unsigned fl1,
                     int kind) {
        constexpr bool SELF = decltype(self_tag)::value;
        bool ok[4];
        unsigned sj[4];
        float4 p[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            ok[u] = t + u < total && (!SELF || t + u != kh);
            if (SELF) {
                sj[u] = (unsigned)(base + (ok[u] ? t + u : 0));
            } else {
                const unsigned e = ldsr_u16(lb + 2u * (unsigned)(t + u));   // in the segment or just past it
                sj[u] = ok[u] ? e : 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) p[u] = ldsr_f4(S.P + 16u * sj[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float hx = x, hy = y, hz = z;
            unsigned fl = 0;
            if (FRAMES && !SELF) {
                fl = t + u < len0 ? fl0 : fl1;
                home_of(fl, hx, hy, hz);
            }
            const float dx = hx - p[u].x, dy = hy - p[u].y, dz = hz - p[u].z;
            const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            if (COUNT) cand[kind] += ok[u] ? 1u : 0u;
            if (ok[u] && r2 < H2) {
                sts_u16(qp, FRAMES ? (sj[u] | (fl << 12)) : sj[u]);
                qp += 64u;
                if (COUNT) ++hits[kind];
            }
        }
    };

    // candidates t .. t+3 of two consecutive windows (directions d0, d0 + 1 of a pair):
    // L[lb0 ...] for the first tot0, then L[lb1 ...]
    auto step4pair = [&](int t, unsigned lb0, int tot0, int len00, unsigned fl00, unsigned fl10, int kind0,
                         unsigned lb1m, int tot1, int len01, unsigned fl01, unsigned fl11, int kind1) {
        bool ok[4], in0[4];
        unsigned sj[4];
        float4 p[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int tt = t + u;
            in0[u] = tt < tot0;
            ok[u] = tt < tot0 + tot1;
            // lb1 - 2 tot0 precomputed: select the base, add 2 tt (2 u folds into the address)
            const unsigned e = ldsr_u16((in0[u] ? lb0 : lb1m) + 2u * (unsigned)t + 2u * (unsigned)u);
            sj[u] = ok[u] ? e : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) p[u] = ldsr_f4(S.P + 16u * sj[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float hx = x, hy = y, hz = z;
            unsigned fl = 0;
            if (FRAMES) {
                const int tt = t + u;
                fl = in0[u] ? (tt < len00 ? fl00 : fl10) : (tt - tot0 < len01 ? fl01 : fl11);
                home_of(fl, hx, hy, hz);
            }
            const float dx = hx - p[u].x, dy = hy - p[u].y, dz = hz - p[u].z;
            const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            const int kind = in0[u] ? kind0 : kind1;
            if (COUNT) cand[kind] += ok[u] ? 1u : 0u;
            if (ok[u] && r2 < H2) {
                sts_u16(qp, FRAMES ? (sj[u] | (fl << 12)) : sj[u]);
                qp += 64u;
                if (COUNT) ++hits[kind];
            }
        }
    };

    // the self cell: all j != i of the home cell
    {
        const int total = active ? eh.y : 0;
        const int trip = __reduce_max_sync(0xffffffffu, total);
        int t = 0;
        for (; t + 4 < trip; t += 8) {
            step4(std::true_type{}, 0u, eh.x, t, total, total, 0u, 0u, 0);
            step4(std::true_type{}, 0u, eh.x, t + 4, total, total, 0u, 0u, 0);
            drain_check();
        }
        if (t < trip) {
            step4(std::true_type{}, 0u, eh.x, t, total, total, 0u, 0u, 0);
            drain_check();
        }
    }
    int pos = lpos;                                       // this home cell's direction segments
    // reversed +d list, then reversed -d list, so that the lane's two windows (a prefix of +d,
    // a suffix of -d) are contiguous: L[wb, wb + total); directions in pairs for the searches
    for (int d0 = 0; d0 < 13; d0 += 2) {
        const int nd = d0 + 1 < 13 ? 2 : 1;
        int wbv[2] = {0, 0}, len0v[2] = {0, 0}, totv[2] = {0, 0};
        unsigned fl0v[2] = {0, 0}, fl1v[2] = {0, 0};
        int f[4] = {0, 0, 0, 0}, nn[4] = {0, 0, 0, 0};
        float hh[4][3];
        float Hkv[2] = {0.0f, 0.0f};
        int nmax = 0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int d = d0 + k;
            hh[2 * k][0] = hh[2 * k + 1][0] = x;
            hh[2 * k][1] = hh[2 * k + 1][1] = y;
            hh[2 * k][2] = hh[2 * k + 1][2] = z;
            if (k < nd) {
                const int kind = v4_kind(d);
                Hkv[k] = kind == 1 ? Hd : (kind == 2 ? Hd2 : Hd3);
                if (active) {
                    const int a0 = dir_component(d, 0), a1 = dir_component(d, 1), a2 = dir_component(d, 2);
                    const int4 ep = S.tab[scell(a0, a1, a2)];
                    const int4 em = S.tab[scell(-a0, -a1, -a2)];
                    const int mid = pos + ep.y;           // boundary between the two reversed segments
                    pos = mid + em.y;
                    f[2 * k] = mid - 1;
                    f[2 * k + 1] = mid;
                    nn[2 * k] = ep.y;
                    nn[2 * k + 1] = em.y;
                    wbv[k] = mid;
                    nmax = max(nmax, max(ep.y, em.y));
                    if (FRAMES) {
                        fl0v[k] = (unsigned)ep.w & 7u;
                        fl1v[k] = (unsigned)em.w & 7u;
                        home_of(fl0v[k], hh[2 * k][0], hh[2 * k][1], hh[2 * k][2]);
                        home_of(fl1v[k], hh[2 * k + 1][0], hh[2 * k + 1][1], hh[2 * k + 1][2]);
                    }
                }
            }
        }
        nmax = __reduce_max_sync(0xffffffffu, nmax);
        const int top = nmax > 0 ? 1 << (31 - __clz(nmax)) : 0;
        if (active) {
            int len[4];
            PH_T0(ts0)
            if (nd == 2) {
                v4_windows2(S, d0 >> 1, top, f, nn, hh, Hkv, len);
            } else {
                v4_windows(S, d0, top, f[0], nn[0], f[1], nn[1], hh[0][0], hh[0][1], hh[0][2], hh[1][0], hh[1][1],
                           hh[1][2], Hkv[0], len[0], len[1]);
                len[2] = len[3] = 0;
            }
            PH_ADD(1, ts0);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                len0v[k] = len[2 * k];
                totv[k] = len[2 * k] + len[2 * k + 1];
                wbv[k] -= len[2 * k];
            }
        }
        // one sweep over both directions' windows (one trip count for the pair)
        const int kind0 = v4_kind(d0), kind1 = nd == 2 ? v4_kind(d0 + 1) : 0;
        const int trip = __reduce_max_sync(0xffffffffu, totv[0] + totv[1]);
        const unsigned lb0 = S.L + 2u * (unsigned)wbv[0], lb1m = S.L + 2u * (unsigned)(wbv[1] - totv[0]);
        PH_T0(tw0)
        int t = 0;
        for (; t + 4 < trip; t += 8) {
            step4pair(t, lb0, totv[0], len0v[0], fl0v[0], fl1v[0], kind0, lb1m, totv[1], len0v[1], fl0v[1], fl1v[1],
                      kind1);
            step4pair(t + 4, lb0, totv[0], len0v[0], fl0v[0], fl1v[0], kind0, lb1m, totv[1], len0v[1], fl0v[1],
                      fl1v[1], kind1);
            drain_check();
        }
        if (t < trip) {                                   // a tail of <= 4 candidates
            step4pair(t, lb0, totv[0], len0v[0], fl0v[0], fl1v[0], kind0, lb1m, totv[1], len0v[1], fl0v[1], fl1v[1],
                      kind1);
            drain_check();
        }
        PH_ADD(2, tw0);
    }
    PH_T0(tf0)
    while (__any_sync(0xffffffffu, qp != sQ)) drain(std::true_type{});
    PH_ADD(4, tf0);

    if (active) {
        // finalise (self term w(0) = 1/2, t(0) = 3/2), as finalise() in density.cuh
        const float K3 = (16.0f / kPi) * Hinv * Hinv * Hinv;
        const float rho = K3 * fmaf(0.5f, m, sum2(A.rho));
        const float wc = K3 * (0.5f + sum2(A.wc));
        const float dh = -K3 * g.gamma * Hinv;
        const float rho_dh = dh * fmaf(1.5f, m, sum2(A.srt));
        const float wc_dh = dh * (1.5f + sum2(A.st));
        const float gf = K3 * Hinv;
        const float rinv = 1.0f / rho;
        store_rec(orec, c.perm[i], rho, wc, rho_dh, wc_dh, gf * sum2(A.Dn) * rinv, gf * (sum2(A.Px) - sum2(A.Nx)) * rinv,
                  gf * (sum2(A.Py) - sum2(A.Ny)) * rinv, gf * (sum2(A.Pz) - sum2(A.Nz)) * rinv, nngb);
    }
}

// Staged cell s of a tile (s = row * nzs + col; row = (ox + 1) * 4 + (oy + 1) relative to
// the tile's first row, col = uz - z_a + 1): local cell id and periodic flags (bits 0-2
// home shift for a +L image, bits 3-5 pre-shift of a -L image).
struct TileGeom {
    int xo, y0, za, zb, first, cnt, nzs, nzh, nh;
    bool hasB, staged, frames;
};

__device__ __forceinline__ TileGeom tile_geom(const DevGrid &g, const RowPairs &rp, int4 td)
{
    TileGeom t;
    int yp;
    key_rowpair(rp, td.x, t.xo, yp);
    t.y0 = 2 * yp;
    t.hasB = t.y0 + 1 < g.ny;
    t.za = td.y & 0xffff;
    t.zb = td.y >> 16;
    t.first = td.z;
    t.cnt = td.w;
    t.nzs = t.zb - t.za + 3;
    t.nzh = t.zb - t.za + 1;
    t.nh = (t.hasB ? 2 : 1) * t.nzh;
    t.staged = t.cnt > 0 && t.nzs <= V4_MAXZ;
    // a staged neighbour beyond a high face (home shift needed): x plane, y row or z column
    t.frames = g.x_lo + t.xo + 1 >= g.nc[0] || t.y0 + 2 >= g.ny || t.zb + 1 >= g.nz;
    return t;
}

__device__ __forceinline__ long long staged_cell(const DevGrid &g, const TileGeom &t, int s, unsigned &fl)
{
    const int r = s / t.nzs, q = s % t.nzs;
    const StagedRow sr = staged_row(g, t.xo, t.y0, r);
    const int uz = t.za - 1 + q;
    fl = (sr.gx >= g.nc[0] ? 1u : 0u) | (sr.uy >= g.ny ? 2u : 0u) | (uz >= g.nz ? 4u : 0u) | (sr.gx < 0 ? 8u : 0u) |
         (sr.uy < 0 ? 16u : 0u) | (uz < 0 ? 32u : 0u);
    return sr.base + wrap_i(uz, g.nz);
}

// Persistent CTAs take tiles in order from an atomic counter.  The next tile's
// descriptor and the cell counts of its staged neighbourhood are fetched while the
// current tile computes, so staging starts without a global-memory round trip.
template <bool COUNT>
__global__ void __launch_bounds__(V4_TP, V4_CTAS) k_density_v4(DevGrid g, DevCells c, OutRec *orec, sph_stats *st,
                                                         const int4 *__restrict__ tiles,
                                                         const int *__restrict__ ntiles_p, int *tile_counter,
                                                         const unsigned *__restrict__ genp)
{
    extern __shared__ __align__(16) unsigned char v4_smem[];
    float4 *P = reinterpret_cast<float4 *>(v4_smem);
    float4 *V = P + V4_MS;
    int4 *tab = reinterpret_cast<int4 *>(V + V4_MS);
    uint16_t *L = reinterpret_cast<uint16_t *>(tab + V4_MAXCELLS);
    int *hoff = reinterpret_cast<int *>(L + V4_ML);
    uint16_t *queue = reinterpret_cast<uint16_t *>(hoff + V4_HOFF);
    int4 *seq = reinterpret_cast<int4 *>(queue + V4_WARPS * V4_Q * 32);
    __shared__ int4 s_next;
    __shared__ int s_wsum[V4_WARPS];
    __shared__ __align__(8) unsigned long long s_mbar;
    const unsigned mbar = smem_addr(&s_mbar);
    unsigned mbar_phase = 0;
    static_assert(V4_MAXCELLS <= 2 * V4_TP, "two table entries per thread");

    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const RowPairs rp = row_pairs(g);
    const int ntiles = *ntiles_p;
    unsigned cand[4] = {0, 0, 0, 0}, hits[4] = {0, 0, 0, 0};
    const int4 kEnd = make_int4(-1, 0, 0, 0);

    // prefetch of a tile's staged-cell counts: thread owns table entries 2 tid, 2 tid + 1
    int pf_start[2] = {0, 0}, pf_end[2] = {0, 0}, pf_nh[2] = {0, 0};
    auto prefetch = [&](int4 td) {
        if (td.x < 0) return;
        const TileGeom t = tile_geom(g, rp, td);
        if (!t.staged) return;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int s = 2 * threadIdx.x + k;
            if (s < V4_ROWS * t.nzs) {
                unsigned fl;
                const long long cell = staged_cell(g, t, s, fl);
                pf_start[k] = c.cell_start[cell];
                pf_end[k] = c.cell_start[cell + 1];
                pf_nh[k] = c.cell_nhome[cell];
            }
        }
    };
    if (threadIdx.x == 0) {
        const int t0 = atomicAdd(tile_counter, 1);
        s_next = t0 < ntiles ? tiles[t0] : kEnd;
        s_gen = *genp;
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int4 td = s_next;
    prefetch(td);

    while (td.x >= 0) {
        PH_T0(tb0)
        __syncthreads();                                  // s_next consumed by every thread
        PH_ADD(5, tb0);
        PH_T0(tst0)
        if (threadIdx.x == 0) {                           // claim the next tile early
            const int t1 = atomicAdd(tile_counter, 1);
            s_next = t1 < ntiles ? tiles[t1] : kEnd;
        }
        const TileGeom T = tile_geom(g, rp, td);
        bool staged = T.staged;
        if (staged) {
            // staged cell table from the prefetched counts
            const int ncs = V4_ROWS * T.nzs;
            int cnt2[2] = {0, 0};
            int4 ent[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int s = 2 * threadIdx.x + k;
                ent[k] = make_int4(0, 0, 0, 0);
                if (s < ncs) {
                    unsigned fl;
                    staged_cell(g, T, s, fl);
                    cnt2[k] = pf_end[k] - pf_start[k];
                    ent[k] = make_int4(0, cnt2[k], pf_start[k], (int)fl | (pf_nh[k] << 8));   // w: flags | home count << 8
                }
            }
            // counts first; bases and list offsets then come from ONE block scan of packed
            // (particles | list entries << 16) values (both totals < 2^16: V4_MS, V4_ML)
            if (2 * threadIdx.x < ncs) tab[2 * threadIdx.x] = ent[0];
            if (2 * threadIdx.x + 1 < ncs) tab[2 * threadIdx.x + 1] = ent[1];
            __syncthreads();
            // list segments: for home cell h, segment k = 2 d (+d neighbour) or 2 d + 1 (-d),
            // d = 0..12; global segment g = 26 h + k (4 per thread, consecutive)
            static_assert(26 * V4_MAXH <= 4 * V4_TP, "four list segments per thread");
            static_assert(V4_MS < 65536 && V4_ML < 65536, "packed scan");
            const int nseg = 26 * T.nh;
            int ssz[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int gseg = 4 * threadIdx.x + j;
                ssz[j] = 0;
                if (gseg < nseg) {
                    const int h = gseg / 26, k = gseg % 26, d = k >> 1, sg = (k & 1) ? -1 : 1;
                    const int r = h / T.nzh, q = h % T.nzh + 1;
                    ssz[j] = tab[((sg * dir_component(d, 0) + 1) * 4 + sg * dir_component(d, 1) + r + 1) * T.nzs + q +
                                 sg * dir_component(d, 2)].y;
                }
            }
            if (wl == V4_WARPS - 1) {
                // slice k: {A start, A count, B start, first sequence index}, k < nzh
                int4 sl = make_int4(0, 0, 0, 0);
                int ns = 0;
                if (lane < T.nzh) {
                    // home particles lead each cell: {A start, A home count, B start}
                    const int4 ea = tab[5 * T.nzs + lane + 1];
                    const int4 eb = tab[6 * T.nzs + lane + 1];
                    sl = make_int4(ea.z, ea.w >> 8, eb.z, 0);
                    ns = (ea.w >> 8) + (T.hasB ? (eb.w >> 8) : 0);
                }
                int x = ns;
#pragma unroll
                for (int o2 = 1; o2 < 32; o2 <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, o2);
                    if (lane >= o2) x += y;
                }
                sl.w = x - ns;
                if (lane < T.nzh) seq[lane] = sl;
            }
            int ptot;
            PH_T0(tsc0)
            const int pp = block_exscan((cnt2[0] + cnt2[1]) | ((ssz[0] + ssz[1] + ssz[2] + ssz[3]) << 16), s_wsum, ptot);
            PH_ADD(8, tsc0);
            const int total = ptot & 0xffff, ltotal = ptot >> 16;
            const int pre = pp & 0xffff;
            int lpre = pp >> 16;
            if (2 * threadIdx.x < ncs) tab[2 * threadIdx.x].x = pre;
            if (2 * threadIdx.x + 1 < ncs) tab[2 * threadIdx.x + 1].x = pre + cnt2[0];
            int *segoff = reinterpret_cast<int *>(queue);        // scratch: the hit stacks are idle now
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int gseg = 4 * threadIdx.x + j;
                if (gseg < nseg) {
                    segoff[gseg] = lpre;
                    if (gseg % 26 == 0) hoff[gseg / 26] = lpre;
                }
                lpre += ssz[j];
            }
            if (total > V4_MS || ltotal > V4_ML || T.nh > V4_MAXH) staged = false;   // CTA-uniform
            __syncthreads();
            if (staged) {
                // positions and (v, m): bulk copies (the TMA engine) of each staged row's contiguous
                // slot ranges (split where z wraps), issued by warp 0 and overlapped with the list copy
                PH_T0(tpv0)
                if (wl == 0) {
                    if (lane == 0) mbar_expect_tx(mbar, (unsigned)total * 32u);
                    __syncwarp();
                    const bool wlo = T.za == 0, whi = T.zb + 1 >= g.nz;
                    for (int job = lane; job < V4_ROWS * 3; job += 32) {
                        const int r = job / 3, piece = job % 3;
                        // piece 0: column 0 if it wraps (uz = -1); 1: the in-box columns; 2: last column if uz = nz
                        const int q0 = piece == 0 ? 0 : (piece == 1 ? (wlo ? 1 : 0) : T.nzs - 1);
                        const int q1 = piece == 0 ? (wlo ? 1 : 0) : (piece == 1 ? (whi ? T.nzs - 1 : T.nzs) : (whi ? T.nzs : T.nzs - 1));
                        if (q1 <= q0) continue;
                        const int4 ea = tab[r * T.nzs + q0];
                        const int4 eb = tab[r * T.nzs + q1 - 1];
                        const unsigned bytes = (unsigned)(eb.x + eb.y - ea.x) * 16u;
                        if (bytes == 0) continue;
                        bulk_g2s(smem_addr(P + ea.x), c.xyzh + ea.z, bytes, mbar);
                        bulk_g2s(smem_addr(V + ea.x), c.vm + ea.z, bytes, mbar);
                    }
                }
                PH_ADD(6, tpv0);
                PH_T0(tl0)
                // list segments, strided over the threads (balanced): the sorted list reversed,
                // entries turned into staged indices
                for (int gseg = threadIdx.x; gseg < nseg; gseg += V4_TP) {
                    const int h = gseg / 26, k = gseg % 26, d = k >> 1, sg = (k & 1) ? -1 : 1;
                    const int r = h / T.nzh, q = h % T.nzh + 1;
                    const int4 e = tab[((sg * dir_component(d, 0) + 1) * 4 + sg * dir_component(d, 1) + r + 1) * T.nzs + q +
                                       sg * dir_component(d, 2)];
                    const int dst = segoff[gseg] + e.y - 1;
                    // aligned 16-byte words over the segment: an eighth of the L1 wavefronts of
                    // 2-byte loads (each lane of a warp reads a different segment)
                    const uint16_t *src = c.ord + (long long)d * c.cap + e.z;
                    const int mis = (int)(((uintptr_t)src >> 1) & 7);
                    const uint4 *wsrc = reinterpret_cast<const uint4 *>(src - mis);
                    const int nw = (mis + e.y + 7) >> 3;
                    for (int w0 = 0; w0 < nw; w0 += 4) {
                        uint4 v[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) v[u] = w0 + u < nw ? __ldg(wsrc + w0 + u) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int k = 8 * (w0 + u) - mis;       // list index of the word's first entry
                            const unsigned wd[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                            for (int t = 0; t < 8; ++t) {
                                const unsigned q = (t & 1) ? wd[t >> 1] >> 16 : wd[t >> 1] & 0xffffu;
                                if (k + t >= 0 && k + t < e.y) L[dst - k - t] = (uint16_t)(e.x + (int)q);
                            }
                        }
                    }
                }
                PH_ADD(7, tl0);
                mbar_wait(mbar, mbar_phase);
                mbar_phase ^= 1u;
                if (T.za == 0 || T.y0 == 0 || g.x_lo + T.xo == 0) {
                    __syncthreads();
                    // staged cells of a -L periodic image (flags 3-5): x_j - L, exact (x_j >= L/2)
                    for (int sc = wl; sc < V4_ROWS * T.nzs; sc += V4_WARPS) {
                        const int4 e = tab[sc];
                        if (!(e.w & 56)) continue;
                        const float sx = (e.w & 8) ? g.boxf[0] : 0.0f;
                        const float sy = (e.w & 16) ? g.boxf[1] : 0.0f;
                        const float sz = (e.w & 32) ? g.boxf[2] : 0.0f;
                        for (int k = lane; k < e.y; k += 32) {
                            float4 q = P[e.x + k];
                            q.x -= sx;
                            q.y -= sy;
                            q.z -= sz;
                            P[e.x + k] = q;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // the next tile: descriptor published by thread 0 (visible after the barrier above, or
        // the one below for unstaged tiles); its counts are fetched while this tile computes
        __syncthreads();
        PH_ADD(0, tst0);
        const int4 td_next = s_next;
        prefetch(td_next);

        // home particle of thread h: sequence index first + h from slice za on
        auto home_slot = [&](int h, int &slot, int &yo, int &tz) {
            const int qq = T.first + h;
            int lo = 0, hi = T.nzh - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (seq[mid].w <= qq) lo = mid; else hi = mid - 1;
            }
            const int4 e = seq[lo];
            const int loc = qq - e.w;
            yo = loc < e.y ? 0 : 1;
            slot = yo == 0 ? e.x + loc : e.z + (loc - e.y);
            tz = lo;
        };
        if (staged) {
            const int h = threadIdx.x;
            const bool active = h < T.cnt;
            int i = 0, yoff = 0, tz = 0, lpos = 0;
            if (active) {
                home_slot(h, i, yoff, tz);
                lpos = hoff[yoff * T.nzh + tz];
            } else {
                i = seq[0].x;
            }
            const V4Stage S{smem_addr(P), smem_addr(V), smem_addr(L), tab, T.nzs};
            const unsigned qb = smem_addr(queue + wl * V4_Q * 32);
            if (wl * 32 < T.cnt) {
                if (T.frames)
                    v4_particle_staged<COUNT, true>(g, c, orec, S, qb, active, i, yoff, tz + 1, lpos, cand, hits);
                else
                    v4_particle_staged<COUNT, false>(g, c, orec, S, qb, active, i, yoff, tz + 1, lpos, cand, hits);
            }
        } else if (T.cnt > 0) {
            // global-memory sweep: a tile whose staging check failed (the slices the builder
            // could not stage, cnt < 0, go to k_density_dense)
            const long long rowA = ((long long)(T.xo + g.ghost_x) * g.ny + T.y0) * g.nz;
            const int ntot = T.cnt > 0 ? T.cnt : -T.cnt;
            for (int h = threadIdx.x; h < ntot; h += V4_TP) {
                // slices from z_a on: row-A cell then row-B cell
                int qq = T.first + h, z = T.za, slot = 0;
                for (;; ++z) {
                    const long long ca = rowA + z;
                    const int a0 = c.cell_start[ca], na = c.cell_nhome[ca];
                    const int b0 = T.hasB ? c.cell_start[ca + g.nz] : 0;
                    const int nb = T.hasB ? c.cell_nhome[ca + g.nz] : 0;
                    if (qq < na) { slot = a0 + qq; break; }
                    if (qq < na + nb) { slot = b0 + (qq - na); break; }
                    qq -= na + nb;
                }
                v4_particle_global<COUNT>(g, c, orec, slot, cand, hits);
            }
        }
        td = td_next;
    }
    flush_stats<COUNT>(st, cand, hits);
}

}  // namespace pvsph
