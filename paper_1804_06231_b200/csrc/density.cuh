// density.cuh -- the SPH density interaction and the
// pseudo-Verlet pair sweep (Code 2, final loop).
//
// Reference ("v1") engine: one warp per home cell, lane = particle i of the
// cell (chunks of 32), the self cell and the 26 neighbour cells swept in a
// fixed order, each neighbour through its sorted list along the pair's axis
// with the per-particle window of P:151-165 (exact per i: the sweep stops at
// the first sorted j whose projected separation reaches H_i + delta).
// Accumulates in registers and writes once per particle.
//
// Separations use the exact-difference rule of DESIGN.md §4.3: for a pair
// wrapped across the periodic boundary L is subtracted from whichever
// coordinate is >= L/2 (exact by Sterbenz), never added to one near 0.
#pragma once

#include "common.cuh"
#include "packed.cuh"

namespace pvsph {

struct Acc {
    float rho, wc, srt, st, D, Rx, Ry, Rz;
    int nngb;
};

struct IPart {
    float x, y, z;       // position (fp32 input)
    float vx, vy, vz, m, h;
    float H2;            // (gamma h)^2
    float Hinv;          // 1 / (gamma h)
    float Hd;            // gamma h + delta
    double u0, u1, u2;   // local coordinates in the home cell (fp64)
    int slot;
};

__device__ __forceinline__ void acc_zero(Acc &a)
{
    a.rho = a.wc = a.srt = a.st = a.D = a.Rx = a.Ry = a.Rz = 0.0f;
    a.nngb = 0;
}

// M4 cubic spline shape w(x) and w'(x), x = r/H in [0, 1).
__device__ __forceinline__ void m4(float x, float &w, float &dw)
{
    if (x < 0.5f) {
        w = fmaf(x * x, fmaf(3.0f, x, -3.0f), 0.5f);
        dw = x * fmaf(9.0f, x, -6.0f);
    } else {
        float u = 1.0f - x;
        w = u * u * u;
        dw = -3.0f * u * u;
    }
}

// One in-range neighbour j of i (raw sums; scaled in finalise).
__device__ __forceinline__ void interact(const IPart &p, float dx, float dy, float dz, float r2, float4 vmj, Acc &a)
{
    float rinv = r2 > 0.0f ? rsqrt_nr(r2) : 0.0f;
    float r = r2 * rinv;
    float x = r * p.Hinv;
    float w, dw;
    m4(x, w, dw);
    float mj = vmj.w;
    a.rho = fmaf(mj, w, a.rho);
    a.wc += w;
    float t = fmaf(x, dw, 3.0f * w);
    a.srt = fmaf(mj, t, a.srt);
    a.st += t;
    float dvx = p.vx - vmj.x, dvy = p.vy - vmj.y, dvz = p.vz - vmj.z;
    float vdx = fmaf(dvx, dx, fmaf(dvy, dy, dvz * dz));
    float fac = mj * dw * rinv;
    a.D = fmaf(fac, vdx, a.D);
    a.Rx = fmaf(fac, fmaf(dvy, dz, -dvz * dy), a.Rx);
    a.Ry = fmaf(fac, fmaf(dvz, dx, -dvx * dz), a.Ry);
    a.Rz = fmaf(fac, fmaf(dvx, dy, -dvy * dx), a.Rz);
    a.nngb += 1;
}

__device__ __forceinline__ IPart load_i(const DevGrid &g, const DevCells &c, int slot, const double corner[3])
{
    IPart p;
    float4 a = c.xyzh[slot];
    float4 b = c.vm[slot];
    p.x = a.x; p.y = a.y; p.z = a.z; p.h = a.w;
    p.vx = b.x; p.vy = b.y; p.vz = b.z; p.m = b.w;
    double H = (double)g.gamma * (double)a.w;   // exact product; H^2, 1/H rounded once
    p.H2 = (float)(H * H);
    p.Hinv = (float)(1.0 / H);
    p.Hd = (float)H + g.delta;
    p.u0 = (double)a.x - corner[0];
    p.u1 = (double)a.y - corner[1];
    p.u2 = (double)a.z - corner[2];
    p.slot = slot;
    return p;
}

// Self cell: all j != i of the home cell, in the order of its d = 0 list.  Batches of four
// candidates keep their global loads in flight together (the loop is latency-bound).
template <bool COUNT>
__device__ __forceinline__ void sweep_self(const DevCells &c, const IPart &p, int s0, int s1, Acc &a,
                                           unsigned &cand, unsigned &hits)
{
    for (int q0 = s0; q0 < s1; q0 += 4) {
        int j[4];
        float4 e[4], v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) j[u] = q0 + u < s1 ? s0 + c.ord[q0 + u] : p.slot;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            e[u] = c.xyzh[j[u]];
            v[u] = c.vm[j[u]];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (j[u] == p.slot) continue;                  // i itself, or past the cell
            float dx = p.x - e[u].x, dy = p.y - e[u].y, dz = p.z - e[u].z;
            float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            if (COUNT) ++cand;
            if (r2 < p.H2) {
                interact(p, dx, dy, dz, r2, v[u], a);
                if (COUNT) ++hits;
            }
        }
    }
}

// Unit vector of sort direction d (fp32).
__device__ __forceinline__ void dir_unit(int d, float &ax, float &ay, float &az)
{
    const int a0 = dir_component(d, 0), a1 = dir_component(d, 1), a2 = dir_component(d, 2);
    const int kd = (a0 != 0) + (a1 != 0) + (a2 != 0);
    const float inv = kd == 1 ? 1.0f : (kd == 2 ? 0.70710678118654752f : 0.57735026918962576f);
    ax = (float)a0 * inv;
    ay = (float)a1 * inv;
    az = (float)a2 * inv;
}

// Neighbour cell at offset (ox,oy,oz) with periodic-image flags sh[k] in
// {-1,0,+1} (neighbour lies beyond the low / high face of the box).  The list
// of cj sorted along d = canon(o) is swept from the end nearest to the home
// cell; the sweep stops at the first j whose projected separation
// sep = (x_j - x_i) . o/|o| reaches H_i + delta (Code 2; the per-particle
// bound of P:156).  sep is computed from the exact coordinate differences, so no
// cell corner enters.
template <bool COUNT>
__device__ __forceinline__ void sweep_pair(const DevGrid &g, const DevCells &c, const IPart &p, int cj, int ox, int oy,
                                           int oz, const int sh[3], Acc &a, unsigned &cand, unsigned &hits)
{
    int s;
    int d = canon_dir(ox, oy, oz, s);
    float ax, ay, az;
    dir_unit(d, ax, ay, az);
    const float sx = -s * ax, sy = -s * ay, sz = -s * az;   // sep = (dx, dy, dz) . (sx, sy, sz), dx = x_i - x_j
    // exact-difference coordinates
    float xi = sh[0] > 0 ? p.x - g.boxf[0] : p.x;
    float yi = sh[1] > 0 ? p.y - g.boxf[1] : p.y;
    float zi = sh[2] > 0 ? p.z - g.boxf[2] : p.z;
    float sjx = sh[0] < 0 ? g.boxf[0] : 0.0f;
    float sjy = sh[1] < 0 ? g.boxf[1] : 0.0f;
    float sjz = sh[2] < 0 ? g.boxf[2] : 0.0f;
    const uint16_t *L = c.ord + (long long)d * c.cap;
    int s0 = c.cell_start[cj], s1 = c.cell_start[cj + 1];
    const int n = s1 - s0;
    // batches of four in sweep order (loads in flight together); the sweep stops at the first
    // candidate whose projected separation reaches H_i + delta
    for (int k0 = 0; k0 < n; k0 += 4) {
        int j[4];
        float4 e[4], v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = min(k0 + u, n - 1);
            j[u] = s0 + L[s > 0 ? s0 + k : s1 - 1 - k];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            e[u] = c.xyzh[j[u]];
            v[u] = c.vm[j[u]];
        }
        bool stop = false;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (stop || k0 + u >= n) break;
            float dx = xi - (e[u].x - sjx), dy = yi - (e[u].y - sjy), dz = zi - (e[u].z - sjz);
            if (!(fmaf(dx, sx, fmaf(dy, sy, dz * sz)) < p.Hd)) {   // sorted early exit
                stop = true;
                break;
            }
            float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            if (COUNT) ++cand;
            if (r2 < p.H2) {
                interact(p, dx, dy, dz, r2, v[u], a);
                if (COUNT) ++hits;
            }
        }
        if (stop) break;
    }
}

// Final values from the raw sums (self term w(0) = 1/2, t(0) = 3/2).
struct Final {
    float rho, wc, rho_dh, wc_dh, div, cx, cy, cz;
};

__device__ __forceinline__ Final finalise(const DevGrid &g, const IPart &p, const Acc &a, bool self_term)
{
    float Hinv = p.Hinv;
    float K3 = (16.0f / kPi) * Hinv * Hinv * Hinv;
    float st = self_term ? 1.0f : 0.0f;
    Final f;
    f.rho = K3 * fmaf(0.5f * st, p.m, a.rho);
    f.wc = K3 * (0.5f * st + a.wc);
    float dh = -K3 * g.gamma * Hinv;
    f.rho_dh = dh * fmaf(1.5f * st, p.m, a.srt);
    f.wc_dh = dh * (1.5f * st + a.st);
    float gf = K3 * Hinv;
    f.div = -gf * a.D;   // rho * div v
    f.cx = gf * a.Rx;    // rho * curl v
    f.cy = gf * a.Ry;
    f.cz = gf * a.Rz;
    return f;
}

// Home cell coordinates of local cell `cell`, its global x plane, corner.
struct HomeCell {
    int ixl, iy, iz, ixg;
    double corner[3];
};

__device__ __forceinline__ HomeCell home_cell(const DevGrid &g, long long cell)
{
    HomeCell h;
    long long plane = (long long)g.ny * g.nz;
    h.ixl = (int)(cell / plane);
    h.iy = (int)((cell / g.nz) % g.ny);
    h.iz = (int)(cell % g.nz);
    h.ixg = wrap_i(h.ixl - g.ghost_x + g.x_lo, g.nc[0]);
    h.corner[0] = (double)h.ixg * g.cl[0];
    h.corner[1] = (double)h.iy * g.cl[1];
    h.corner[2] = (double)h.iz * g.cl[2];
    return h;
}

// Neighbour at offset o of a home cell: local cell id and periodic flags.
// Returns false if it falls outside the local grid (ghost home cells only).
__device__ __forceinline__ bool neighbour(const DevGrid &g, const HomeCell &h, int ox, int oy, int oz, int &cj,
                                          int sh[3])
{
    int jxl, jy = h.iy + oy, jz = h.iz + oz;
    int gx = h.ixg + ox;
    sh[0] = gx < 0 ? -1 : (gx >= g.nc[0] ? 1 : 0);
    if (g.ghost_x) {
        jxl = h.ixl + ox;
        if (jxl < 0 || jxl >= g.nxl) return false;
    } else {
        jxl = wrap_i(h.ixl + ox, g.nc[0]);
    }
    sh[1] = jy < 0 ? -1 : (jy >= g.ny ? 1 : 0);
    sh[2] = jz < 0 ? -1 : (jz >= g.nz ? 1 : 0);
    jy = wrap_i(jy, g.ny);
    jz = wrap_i(jz, g.nz);
    cj = (jxl * g.ny + jy) * g.nz + jz;
    return true;
}

__device__ __forceinline__ int kind_of(int ox, int oy, int oz)
{
    return (ox != 0) + (oy != 0) + (oz != 0);
}

template <bool COUNT>
__device__ __forceinline__ void flush_stats(sph_stats *st, const unsigned cand[4], const unsigned hits[4],
                                            unsigned band = 0)
{
    if (!COUNT || !st) return;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        unsigned long long cv = cand[k], hv = hits[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cv += __shfl_xor_sync(0xffffffffu, cv, o);
            hv += __shfl_xor_sync(0xffffffffu, hv, o);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&st->cand[k], cv);
            atomicAdd(&st->hits[k], hv);
        }
    }
    unsigned long long bv = band;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bv += __shfl_xor_sync(0xffffffffu, bv, o);
    if ((threadIdx.x & 31) == 0 && bv) atomicAdd(&st->band, bv);
}

// ---- sph_density_all, reference engine: one warp per owned home cell -------
constexpr int V1_WARPS = 4;

template <bool COUNT>
__global__ void __launch_bounds__(V1_WARPS * 32) k_density_all_v1(DevGrid g, DevCells c, DevOut o, sph_stats *st)
{
    const int lane = threadIdx.x & 31;
    long long w = (long long)blockIdx.x * V1_WARPS + (threadIdx.x >> 5);
    unsigned cand[4] = {0, 0, 0, 0}, hits[4] = {0, 0, 0, 0};
    if (w < g.n_owned_cells) {
        long long plane = (long long)g.ny * g.nz;
        long long cell = (w / plane + g.ghost_x) * plane + (w % plane);
        HomeCell hc = home_cell(g, cell);
        int s0 = c.cell_start[cell], s1 = c.cell_start[cell + 1];
        for (int base = s0; base < s1; base += 32) {
            int i = base + lane;
            if (i >= s1) break;
            IPart p = load_i(g, c, i, hc.corner);
            Acc a;
            acc_zero(a);
            sweep_self<COUNT>(c, p, s0, s1, a, cand[0], hits[0]);
            for (int ox = -1; ox <= 1; ++ox)
                for (int oy = -1; oy <= 1; ++oy)
                    for (int oz = -1; oz <= 1; ++oz) {
                        if (!(ox | oy | oz)) continue;
                        int cj, sh[3];
                        if (!neighbour(g, hc, ox, oy, oz, cj, sh)) continue;
                        int k = kind_of(ox, oy, oz);
                        sweep_pair<COUNT>(g, c, p, cj, ox, oy, oz, sh, a, cand[k], hits[k]);
                    }
            Final f = finalise(g, p, a, true);
            int out = c.perm[i];
            if (out < o.n_out) {
                float rinv = 1.0f / f.rho;
                o.rho[out] = f.rho;
                o.wcount[out] = f.wc;
                o.rho_dh[out] = f.rho_dh;
                o.wcount_dh[out] = f.wc_dh;
                o.div_v[out] = f.div * rinv;
                o.curl_v[out] = f.cx * rinv;
                o.curl_v[o.n_out + out] = f.cy * rinv;
                o.curl_v[2 * o.n_out + out] = f.cz * rinv;
                o.nngb[out] = a.nngb;
            }
        }
    }
    flush_stats<COUNT>(st, cand, hits);
}

// ---- accumulating API kernels (sph_density_self / sph_density_pair) -------
__device__ __forceinline__ void atomic_out(const DevOut &o, int out, const Final &f, int nngb)
{
    if (out >= o.n_out) return;
    atomicAdd(&o.rho[out], f.rho);
    atomicAdd(&o.wcount[out], f.wc);
    atomicAdd(&o.rho_dh[out], f.rho_dh);
    atomicAdd(&o.wcount_dh[out], f.wc_dh);
    atomicAdd(&o.div_v[out], f.div);
    atomicAdd(&o.curl_v[out], f.cx);
    atomicAdd(&o.curl_v[o.n_out + out], f.cy);
    atomicAdd(&o.curl_v[2 * o.n_out + out], f.cz);
    atomicAdd(&o.nngb[out], nngb);
}

// The same without atomics, for passes whose launches write disjoint particles (the colour
// phases of sph_density_all_sym): a read-modify-write in a fixed order, so deterministic.
__device__ __forceinline__ void plain_out(const DevOut &o, int out, const Final &f, int nngb)
{
    if (out >= o.n_out) return;
    o.rho[out] += f.rho;
    o.wcount[out] += f.wc;
    o.rho_dh[out] += f.rho_dh;
    o.wcount_dh[out] += f.wc_dh;
    o.div_v[out] += f.div;
    o.curl_v[out] += f.cx;
    o.curl_v[o.n_out + out] += f.cy;
    o.curl_v[2 * o.n_out + out] += f.cz;
    o.nngb[out] += nngb;
}

__device__ __forceinline__ bool owned_cell(const DevGrid &g, long long cell)
{
    long long plane = (long long)g.ny * g.nz;
    if (cell < 0 || cell >= g.ncell) return false;
    int ixl = (int)(cell / plane);
    return ixl >= g.ghost_x && ixl < g.nxl - g.ghost_x;
}

constexpr int API_WARPS = 4;

template <bool COUNT>
// nlist < 0: |nlist| is the list's stride in ints and nlist_dev the device-side count (the
// self pass of sph_density_all_sym reads the first int of its (c, c) records).
__global__ void __launch_bounds__(API_WARPS * 32) k_density_self(DevGrid g, DevCells c, DevOut o, const int *list,
                                                                  long long nlist, sph_stats *st, unsigned *status,
                                                                  const int *nlist_dev = nullptr)
{
    const int lane = threadIdx.x & 31;
    long long w = (long long)blockIdx.x * API_WARPS + (threadIdx.x >> 5);
    unsigned cand[4] = {0, 0, 0, 0}, hits[4] = {0, 0, 0, 0};
    const long long stride = nlist < 0 ? -nlist : 1;
    if (nlist < 0) nlist = nlist_dev ? *nlist_dev : 0;
    if (w < nlist) {
        long long cell = list[w * stride];
        if (!owned_cell(g, cell)) {
            if (lane == 0) set_status(status, ST_EINVAL);
        } else {
            HomeCell hc = home_cell(g, cell);
            int s0 = c.cell_start[cell], s1 = c.cell_start[cell + 1];
            for (int base = s0; base < s1; base += 32) {
                int i = base + lane;
                if (i >= s1) break;
                IPart p = load_i(g, c, i, hc.corner);
                Acc a;
                acc_zero(a);
                sweep_self<COUNT>(c, p, s0, s1, a, cand[0], hits[0]);
                atomic_out(o, c.perm[i], finalise(g, p, a, true), a.nngb);
            }
        }
    }
    flush_stats<COUNT>(st, cand, hits);
}

__global__ void k_finalize(DevOut o, long long n)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        float r = o.rho[i];
        float rinv = r != 0.0f ? 1.0f / r : 0.0f;
        o.div_v[i] *= rinv;
        o.curl_v[i] *= rinv;
        o.curl_v[o.n_out + i] *= rinv;
        o.curl_v[2 * o.n_out + i] *= rinv;
    }
}

}  // namespace pvsph
