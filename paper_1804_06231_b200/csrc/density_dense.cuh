// density_dense.cuh -- the tiles k_v4_tiles cannot stage (a slice whose 12-row neighbourhood
// exceeds the tile's shared memory: dense clustered cells, c4) as a warp-level engine
// (DESIGN.md §4.4).
//
//  * Work: the builder lists these tiles (each one slice: at most two home cells, <= V4_TP
//    home particles); a warp claims a tile and takes its home cells in chunks of 32
//    particles (lane = i), in the order of the home cell's list along DENSE_SELF_DIR (z), so
//    the 32 lanes are neighbours along z.  No CTA barrier anywhere: warps run independently.
//  * Per neighbour cell (26, then the home cell itself) the warp stages the cell's sorted list
//    from the end nearest to the home cell, DENSE_K entries at a time, as positions (low-face
//    images pre-shifted by -L) and (v, m) in its own shared-memory slice.  Each lane's window
//    (the exact per-particle bound) is found by bisection inside the chunk; a
//    further chunk is staged only while some lane's window runs past the current one, so a
//    huge neighbour cell costs only its near part.  The home cell itself is swept the same
//    way along its z list, up and down from the warp's lowest position (R19): a
//    cell of n particles with H << C_l costs ~n 2H/C_l candidates per particle, not n.
//  * Hits go to the lane's LIFO stack and are drained two at a time with FFMA2 (as in
//    k_density_v4); a chunk's hits are drained before the chunk is overwritten.  Sums stay
//    in registers; one 64-byte record per particle at its input index (no atomics).
#pragma once

#include "common.cuh"
#include "density.cuh"
#include "density_v4.cuh"
#include "packed.cuh"

namespace pvsph {

constexpr int DENSE_WARPS = 8;
#ifndef DENSE_K_ENTRIES
#define DENSE_K_ENTRIES 128   // A/B on c4: 64 / 96 / 128 / 160 / 256 / 512 -> density 23.9 / 24.1 / 23.8 / 24.1 / 24.2 / 30.5 ms
#endif
#ifndef DENSE_Q_DEPTH
#define DENSE_Q_DEPTH 16
#endif
constexpr int DENSE_K = DENSE_K_ENTRIES; // staged entries per chunk (per warp)
constexpr int DENSE_Q = DENSE_Q_DEPTH;   // hit stack depth per lane
constexpr int DENSE_MAP = 256;           // home rank -> sorted position map of one tile part (>= V4_TP)
constexpr size_t DENSE_WARP_SMEM = (size_t)DENSE_K * 32 + (size_t)DENSE_Q * 32 * 2 + (size_t)DENSE_MAP * 2;
static_assert(DENSE_MAP >= V4_TP, "a tile part holds at most V4_TP home particles");
constexpr size_t DENSE_SMEM = DENSE_WARP_SMEM * DENSE_WARPS;

template <bool COUNT>
__global__ void __launch_bounds__(DENSE_WARPS * 32, 2) k_density_dense(DevGrid g, DevCells c, OutRec *orec,
                                                                       sph_stats *st, const int4 *__restrict__ tiles,
                                                                       const int *__restrict__ gtiles,
                                                                       const int *__restrict__ gcount, int *counter,
                                                                       const unsigned *__restrict__ genp)
{
    extern __shared__ __align__(16) unsigned char dense_smem[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    unsigned char *mine = dense_smem + (size_t)wl * DENSE_WARP_SMEM;
    float4 *P = reinterpret_cast<float4 *>(mine);
    float4 *V = P + DENSE_K;
    const unsigned sP = smem_addr(P), sV = smem_addr(V);
    const unsigned sQ = smem_addr(V + DENSE_K) + 2u * lane;
    uint16_t *pmap = reinterpret_cast<uint16_t *>(mine + (size_t)DENSE_K * 32 + (size_t)DENSE_Q * 32 * 2);
    if (threadIdx.x == 0) s_gen = *genp;
    __syncthreads();                                      // the only barrier: s_gen published
    unsigned cand[4] = {0, 0, 0, 0}, hits[4] = {0, 0, 0, 0}, band = 0;
    const RowPairs rp = row_pairs(g);
    const int ntiles = *gcount;
    const float bx = g.boxf[0], by = g.boxf[1], bz = g.boxf[2];

    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntiles) break;
        const TileGeom T = tile_geom(g, rp, tiles[gtiles[t]]);
        const long long ca = ((long long)(T.xo + g.ghost_x) * g.ny + T.y0) * g.nz + T.za;
        const int na = c.cell_nhome[ca], nb = T.hasB ? c.cell_nhome[ca + g.nz] : 0;
        const int q0 = T.first, q1 = T.first + (T.cnt > 0 ? T.cnt : -T.cnt);
        // the tile's particles: [q0, q1) of (row A's home particles, then row B's)
        for (int part = 0; part < 2; ++part) {
            const long long hcell = part == 0 ? ca : ca + g.nz;
            const int lo = part == 0 ? max(q0, 0) : max(q0, na), hi = part == 0 ? min(q1, na) : min(q1, na + nb);
            if (lo >= hi) continue;
            const int cs = c.cell_start[hcell];
            const int ncl = c.cell_start[hcell + 1] - cs;
            const int nhome = part == 0 ? na : nb;
            const int rlo = part == 0 ? lo : lo - na, rhi = part == 0 ? hi : hi - na;
            const HomeCell hc = home_cell(g, hcell);
            // The part's particles are the home particles of ranks [rlo, rhi) in the home cell's
            // list along DENSE_SELF_DIR (home = in-cell index < nhome: home-first slots), so a
            // warp's 32 lanes are neighbours along that axis and share their self-cell windows.
            const uint16_t *Ls = c.ord + (long long)DENSE_SELF_DIR * c.cap + cs;
            if (nhome == ncl) {
                for (int r = lane; r < rhi - rlo; r += 32) pmap[r] = (uint16_t)(rlo + r);
            } else {
                int run = 0;                                  // home entries before position q0
                for (int q0 = 0; q0 < ncl && run < rhi; q0 += 32) {
                    const int q = q0 + lane;
                    const bool home = q < ncl && (int)Ls[q] < nhome;
                    const unsigned b = __ballot_sync(0xffffffffu, home);
                    const int r = run + __popc(b & ((1u << lane) - 1u));
                    if (home && r >= rlo && r < rhi) pmap[r - rlo] = (uint16_t)q;
                    run += __popc(b);
                }
            }
            __syncwarp();
            for (int k0 = 0; k0 < rhi - rlo; k0 += 32) {
                const bool active = k0 + lane < rhi - rlo;
                const int pi = pmap[k0 + (active ? lane : 0)];       // this lane's sorted position
                const int p0 = pmap[k0];                             // the warp's lowest
                const int i = cs + Ls[pi];
                float x = 0.f, y = 0.f, z = 0.f, vx = 0.f, vy = 0.f, vz = 0.f, m = 0.f, H2 = -1.f, Hinv = 0.f,
                      Hd = 0.f;
                if (active) {
                    const float4 a = c.xyzh[i], b = c.vm[i];
                    x = a.x; y = a.y; z = a.z;
                    vx = b.x; vy = b.y; vz = b.z; m = b.w;
                    const double H = (double)g.gamma * (double)a.w;   // as load_i: H^2, 1/H rounded once
                    H2 = (float)(H * H);
                    Hinv = (float)(1.0 / H);
                    Hd = (float)H + g.delta;
                }
                Acc2 A;
                A.rho = A.wc = A.srt = A.st = A.Dn = A.Px = A.Nx = A.Py = A.Ny = A.Pz = A.Nz = zero2();
                unsigned qp = sQ;
                int nngb = 0;
                const f2 Hinv2 = bc2(Hinv);
                float hx = x, hy = y, hz = z;                 // home coordinate of the current neighbour
                auto drain = [&](bool final) {
                    const unsigned n = (qp - sQ) >> 6;
                    if (n >= 2 || (final && n == 1)) {
                        const bool two = n >= 2;
                        const unsigned s0 = lds_u16(qp - 64u), s1 = two ? lds_u16(qp - 128u) : s0;
                        qp -= two ? 128u : 64u;
                        nngb += two ? 2 : 1;
                        const float4 p0 = ldsr_f4(sP + 16u * s0), p1 = ldsr_f4(sP + 16u * s1);
                        const float4 v0 = ldsr_f4(sV + 16u * s0), v1 = ldsr_f4(sV + 16u * s1);
                        interact_pair<true>(Hinv2, pk(hx - p0.x, hx - p1.x), pk(hy - p0.y, hy - p1.y),
                                            pk(hz - p0.z, hz - p1.z), pk(v0.w, v1.w), pk(v0.x - vx, v1.x - vx),
                                            pk(v0.y - vy, v1.y - vy), pk(v0.z - vz, v1.z - vz),
                                            pk(1.0f, two ? 1.0f : 0.0f), A);
                    }
                };
                auto drain_check = [&]() {
                    for (;;) {
                        const unsigned n = (qp - sQ) >> 6;
                        if (!(__popc(__ballot_sync(0xffffffffu, n >= 2)) >= 24 ||
                              __any_sync(0xffffffffu, n >= DENSE_Q - 4)))
                            break;
                        drain(false);
                    }
                };
                auto drain_all = [&]() {
                    while (__any_sync(0xffffffffu, qp != sQ)) drain(true);
                };
                // candidates [b, e) of the staged chunk for this lane (4 per step)
                auto sweep = [&](int b, int e, int kind, int skip) {
                    const int trip = __reduce_max_sync(0xffffffffu, e - b);
                    for (int t4 = 0; t4 < trip; t4 += 4) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int k = b + t4 + u;
                            const bool ok = k < e && k != skip;
                            const float4 p = ldsr_f4(sP + 16u * (unsigned)(ok ? k : 0));
                            const float dx = hx - p.x, dy = hy - p.y, dz = hz - p.z;
                            const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                            if (COUNT) {
                                cand[kind] += ok ? 1u : 0u;
                                band += ok && fabsf(r2 - H2) < 1e-6f * H2 ? 1u : 0u;
                            }
                            if (ok && r2 < H2) {
                                sts_u16(qp, (unsigned)k);
                                qp += 64u;
                                if (COUNT) ++hits[kind];
                            }
                        }
                        drain_check();
                    }
                };

                // One sorted sweep: staged chunks of the list L (entry q of the sweep = cell slot
                // at(q)), positions pre-shifted by (px, py, pz); each lane's window is the leading
                // entries with sep = (x_j - x_i) . a < H_i + delta (ascending along the sweep, up to
                // the list order's disorder, which delta covers: R5), found by bisection inside
                // the chunk; a further chunk is staged while some lane's window runs on.
                auto windowed = [&](int nq, auto at, float ax, float ay, float az, float px, float py, float pz,
                                    int kind, int skipq) {
                    bool open = active;
                    for (int j0 = 0; j0 < nq; j0 += DENSE_K) {
                        if (!__any_sync(0xffffffffu, open)) break;
                        const int kn = min(DENSE_K, nq - j0);
                        for (int e = lane; e < kn; e += 32) {
                            const int jj = at(j0 + e);
                            float4 p = c.xyzh[jj];
                            p.x -= px; p.y -= py; p.z -= pz;
                            P[e] = p;
                            V[e] = c.vm[jj];
                        }
                        __syncwarp();
                        int top = 1;
                        while (2 * top <= kn) top <<= 1;
                        int len = 0;
                        for (int stp = top; stp > 0; stp >>= 1) {
                            const int kk = len + stp;
                            const bool v = open && kk <= kn;
                            const float4 p = ldsr_f4(sP + 16u * (unsigned)(v ? kk - 1 : 0));
                            const float sep = fmaf(ax, p.x - hx, fmaf(ay, p.y - hy, az * (p.z - hz)));
                            if (v && sep < Hd) len = kk;
                        }
                        sweep(0, open ? len : 0, kind, skipq - j0);
                        drain_all();
                        open = open && len == kn;
                        __syncwarp();
                    }
                };

                // ---- the home cell: along DENSE_SELF_DIR from the warp's lowest position p0, up
                // (p0, p0 + 1, ...; i itself skipped) and down (p0 - 1, p0 - 2, ...) -------------
                {
                    float ax, ay, az;
                    dir_unit(DENSE_SELF_DIR, ax, ay, az);
                    hx = x; hy = y; hz = z;
                    windowed(ncl - p0, [&](int q) { return cs + (int)Ls[p0 + q]; }, ax, ay, az, 0.f, 0.f, 0.f, 0,
                             pi - p0);
                    windowed(p0, [&](int q) { return cs + (int)Ls[p0 - 1 - q]; }, -ax, -ay, -az, 0.f, 0.f, 0.f, 0,
                             -1 - (1 << 30));
                }
                // ---- the 26 neighbours: windows from the near end of the sorted lists ----------
                for (int ox = -1; ox <= 1; ++ox)
                    for (int oy = -1; oy <= 1; ++oy)
                        for (int oz = -1; oz <= 1; ++oz) {
                            if (!(ox | oy | oz)) continue;
                            int cj, sh[3];
                            if (!neighbour(g, hc, ox, oy, oz, cj, sh)) continue;
                            const int kind = kind_of(ox, oy, oz);
                            int sgn;
                            const int d = canon_dir(ox, oy, oz, sgn);
                            float ax, ay, az;
                            dir_unit(d, ax, ay, az);
                            // sep = (x_j - x_i) . d s >= 0 grows along the sweep
                            ax *= (float)sgn; ay *= (float)sgn; az *= (float)sgn;
                            hx = sh[0] > 0 ? x - bx : x;           // exact differences
                            hy = sh[1] > 0 ? y - by : y;
                            hz = sh[2] > 0 ? z - bz : z;
                            const float px = sh[0] < 0 ? bx : 0.0f, py = sh[1] < 0 ? by : 0.0f,
                                        pz = sh[2] < 0 ? bz : 0.0f;
                            const int sj = c.cell_start[cj], nj = c.cell_start[cj + 1] - sj;
                            const uint16_t *L = c.ord + (long long)d * c.cap + sj;
                            windowed(nj, [&](int q) { return sj + (int)L[sgn > 0 ? q : nj - 1 - q]; }, ax, ay, az,
                                     px, py, pz, kind, -1 - (1 << 30));
                        }
                if (active) {
                    const float K3 = (16.0f / kPi) * Hinv * Hinv * Hinv;
                    const float rho = K3 * fmaf(0.5f, m, sum2(A.rho));
                    const float wc = K3 * (0.5f + sum2(A.wc));
                    const float dh = -K3 * g.gamma * Hinv;
                    const float rho_dh = dh * fmaf(1.5f, m, sum2(A.srt));
                    const float wc_dh = dh * (1.5f + sum2(A.st));
                    const float gf = K3 * Hinv;
                    const float rinv = 1.0f / rho;
                    store_rec(orec, c.perm[i], rho, wc, rho_dh, wc_dh, gf * sum2(A.Dn) * rinv,
                              gf * (sum2(A.Px) - sum2(A.Nx)) * rinv, gf * (sum2(A.Py) - sum2(A.Ny)) * rinv,
                              gf * (sum2(A.Pz) - sum2(A.Nz)) * rinv, nngb);
                }
            }
        }
    }
    flush_stats<COUNT>(st, cand, hits, band);
}

}  // namespace pvsph
