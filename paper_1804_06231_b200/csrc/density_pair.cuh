// density_pair.cuh -- sph_density_pair: the paper's pair interaction
// as one CTA per cell pair (ci <- cj), the literal form of the per-pair sweep
// (kernel K6).
//
//  * Staging: the positions and (v, m) of both cells are bulk-copied into shared memory
//    (cp.async.bulk + mbarrier); cj's list sorted along the pair's direction d is copied as
//    staged indices.  cj particles beyond a low box face are pre-shifted by -L, ci's home
//    coordinate by -L where cj lies beyond a high face (exact differences).
//  * Warps take tiles of 32 ci particles (lane = i).  A lane's window in cj is exact: the
//    prefix (cj at +d) or suffix (cj at -d) of the sorted list whose projected separation is
//    below H_i + delta, found by branch-free bisection.
//  * In-range candidates are pushed on the lane's stack; when __ballot_sync/__popc show that
//    most lanes hold two, every lane pops two and evaluates both interactions with
//    FFMA2 (the left-packing of P:185-187).  Register accumulation; the pair's partial sums
//    are added to the outputs with red.global.add (other pairs update the same ci).
//  * Cells above PAIR_MAXN particles take the per-thread global-memory sweep of density.cuh.
#pragma once

#include "common.cuh"
#include "density.cuh"
#include "density_v4.cuh"
#include "packed.cuh"

namespace pvsph {

constexpr int PAIR_WARPS = 4;
constexpr int PAIR_MAXN = 1024;          // staged particles per cell
constexpr int PAIR_Q = 16;               // hit stack depth per lane
constexpr size_t PAIR_SMEM = (size_t)PAIR_MAXN * 16 * 3 + (size_t)PAIR_MAXN * 2 + (size_t)PAIR_WARPS * PAIR_Q * 32 * 2;

template <bool COUNT>
__global__ void __launch_bounds__(PAIR_WARPS * 32) k_density_pair_staged(DevGrid g, DevCells c, DevOut o,
                                                                         const int2 *pairs, long long npairs,
                                                                         sph_stats *st, unsigned *status)
{
    extern __shared__ __align__(16) unsigned char pair_smem[];
    float4 *Pi = reinterpret_cast<float4 *>(pair_smem);          // ci positions
    float4 *Pj = Pi + PAIR_MAXN;                                   // cj positions
    float4 *Vj = Pj + PAIR_MAXN;                                   // cj (v, m)
    uint16_t *Lj = reinterpret_cast<uint16_t *>(Vj + PAIR_MAXN);   // cj sorted along d (staged indices)
    uint16_t *stacks = Lj + PAIR_MAXN;
    __shared__ __align__(8) unsigned long long s_mbar;
    const unsigned mbar = smem_addr(&s_mbar);
    unsigned phase = 0;
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned cand[4] = {0, 0, 0, 0}, hits[4] = {0, 0, 0, 0};

    for (long long q = blockIdx.x; q < npairs; q += gridDim.x) {
        const int2 pr = pairs[q];
        const long long ci = pr.x, cj = pr.y;
        if (!owned_cell(g, ci) || cj < 0 || cj >= g.ncell) {
            if (threadIdx.x == 0) set_status(status, ST_EINVAL);
            continue;
        }
        const HomeCell hc = home_cell(g, ci);
        const long long plane = (long long)g.ny * g.nz;
        const int jxl = (int)(cj / plane), jy = (int)((cj / g.nz) % g.ny), jz = (int)(cj % g.nz);
        int ox = jxl - hc.ixl, oy = jy - hc.iy, oz = jz - hc.iz;
        if (!g.ghost_x) ox = ox == g.nc[0] - 1 ? -1 : (ox == 1 - g.nc[0] ? 1 : ox);
        oy = oy == g.ny - 1 ? -1 : (oy == 1 - g.ny ? 1 : oy);
        oz = oz == g.nz - 1 ? -1 : (oz == 1 - g.nz ? 1 : oz);
        if (ox < -1 || ox > 1 || oy < -1 || oy > 1 || oz < -1 || oz > 1 || !(ox | oy | oz)) {
            if (threadIdx.x == 0) set_status(status, ST_EINVAL);
            continue;
        }
        int cjc, sh[3];
        neighbour(g, hc, ox, oy, oz, cjc, sh);
        const int kind = kind_of(ox, oy, oz);
        int sgn;
        const int d = canon_dir(ox, oy, oz, sgn);
        const int si = c.cell_start[ci], ni = c.cell_start[ci + 1] - si;
        const int sj = c.cell_start[cjc], nj = c.cell_start[cjc + 1] - sj;
        if (ni == 0 || nj == 0) continue;
        if (ni > PAIR_MAXN || nj > PAIR_MAXN) {
            // dense cells: the per-thread sweep reading global memory
            for (int i = si + threadIdx.x; i < si + ni; i += blockDim.x) {
                IPart p = load_i(g, c, i, hc.corner);
                Acc a;
                acc_zero(a);
                sweep_pair<COUNT>(g, c, p, cjc, ox, oy, oz, sh, a, cand[kind], hits[kind]);
                if (a.nngb > 0) atomic_out(o, c.perm[i], finalise(g, p, a, false), a.nngb);
            }
            continue;
        }
        // ---- staging: bulk copies of both cells, then cj's sorted list ------------------
        if (threadIdx.x == 0) {
            mbar_expect_tx(mbar, (unsigned)(ni + 2 * nj) * 16u);
            bulk_g2s(smem_addr(Pi), c.xyzh + si, (unsigned)ni * 16u, mbar);
            bulk_g2s(smem_addr(Pj), c.xyzh + sj, (unsigned)nj * 16u, mbar);
            bulk_g2s(smem_addr(Vj), c.vm + sj, (unsigned)nj * 16u, mbar);
        }
        const uint16_t *src = c.ord + (long long)d * c.cap + sj;
        for (int k = threadIdx.x; k < nj; k += blockDim.x) Lj[k] = src[k];
        mbar_wait(mbar, phase);
        phase ^= 1u;
        const float bx = g.boxf[0], by = g.boxf[1], bz = g.boxf[2];
        if (sh[0] < 0 || sh[1] < 0 || sh[2] < 0) {
            // cj beyond a low face: x_j - L, exact (x_j >= L/2)
            for (int k = threadIdx.x; k < nj; k += blockDim.x) {
                float4 p = Pj[k];
                p.x -= sh[0] < 0 ? bx : 0.0f;
                p.y -= sh[1] < 0 ? by : 0.0f;
                p.z -= sh[2] < 0 ? bz : 0.0f;
                Pj[k] = p;
            }
        }
        __syncthreads();

        // ---- warps over tiles of 32 ci particles -------------------------------------------
        const unsigned sP = smem_addr(Pj), sV = smem_addr(Vj), sL = smem_addr(Lj);
        const unsigned sQ = smem_addr(stacks + wl * PAIR_Q * 32) + 2u * lane;
        const float c0 = (float)dir_component(d, 0), c1 = (float)dir_component(d, 1), c2 = (float)dir_component(d, 2);
        const float rk = kind == 1 ? 1.0f : (kind == 2 ? 1.41421356237309505f : 1.73205080756887729f);
        for (int t0 = wl * 32; t0 < ni; t0 += PAIR_WARPS * 32) {
            const int e = t0 + lane;
            const bool active = e < ni;
            float x = 0.f, y = 0.f, z = 0.f, vx = 0.f, vy = 0.f, vz = 0.f, H2 = -1.f, Hinv = 0.f, Hk = 0.f, m = 0.f;
            if (active) {
                const float4 a = Pi[e];
                const float4 b = c.vm[si + e];
                // home coordinate shifted by -L where cj lies beyond a high face (exact: x_i >= L/2)
                x = sh[0] > 0 ? a.x - bx : a.x;
                y = sh[1] > 0 ? a.y - by : a.y;
                z = sh[2] > 0 ? a.z - bz : a.z;
                vx = b.x; vy = b.y; vz = b.z; m = b.w;
                const double H = (double)g.gamma * (double)a.w;
                H2 = (float)(H * H);
                Hinv = (float)(1.0 / H);
                Hk = ((float)H + g.delta) * rk;
            }
            // window: sgn > 0 (cj at +d): prefix of the ascending list with (x_j - x_i) . d < Hk;
            // sgn < 0 (cj at -d): suffix with (x_i - x_j) . d < Hk
            int top = 1;
            while (2 * top <= nj) top <<= 1;
            int lo = 0;
            for (int stp = top; stp > 0; stp >>= 1) {
                const int kk = lo + stp;
                const bool v = active && kk <= nj;
                const int pos = sgn > 0 ? kk - 1 : nj - kk;
                const unsigned id = v ? ldsr_u16(sL + 2u * (unsigned)pos) : 0u;
                const float4 p = ldsr_f4(sP + 16u * id);
                const float sep = (float)sgn * fmaf(c0, p.x - x, fmaf(c1, p.y - y, c2 * (p.z - z)));
                if (v && sep < Hk) lo = kk;
            }
            const int len = lo, first = sgn > 0 ? 0 : nj - len;
            Acc2 A;
            A.rho = A.wc = A.srt = A.st = A.Dn = A.Px = A.Nx = A.Py = A.Ny = A.Pz = A.Nz = zero2();
            unsigned qp = sQ;
            int nngb = 0;
            const f2 Hinv2 = bc2(Hinv);
            auto drain = [&](bool final) {
                const unsigned n = (qp - sQ) >> 6;
                if (n >= 2 || (final && n == 1)) {
                    const bool two = n >= 2;
                    const unsigned s0 = lds_u16(qp - 64u), s1 = two ? lds_u16(qp - 128u) : s0;
                    qp -= two ? 128u : 64u;
                    nngb += two ? 2 : 1;
                    const float4 p0 = ldsr_f4(sP + 16u * s0), p1 = ldsr_f4(sP + 16u * s1);
                    const float4 v0 = ldsr_f4(sV + 16u * s0), v1 = ldsr_f4(sV + 16u * s1);
                    interact_pair<true>(Hinv2, pk(x - p0.x, x - p1.x), pk(y - p0.y, y - p1.y), pk(z - p0.z, z - p1.z),
                                        pk(v0.w, v1.w), pk(v0.x - vx, v1.x - vx), pk(v0.y - vy, v1.y - vy),
                                        pk(v0.z - vz, v1.z - vz), pk(1.0f, two ? 1.0f : 0.0f), A);
                }
            };
            const int trip = __reduce_max_sync(0xffffffffu, len);
            for (int t = 0; t < trip; t += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool ok = t + u < len;
                    const unsigned id = ok ? ldsr_u16(sL + 2u * (unsigned)(first + t + u)) : 0u;
                    const float4 p = ldsr_f4(sP + 16u * id);
                    const float dx = x - p.x, dy = y - p.y, dz = z - p.z;
                    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                    if (COUNT) cand[kind] += ok ? 1u : 0u;
                    if (ok && r2 < H2) {
                        sts_u16(qp, id);
                        qp += 64u;
                        if (COUNT) ++hits[kind];
                    }
                }
                // left-packing: drain when most lanes hold two hits, or a stack could overflow
                for (;;) {
                    const unsigned n = (qp - sQ) >> 6;
                    if (!(__popc(__ballot_sync(0xffffffffu, n >= 2)) >= 24 ||
                          __any_sync(0xffffffffu, n >= PAIR_Q - 4)))
                        break;
                    drain(false);
                }
            }
            while (__any_sync(0xffffffffu, qp != sQ)) drain(true);
            if (active && nngb > 0) {
                const float K3 = (16.0f / kPi) * Hinv * Hinv * Hinv;
                const float gf = K3 * Hinv;
                Final f;
                f.rho = K3 * sum2(A.rho);
                f.wc = K3 * sum2(A.wc);
                f.rho_dh = -K3 * g.gamma * Hinv * sum2(A.srt);
                f.wc_dh = -K3 * g.gamma * Hinv * sum2(A.st);
                f.div = gf * sum2(A.Dn);                   // rho * div v
                f.cx = gf * (sum2(A.Px) - sum2(A.Nx));     // rho * curl v
                f.cy = gf * (sum2(A.Py) - sum2(A.Ny));
                f.cz = gf * (sum2(A.Pz) - sum2(A.Nz));
                atomic_out(o, c.perm[si + e], f, nngb);
            }
            (void)m;
        }
        __syncthreads();                          // shared memory reused by the next pair
    }
    flush_stats<COUNT>(st, cand, hits);
}

// ---- symmetric pair kernel -------------------------------------
// One CTA per UNORDERED neighbour pair (ci, cj): every distance of the pair is evaluated once
// and both particles take their share.  Phase 1, lane = i in ci (as k_density_pair_staged):
// the window in cj's sorted list uses max(H_i, gamma hmax(cj)) + delta, so every j that
// reaches i (r < H_j) is a candidate too; r < H_i goes to the lane's stack (FFMA2 drains,
// register sums), r < H_j records i in j's bucket in shared memory (one shared atomic for
// the slot).  Phase 2, lane = j in cj: the bucket's interactions with H_j and m_i (x_ji =
// -x_ij, v_ji = -v_ij leave every product unchanged), two per step with FFMA2, register
// sums.  Both sides reach the outputs with red.global.add, as in the one-sided kernel; j in
// a ghost cell (slabs) is skipped.  A bucket that overflows adds that hit's share directly.
constexpr int SYM_WARPS = 4;
constexpr int SYM_MAXN = 512;            // staged particles per cell (3 CTAs per SM)
constexpr int SYM_Q = 16;
constexpr int SYM_JCAP = 32;             // bucket entries per j
// shared memory of one team (TW warps working on one pair at a time, MAXN staged per cell)
__host__ __device__ constexpr size_t sym_team_smem(int maxn, int tw)
{
    return (size_t)maxn * 16 * 4 + (size_t)maxn * 4 * 2 + (size_t)maxn * 2 + (size_t)tw * SYM_Q * 32 * 2 +
           (size_t)maxn * SYM_JCAP * 2;
}
constexpr size_t SYM_SMEM = sym_team_smem(SYM_MAXN, SYM_WARPS);
// sph_density_all_sym's colour phases: one warp per pair of cells of <= SYMW_MAXN particles
// (16 pairs in flight per SM instead of three CTAs); larger pairs are deferred to the CTA form
constexpr int SYMW_MAXN = 64;
constexpr int SYMW_WARPS = 8;
constexpr size_t SYMW_SMEM = sym_team_smem(SYMW_MAXN, 1) * SYMW_WARPS;
static_assert(sym_team_smem(SYMW_MAXN, 1) % 16 == 0, "team slices must stay 16-byte aligned");

// Per-slot accumulators of sph_density_all_sym (the ws output-record region, cell-sorted slot
// order): a cell's particles are contiguous, so a pair's read-modify-writes are coalesced
// 32-byte sectors instead of nine scattered words per particle; k_sym_merge adds them to the
// outputs (input order) once at the end.
struct alignas(32) SlotAcc {
    float4 a, b;                 // rho, wcount, rho_dh, wcount_dh | rho div v, rho curl v
    int nngb, pad[7];
};

__device__ __forceinline__ void slot_out(SlotAcc *acc, const Final &f, int nngb)
{
    float4 a = acc->a, b = acc->b;
    a.x += f.rho; a.y += f.wc; a.z += f.rho_dh; a.w += f.wc_dh;
    b.x += f.div; b.y += f.cx; b.z += f.cy; b.w += f.cz;
    acc->a = a;
    acc->b = b;
    acc->nngb += nngb;
}

template <bool PLAIN>
__device__ __forceinline__ void sym_flush(const DevGrid &g, const DevOut &o, SlotAcc *sacc, int slot, int out,
                                          float Hinv, const Acc2 &B, int nn)
{
    const float K3 = (16.0f / kPi) * Hinv * Hinv * Hinv, gf = K3 * Hinv;
    Final f;
    f.rho = K3 * sum2(B.rho);
    f.wc = K3 * sum2(B.wc);
    f.rho_dh = -K3 * g.gamma * Hinv * sum2(B.srt);
    f.wc_dh = -K3 * g.gamma * Hinv * sum2(B.st);
    f.div = gf * sum2(B.Dn);                       // rho * div v
    f.cx = gf * (sum2(B.Px) - sum2(B.Nx));         // rho * curl v
    f.cy = gf * (sum2(B.Py) - sum2(B.Ny));
    f.cz = gf * (sum2(B.Pz) - sum2(B.Nz));
    if (PLAIN && sacc) slot_out(sacc + slot, f, nn);
    else if (PLAIN) plain_out(o, out, f, nn);
    else atomic_out(o, out, f, nn);
}

// PLAIN (sph_density_all_sym's colour phases): no two pairs of a launch share a cell, so the
// outputs take plain read-modify-writes, and each j sums its bucket in ascending i (the buckets
// are sorted first): deterministic.  npairs_dev (optional): the device-side pair count.
// Teams: the CTA's NWARPS warps form NWARPS / TW teams of TW warps, each with its own shared-
// memory slice and mbarrier, each working on its own pair (TW = 1: a warp per pair, warp
// syncs only).  A pair with a cell above MAXN goes to big_pairs (when given: the caller runs
// it through the CTA form afterwards), else to the per-thread global-memory sweeps.
template <int TW, int NWARPS>
__device__ __forceinline__ void team_sync(int team)
{
    if constexpr (TW == 1) __syncwarp();
    else if constexpr (TW == NWARPS) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(TW * 32) : "memory");
}

template <bool COUNT, bool PLAIN = false, int MAXN = SYM_MAXN, int TW = SYM_WARPS, int NWARPS = SYM_WARPS>
__global__ void __launch_bounds__(NWARPS * 32) k_density_pair_sym(DevGrid g, DevCells c, DevOut o,
                                                                  const int2 *pairs, long long npairs,
                                                                  sph_stats *st, unsigned *status,
                                                                  const int *npairs_dev = nullptr,
                                                                  int2 *big_pairs = nullptr, int *big_count = nullptr,
                                                                  SlotAcc *sacc = nullptr)
{
    constexpr int NTEAM = NWARPS / TW, TT = TW * 32;
    static_assert(NWARPS % TW == 0, "teams must tile the CTA");
    extern __shared__ __align__(16) unsigned char sym_smem[];
    const int team = threadIdx.x / TT, tt = threadIdx.x % TT;
    float4 *Pi = reinterpret_cast<float4 *>(sym_smem + sym_team_smem(MAXN, TW) * team);   // ci positions (home shift applied)
    float4 *Vi = Pi + MAXN;                                          // ci (v, m)
    float4 *Pj = Vi + MAXN;                                          // cj positions (pre-shifted), w = H_j^2
    float4 *Vj = Pj + MAXN;                                          // cj (v, m)
    float *HinvJ = reinterpret_cast<float *>(Vj + MAXN);             // 1 / H_j
    int *JC = reinterpret_cast<int *>(HinvJ + MAXN);                 // bucket fill of each j
    uint16_t *Lj = reinterpret_cast<uint16_t *>(JC + MAXN);          // cj sorted along d
    uint16_t *stacks = Lj + MAXN;
    uint16_t *JB = stacks + TW * SYM_Q * 32;                         // [MAXN][SYM_JCAP] i of j's hits
    __shared__ __align__(8) unsigned long long s_mbar[NTEAM];
    const unsigned mbar = smem_addr(&s_mbar[team]);
    unsigned phase = 0;
    const int lane = threadIdx.x & 31, wl = tt >> 5;                 // wl: warp within the team
    if (tt == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned cand[4] = {0, 0, 0, 0}, hits[4] = {0, 0, 0, 0};
    if (npairs_dev) npairs = min(npairs, (long long)*npairs_dev);

    for (long long q = (long long)blockIdx.x * NTEAM + team; q < npairs; q += (long long)gridDim.x * NTEAM) {
        const int2 pr = pairs[q];
        const long long ci = pr.x, cj = pr.y;
        // (PLAIN: ci may be a ghost cell whose +d neighbour is owned; only j accumulates then)
        const bool i_owned = owned_cell(g, ci);
        if ((!PLAIN && !i_owned) || ci < 0 || ci >= g.ncell || cj < 0 || cj >= g.ncell) {
            if (tt == 0) set_status(status, ST_EINVAL);
            continue;
        }
        const HomeCell hc = home_cell(g, ci);
        const long long plane = (long long)g.ny * g.nz;
        const int jxl = (int)(cj / plane), jy = (int)((cj / g.nz) % g.ny), jz = (int)(cj % g.nz);
        int ox = jxl - hc.ixl, oy = jy - hc.iy, oz = jz - hc.iz;
        if (!g.ghost_x) ox = ox == g.nc[0] - 1 ? -1 : (ox == 1 - g.nc[0] ? 1 : ox);
        oy = oy == g.ny - 1 ? -1 : (oy == 1 - g.ny ? 1 : oy);
        oz = oz == g.nz - 1 ? -1 : (oz == 1 - g.nz ? 1 : oz);
        if (ox < -1 || ox > 1 || oy < -1 || oy > 1 || oz < -1 || oz > 1 || !(ox | oy | oz)) {
            if (tt == 0) set_status(status, ST_EINVAL);
            continue;
        }
        int cjc, sh[3];
        neighbour(g, hc, ox, oy, oz, cjc, sh);
        const int kind = kind_of(ox, oy, oz);
        int sgn;
        const int d = canon_dir(ox, oy, oz, sgn);
        const int si = c.cell_start[ci], ni = c.cell_start[ci + 1] - si;
        const int sj = c.cell_start[cjc], nj = c.cell_start[cjc + 1] - sj;
        if (ni == 0 || nj == 0) continue;
        const bool j_owned = owned_cell(g, cjc);
        if (ni > MAXN || nj > MAXN) {
            if (big_pairs) {                      // the CTA form takes it after this launch
                if (tt == 0) big_pairs[atomicAdd(big_count, 1)] = pr;
                continue;
            }
            // dense cells: the two one-sided per-thread sweeps reading global memory
            for (int i = si + tt; i_owned && i < si + ni; i += TT) {
                IPart p = load_i(g, c, i, hc.corner);
                Acc a;
                acc_zero(a);
                sweep_pair<COUNT>(g, c, p, cjc, ox, oy, oz, sh, a, cand[kind], hits[kind]);
                if (a.nngb > 0) {
                    if (PLAIN && sacc) slot_out(sacc + i, finalise(g, p, a, false), a.nngb);
                    else if (PLAIN) plain_out(o, c.perm[i], finalise(g, p, a, false), a.nngb);
                    else atomic_out(o, c.perm[i], finalise(g, p, a, false), a.nngb);
                }
            }
            team_sync<TW, NWARPS>(team);              // (PLAIN) ci's outputs written before cj's sweep reads nothing of them
            if (j_owned) {
                const HomeCell hj = home_cell(g, cjc);
                int cic, sh2[3];
                neighbour(g, hj, -ox, -oy, -oz, cic, sh2);
                for (int j = sj + tt; j < sj + nj; j += TT) {
                    IPart p = load_i(g, c, j, hj.corner);
                    Acc a;
                    acc_zero(a);
                    unsigned dummy = 0;
                    sweep_pair<COUNT>(g, c, p, cic, -ox, -oy, -oz, sh2, a, dummy, hits[kind]);
                    if (a.nngb > 0) {
                        if (PLAIN && sacc) slot_out(sacc + j, finalise(g, p, a, false), a.nngb);
                        else if (PLAIN) plain_out(o, c.perm[j], finalise(g, p, a, false), a.nngb);
                        else atomic_out(o, c.perm[j], finalise(g, p, a, false), a.nngb);
                    }
                }
            }
            continue;
        }
        // ---- staging: both cells (positions and v, m), cj's sorted list, empty buckets ----------
        if (tt == 0) {
            mbar_expect_tx(mbar, (unsigned)(2 * ni + 2 * nj) * 16u);
            bulk_g2s(smem_addr(Pi), c.xyzh + si, (unsigned)ni * 16u, mbar);
            bulk_g2s(smem_addr(Vi), c.vm + si, (unsigned)ni * 16u, mbar);
            bulk_g2s(smem_addr(Pj), c.xyzh + sj, (unsigned)nj * 16u, mbar);
            bulk_g2s(smem_addr(Vj), c.vm + sj, (unsigned)nj * 16u, mbar);
        }
        const uint16_t *src = c.ord + (long long)d * c.cap + sj;
        for (int k = tt; k < nj; k += TT) {
            Lj[k] = src[k];
            JC[k] = 0;
        }
        mbar_wait(mbar, phase);
        phase ^= 1u;
        const float bx = g.boxf[0], by = g.boxf[1], bz = g.boxf[2];
        for (int k = tt; k < nj; k += TT) {
            float4 p = Pj[k];
            // cj beyond a low face: x_j - L, exact (x_j >= L/2); w <- H_j^2 as the gather rounds it
            p.x -= sh[0] < 0 ? bx : 0.0f;
            p.y -= sh[1] < 0 ? by : 0.0f;
            p.z -= sh[2] < 0 ? bz : 0.0f;
            const double H = (double)g.gamma * (double)p.w;
            p.w = (float)(H * H);
            HinvJ[k] = (float)(1.0 / H);
            Pj[k] = p;
        }
        for (int k = tt; k < ni; k += TT) {
            // ci's home coordinate shifted by -L where cj lies beyond a high face (exact: x_i >= L/2)
            float4 p = Pi[k];
            p.x -= sh[0] > 0 ? bx : 0.0f;
            p.y -= sh[1] > 0 ? by : 0.0f;
            p.z -= sh[2] > 0 ? bz : 0.0f;
            Pi[k] = p;
        }
        const float Hjmax = (float)((double)g.gamma * (double)c.cell_hmax[cjc]);
        team_sync<TW, NWARPS>(team);

        const unsigned sP = smem_addr(Pj), sV = smem_addr(Vj), sL = smem_addr(Lj);
        const unsigned sQ = smem_addr(stacks + wl * SYM_Q * 32) + 2u * lane;
        const float c0 = (float)dir_component(d, 0), c1 = (float)dir_component(d, 1), c2 = (float)dir_component(d, 2);
        const float rk = kind == 1 ? 1.0f : (kind == 2 ? 1.41421356237309505f : 1.73205080756887729f);
        // ---- phase 1: lane = i ------------------------------------------------------------------
        for (int t0 = wl * 32; t0 < ni; t0 += TT) {
            const int e = t0 + lane;
            const bool active = e < ni;
            float x = 0.f, y = 0.f, z = 0.f, vx = 0.f, vy = 0.f, vz = 0.f, H2 = -1.f, Hinv = 0.f, Hk = 0.f, m = 0.f;
            if (active) {
                const float4 a = Pi[e];
                const float4 b = Vi[e];
                x = a.x; y = a.y; z = a.z;
                vx = b.x; vy = b.y; vz = b.z; m = b.w;
                const double H = (double)g.gamma * (double)a.w;   // w is h (only x, y, z were shifted)
                H2 = (float)(H * H);
                Hinv = (float)(1.0 / H);
                Hk = (fmaxf((float)H, Hjmax) + g.delta) * rk;
            }
            int top = 1;
            while (2 * top <= nj) top <<= 1;
            int lo = 0;
            for (int stp = top; stp > 0; stp >>= 1) {
                const int kk = lo + stp;
                const bool v = active && kk <= nj;
                const int pos = sgn > 0 ? kk - 1 : nj - kk;
                const unsigned id = v ? ldsr_u16(sL + 2u * (unsigned)pos) : 0u;
                const float4 p = ldsr_f4(sP + 16u * id);
                const float sep = (float)sgn * fmaf(c0, p.x - x, fmaf(c1, p.y - y, c2 * (p.z - z)));
                if (v && sep < Hk) lo = kk;
            }
            const int len = lo, first = sgn > 0 ? 0 : nj - len;
            Acc2 A;
            A.rho = A.wc = A.srt = A.st = A.Dn = A.Px = A.Nx = A.Py = A.Ny = A.Pz = A.Nz = zero2();
            unsigned qp = sQ;
            int nngb = 0;
            const f2 Hinv2 = bc2(Hinv);
            auto drain = [&](bool final) {
                const unsigned n = (qp - sQ) >> 6;
                if (n >= 2 || (final && n == 1)) {
                    const bool two = n >= 2;
                    const unsigned s0 = lds_u16(qp - 64u), s1 = two ? lds_u16(qp - 128u) : s0;
                    qp -= two ? 128u : 64u;
                    nngb += two ? 2 : 1;
                    const float4 p0 = ldsr_f4(sP + 16u * s0), p1 = ldsr_f4(sP + 16u * s1);
                    const float4 v0 = ldsr_f4(sV + 16u * s0), v1 = ldsr_f4(sV + 16u * s1);
                    interact_pair<true>(Hinv2, pk(x - p0.x, x - p1.x), pk(y - p0.y, y - p1.y), pk(z - p0.z, z - p1.z),
                                        pk(v0.w, v1.w), pk(v0.x - vx, v1.x - vx), pk(v0.y - vy, v1.y - vy),
                                        pk(v0.z - vz, v1.z - vz), pk(1.0f, two ? 1.0f : 0.0f), A);
                }
            };
            const int trip = __reduce_max_sync(0xffffffffu, len);
            for (int t = 0; t < trip; t += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool ok = t + u < len;
                    const unsigned id = ok ? ldsr_u16(sL + 2u * (unsigned)(first + t + u)) : 0u;
                    const float4 p = ldsr_f4(sP + 16u * id);
                    const float dx = x - p.x, dy = y - p.y, dz = z - p.z;
                    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                    const bool hi = ok && r2 < H2, hj = ok && r2 < p.w;
                    if (COUNT) {
                        cand[kind] += ok ? 1u : 0u;
                        hits[kind] += (hi && i_owned ? 1u : 0u) + (hj && j_owned ? 1u : 0u);
                    }
                    if (hi) {
                        sts_u16(qp, id);
                        qp += 64u;
                    }
                    if (hj && j_owned) {
                        const int slot = atomicAdd(&JC[id], 1);
                        if (slot < SYM_JCAP) {
                            JB[id * SYM_JCAP + slot] = (uint16_t)e;
                        } else {
                            // bucket full: this hit's share of j goes to the outputs directly
                            Acc2 B;
                            B.rho = B.wc = B.srt = B.st = B.Dn = B.Px = B.Nx = B.Py = B.Ny = B.Pz = B.Nz = zero2();
                            const float4 vj = Vj[id];
                            interact_pair<true>(bc2(HinvJ[id]), pk(dx, 0.f), pk(dy, 0.f), pk(dz, 0.f), pk(m, 0.f),
                                                pk(vj.x - vx, 0.f), pk(vj.y - vy, 0.f), pk(vj.z - vz, 0.f),
                                                pk(1.0f, 0.0f), B);
                            // (a bucket overflow: several lanes may hit j at once -> atomic even in PLAIN)
                            sym_flush<false>(g, o, nullptr, 0, c.perm[sj + id], HinvJ[id], B, 1);
                        }
                    }
                }
                for (;;) {
                    const unsigned n = (qp - sQ) >> 6;
                    if (!(__popc(__ballot_sync(0xffffffffu, n >= 2)) >= 24 ||
                          __any_sync(0xffffffffu, n >= SYM_Q - 4)))
                        break;
                    drain(false);
                }
            }
            while (__any_sync(0xffffffffu, qp != sQ)) drain(true);
            if (active && nngb > 0 && i_owned) sym_flush<PLAIN>(g, o, sacc, si + e, c.perm[si + e], Hinv, A, nngb);
        }
        team_sync<TW, NWARPS>(team);                          // buckets complete
        // ---- phase 2: lane = j, its bucket of i ---------------------------------------------------
        if (j_owned) {
            for (int t0 = wl * 32; t0 < nj; t0 += TT) {
                const int k = t0 + lane;
                const bool active = k < nj;
                const int nb = active ? min(JC[k], SYM_JCAP) : 0;
                if (PLAIN && nb > 1) {        // ascending i: a fixed summation order (the bucket slots
                    uint16_t *bk = JB + k * SYM_JCAP;   // came from shared-memory atomics in any order)
                    for (int a1 = 1; a1 < nb; ++a1) {
                        const uint16_t key = bk[a1];
                        int b1 = a1 - 1;
                        while (b1 >= 0 && bk[b1] > key) {
                            bk[b1 + 1] = bk[b1];
                            --b1;
                        }
                        bk[b1 + 1] = key;
                    }
                }
                const float4 pj = active ? Pj[k] : make_float4(0.f, 0.f, 0.f, 0.f);
                const float4 vj = active ? Vj[k] : make_float4(0.f, 0.f, 0.f, 0.f);
                const float hinv = active ? HinvJ[k] : 0.0f;
                Acc2 B;
                B.rho = B.wc = B.srt = B.st = B.Dn = B.Px = B.Nx = B.Py = B.Ny = B.Pz = B.Nz = zero2();
                const f2 hj2 = bc2(hinv);
                const int trip = __reduce_max_sync(0xffffffffu, nb);
                for (int t = 0; t < trip; t += 2) {
                    const bool a0 = t < nb, a1 = t + 1 < nb;
                    const int i0 = a0 ? JB[k * SYM_JCAP + t] : 0, i1 = a1 ? JB[k * SYM_JCAP + t + 1] : i0;
                    const float4 p0 = Pi[i0], p1 = Pi[i1];
                    const float4 w0 = Vi[i0], w1 = Vi[i1];
                    // x_ij = x_i - x_j and v_j - v_i, as in phase 1; m_i; H_j
                    interact_pair<true>(hj2, pk(p0.x - pj.x, p1.x - pj.x), pk(p0.y - pj.y, p1.y - pj.y),
                                        pk(p0.z - pj.z, p1.z - pj.z), pk(w0.w, w1.w), pk(vj.x - w0.x, vj.x - w1.x),
                                        pk(vj.y - w0.y, vj.y - w1.y), pk(vj.z - w0.z, vj.z - w1.z),
                                        pk(a0 ? 1.0f : 0.0f, a1 ? 1.0f : 0.0f), B);
                }
                if (nb > 0) sym_flush<PLAIN>(g, o, sacc, sj + k, c.perm[sj + k], hinv, B, nb);
            }
        }
        team_sync<TW, NWARPS>(team);                          // shared memory reused by the next pair
    }
    flush_stats<COUNT>(st, cand, hits);
}

// ---- sph_density_all_sym: the symmetric sweep over the whole pass ----
// Colour of a cell on one axis of n cells: parity, plus a third colour for the last cell of
// an odd periodic axis; two cells of one colour are >= 2 apart (periodically), so for a fixed
// direction d the pairs (c, c + d) of one colour share no cell: a launch per (d, colour)
// writes disjoint particles without atomics.  The x axis of a slab (ghost planes) is not
// periodic inside the rank: parity of the local plane.
__host__ __device__ __forceinline__ int sym_axis_colours(int n, bool periodic)
{
    return periodic && (n & 1) ? 3 : 2;
}

__device__ __forceinline__ int sym_axis_colour(int x, int n, bool periodic)
{
    return periodic && (n & 1) && x == n - 1 ? 2 : (x & 1);
}

// The colour axis of direction d: its first nonzero component.  Two pairs (c, c + d) and
// (c', c' + d) of one direction share a cell only if c' = c +- d, i.e. their coordinates on
// that axis are neighbours, which sym_axis_colour always tells apart: 2 (or 3) phases per
// direction.
__host__ __device__ __forceinline__ int sym_dir_axis(int d)
{
    return dir_component(d, 0) != 0 ? 0 : (dir_component(d, 1) != 0 ? 1 : 2);
}

__host__ __device__ __forceinline__ int sym_dir_colours(const DevGrid &g, int d)
{
    const int a = sym_dir_axis(d);
    return a == 0 ? sym_axis_colours(g.nxl, !g.ghost_x) : sym_axis_colours(a == 1 ? g.ny : g.nz, true);
}

// Pairs (c, c + d) for the cells c of colour `col` along d's colour axis (cells of either side
// empty are skipped); also, with d < 0, the list of all owned non-empty cells (the self pass).
__global__ void k_sym_phase_pairs(DevGrid g, const int *__restrict__ cell_start, int d, int col, int2 *pairs,
                                  int *count)
{
    const long long plane = (long long)g.ny * g.nz;
    const int a0 = d >= 0 ? dir_component(d, 0) : 0, a1 = d >= 0 ? dir_component(d, 1) : 0,
              a2 = d >= 0 ? dir_component(d, 2) : 0;
    const int axis = d >= 0 ? sym_dir_axis(d) : 0;
    // d < 0: the owned cells; else every local cell (a low ghost cell pairs with its owned +d neighbour)
    const long long ncells = d < 0 ? g.n_owned_cells : g.ncell;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < ncells;
         w += (long long)gridDim.x * blockDim.x) {
        const long long cell = d < 0 ? (w / plane + g.ghost_x) * plane + (w % plane) : w;
        if (cell_start[cell + 1] == cell_start[cell]) continue;
        if (d < 0) {
            pairs[atomicAdd(count, 1)] = make_int2((int)cell, (int)cell);
            continue;
        }
        const int ixl = (int)(cell / plane), iy = (int)((cell / g.nz) % g.ny), iz = (int)(cell % g.nz);
        const int colour = axis == 0 ? sym_axis_colour(ixl, g.nxl, !g.ghost_x)
                                     : (axis == 1 ? sym_axis_colour(iy, g.ny, true) : sym_axis_colour(iz, g.nz, true));
        if (colour != col) continue;
        const HomeCell hc = home_cell(g, cell);
        int cj, sh[3];
        if (!neighbour(g, hc, a0, a1, a2, cj, sh)) continue;
        if (cell_start[cj + 1] == cell_start[cj]) continue;
        if (!owned_cell(g, cell) && !owned_cell(g, cj)) continue;   // ghost-ghost: nothing to write
        pairs[atomicAdd(count, 1)] = make_int2((int)cell, cj);
    }
}

// sph_density_all_sym's last step: out[perm[s]] += slot accumulator s (the self pass wrote
// out[] directly), then div v and curl v divided by rho (k_finalize's step) -- every owned
// particle has exactly one slot.  Ghost slots (perm >= n_out) were never written.
__global__ void k_sym_merge(DevOut o, const SlotAcc *__restrict__ acc, const int *__restrict__ perm,
                            const int *__restrict__ n_stored)
{
    const long long n = *n_stored;
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n; s += (long long)gridDim.x * blockDim.x) {
        const int p = perm[s];
        if (p < 0 || p >= o.n_out) continue;
        const float4 a = acc[s].a, b = acc[s].b;
        const float rho = o.rho[p] + a.x;
        const float rinv = rho != 0.0f ? 1.0f / rho : 0.0f;
        o.rho[p] = rho;
        o.wcount[p] += a.y;
        o.rho_dh[p] += a.z;
        o.wcount_dh[p] += a.w;
        o.div_v[p] = (o.div_v[p] + b.x) * rinv;
        o.curl_v[p] = (o.curl_v[p] + b.y) * rinv;
        o.curl_v[o.n_out + p] = (o.curl_v[o.n_out + p] + b.z) * rinv;
        o.curl_v[2 * o.n_out + p] = (o.curl_v[2 * o.n_out + p] + b.w) * rinv;
        o.nngb[p] += acc[s].nngb;
    }
}

}  // namespace pvsph
