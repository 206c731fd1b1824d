// density_v5.cuh -- the production sph_density_all engine (round 2).
//
// Method (identical to every other engine): every home particle i gathers from its own
// cell and the 26 neighbour cells; in a neighbour cell only the window of its list
// sorted along the pair axis whose projected separation is below H_i + delta is tested
// (Code 2; the per-particle bound of P:151-165); in-range pairs are interacted
// and the sums are written once per particle.
//
// What changed against v4 (same tiles from k_v4_tiles, same staging by bulk copies, same
// output records), all to cut issued instructions per candidate and per hit:
//  * List entries are staged as BYTE offsets of the staged particle (P + e, V + e): no
//    index scaling on the hot path.
//  * Each direction is swept on its own: the lane's two windows of direction d (a prefix
//    of the +d list, a suffix of the -d list) are one contiguous range L[wb, wb + tot) of
//    the reversed layout, so a candidate costs no window select.
//  * No per-candidate bounds test: the warp runs its longest window, and a lane whose
//    window is shorter keeps reading ITS -d segment beyond the window.  Those entries have
//    projected separation >= H_i + delta, hence r > H_i: the distance test rejects them
//    (the paper's windows are themselves padded: "max_index_a[i] is padded to a
//    multiple of the SIMD width").  Past the segment end the address is clamped (one
//    VIADDMNMX) onto a sentinel slot that points at a staged particle at infinity.
//  * Drains: two hits per lane with FFMA2/FMUL2/FADD2, w' and the h-derivative factor with
//    the constants folded into the finalisation, rsqrt refined by one Newton step.
//  * COUNT (statistics) counts exactly the window candidates (t < tot), i.e. Code 2.
#pragma once

#include "common.cuh"
#include "density.cuh"
#include "density_v4.cuh"
#include "packed.cuh"

namespace pvsph {

constexpr int V5_WARPS = V4_WARPS;
constexpr int V5_TP = V4_TP;
#ifndef V5_STAGE_V
#define V5_STAGE_V 1   // 0: (v, m) read from global memory (L1/L2) in the drains instead of staged
#endif
#ifndef V5_CTAS
#define V5_CTAS 2
#endif
#ifndef V5_CELLWIN
#define V5_CELLWIN 1   // 1: cell-uniform windows from the tile setup (broadcast sweeps); 0: per-lane bisection
#endif
#ifndef V5_TAIL2
#define V5_TAIL2 1     // sweep tails of 1-2 candidates in a 2-wide step (c5 -0.5 ms)
#endif
#ifndef V5_SELFTAIL
#define V5_SELFTAIL 1  // the self-cell sweep's tail in 4- or 2-wide steps (c5 -0.1 ms)
#endif
#ifndef V5_Q_DEPTH
#if V5_CELLWIN
#define V5_Q_DEPTH 30     // (with TILE_MS 2336 the window table fits beside 30 slots)
#else
#define V5_Q_DEPTH 30     // (two CTAs per SM leave ~1 KB of shared memory at 30)
#endif
#endif
constexpr int V5_Q = V5_Q_DEPTH;                       // hit stack depth per lane, 2-byte entries
#ifndef V5_NP
#define V5_NP 2        // packed pairs per drain round (2 NP hits per lane)
#endif
constexpr int V5_GUARD = 2 * V5_NP;                    // of which padding guard slots (see v5_particle)
#ifndef V5_TRIG
#define V5_TRIG 24     // drain when this many lanes hold 2 NP hits
#endif
#ifndef V5_CHK
#define V5_CHK 8       // candidates between drain checks (stacks kept below V5_Q - V5_GUARD - V5_CHK)
#endif
constexpr int V5_MS = V4_MS;                           // staged particles (+1 sentinel)
constexpr int V5_ML = V4_ML + 14 * V4_MAXH;            // list entries + sentinels: one per (home cell, direction) + one per home cell
constexpr int V5_MLA = (V5_ML + 7) / 8 * 8;
constexpr size_t V5_SMEM = (size_t)(V5_MS + 2) * 16 + (size_t)(V5_STAGE_V ? V5_MS + 2 : 0) * 16 + (size_t)V4_MAXCELLS * 16 +
                           (size_t)V5_MLA * 2 + (size_t)V4_HOFF * 4 + (size_t)V5_WARPS * V5_Q * 32 * 2 +
                           (size_t)V4_MAXZ * 16 + (size_t)V4_MAXCELLS * 4 + (size_t)(V5_CELLWIN ? V4_MAXH * 13 * 4 : 0);
static_assert(!V5_CELLWIN || V5_STAGE_V, "cell windows read h from the staged positions");
static_assert(V5_MS * 16 < 65536, "byte offsets of staged particles fit 16 bits");
static_assert(((V5_MS + 1) * 16) % 16 == 0 && (V5_MLA * 2) % 16 == 0, "16-byte aligned shared arrays");
static_assert(13 * V4_MAXH <= 2 * V5_TP, "two direction segments per thread");

// Dynamic shared memory of k_density_v5 (byte offsets from its start):
//   [0, V5_OFF_V)       P: float4 x, y, z, 0 per staged particle (low-face images pre-shifted
//                       by -L); P[V5_MS] = the far sentinel
//   [V5_OFF_V, ...)     V: float4 vx, vy, vz, m per staged particle
//   tab, L, hoff, hit stacks, seq.
// List entries and hit-stack entries are the 16-bit SHARED ADDRESSES of P entries (the
// kernel checks that P lies below 64 KiB of the shared window), so a candidate is loaded with
// one LDS.128 [e] and its (v, m) with LDS.128 [e + V5_OFF_V]: no base add on the hot path.
constexpr unsigned V5_OFF_V = (V5_MS + 2) * 16;
constexpr unsigned V5_OFF_TAB = V5_OFF_V + (V5_STAGE_V ? (V5_MS + 2) * 16 : 0);
constexpr unsigned V5_OFF_L = V5_OFF_TAB + V4_MAXCELLS * 16;

struct V5Stage {
    const int4 *tab;          // {base, count, gstart, flags | home count << 8}
    const float *tdx;         // per staged cell: max_dx since the build (0 without reuse)
    int nzs;
    unsigned sb;              // shared address of P[0]
    unsigned sl;              // shared address of L[0]
    unsigned sent;            // shared address of the list sentinel P[V5_MS] (NaN)
    unsigned pad;             // shared address of the drain padding P[V5_MS + 1] (far, finite, v = m = 0)
    const unsigned *win;      // V5_CELLWIN: per (home cell, direction) the cell's windows W+ | W- << 16
};

// Packed accumulators.  With q = min(x, u)(u + v) >= 0 the kernel slope is w' = -3 q and
// 3w + x w' = 3 (w - x q); the factors -3 and 3 are applied in the finalisation.
//   rho: m w, wc: w, srt: m (w - x q), st: (w - x q), Dq: m q/r (v_j - v_i).x_ij,
//   P/N: m q/r times the two products of (v_j - v_i) x x_ij.
struct Acc5 {
    f2 rho, wc, srt, st, Dq, Px, Nx, Py, Ny, Pz, Nz;
};

// Two interactions of one lane (hits j0, j1 of particle i), all arithmetic packed.
// M4 in branch-free form: w = u^3 - v^3/2, w' = -3 min(x, u)(u + v), u = max(0, 1 - x),
// v = max(0, 1 - 2x): equal to the two-branch R1 spline on [0, 1) (min(x, u) = u - v there,
// without cancellation) and exactly 0 (w, q and every term) for x >= 1, so a padding entry at
// the far sentinel contributes nothing and no mask is needed.
__device__ __forceinline__ void interact2(f2 nHinv, f2 dx, f2 dy, f2 dz, f2 m, f2 nvx, f2 nvy, f2 nvz, Acc5 &A)
{
    const f2 r2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    // r^2 = 0 (coincident particles, R7): rinv finite, x = 0 and min(x, u) = 0 zero every gradient term
    const f2 rinv = rsqrt_nr2(pk(fmaxf(r2.x, 1e-30f), fmaxf(r2.y, 1e-30f)));
    const f2 nx = mul2(mul2(r2, rinv), nHinv);                 // -x
    f2 u = add2(nx, bc2(1.0f));
    u = pk(fmaxf(u.x, 0.0f), fmaxf(u.y, 0.0f));
    f2 v = fma2(nx, bc2(2.0f), bc2(1.0f));
    v = pk(fmaxf(v.x, 0.0f), fmaxf(v.y, 0.0f));
    const f2 mn = pk(fminf(-nx.x, u.x), fminf(-nx.y, u.y));
    const f2 uu = mul2(u, u);
    const f2 w = fma2(uu, u, mul2(mul2(v, v), mul2(v, bc2(-0.5f))));
    const f2 q = mul2(mn, add2(u, v));
    acc_fma2(A.rho, m, w);
    acc_add2(A.wc, w);
    const f2 t = fma2(nx, q, w);                               // w - x q
    acc_fma2(A.srt, m, t);
    acc_add2(A.st, t);
    const f2 fac = mul2(mul2(m, q), rinv);
    acc_fma2(A.Dq, fac, fma2(nvx, dx, fma2(nvy, dy, mul2(nvz, dz))));
    const f2 fx = mul2(fac, nvx), fy = mul2(fac, nvy), fz = mul2(fac, nvz);
    acc_fma2(A.Px, fz, dy);
    acc_fma2(A.Nx, fy, dz);
    acc_fma2(A.Py, fx, dz);
    acc_fma2(A.Ny, fz, dx);
    acc_fma2(A.Pz, fy, dx);
    acc_fma2(A.Nz, fx, dy);
}

#ifdef V5_VOLATILE_BISECT
#define V5_LDU16 lds_u16
#define V5_LDF4 lds_f4
#else
#define V5_LDU16 ldsr_u16
#define V5_LDF4 ldsr_f4
#endif
// Windows of directions D0, D1 (four bisections in lockstep): the number of leading entries
// of each segment whose projected separation is below Hk.  Segment 2k (+d of direction k, read
// backwards from L[mid - 1]) has sep = (x_j - h) . d, segment 2k+1 (-d, forwards from L[mid])
// sep = (h - x_j) . d.  State per search: the shared address of the last entry known to be
// inside (or of L[mid] / L[mid - 1] when none is).  Probes are clamped onto the sentinel that
// bounds every segment (before the +d reversed list: the previous block's sentinel or the
// home cell's leading one; after the -d list: its own), whose separation is never below Hk,
// so no probe needs a validity test.  `top`: largest power of two <= the warp's longest
// segment, so all lanes run the same steps (the exact per-particle bound).
__device__ __forceinline__ void v5_windows2(int top, const unsigned amid[2], const unsigned lim[4], const float h[4][3],
                                            const float ax[2][3], const float Hk[4], int len[4])
{
    unsigned a[4] = {amid[0], amid[0] - 2u, amid[1], amid[1] - 2u};   // + side: L[mid]; - side: L[mid - 1]
    // (x_j - h, y_j - h) as one FADD2 against the negated home pair: the same bits as two FADDs
    f2 nh[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) nh[k] = pk(-h[k][0], -h[k][1]);
    for (int st = top; st > 0; st >>= 1) {
        const unsigned s2 = 2u * (unsigned)st;
        unsigned pa[4];
        pa[0] = max(a[0] - s2, lim[0]);
        pa[1] = min(a[1] + s2, lim[1]);
        pa[2] = max(a[2] - s2, lim[2]);
        pa[3] = min(a[3] + s2, lim[3]);
        unsigned e[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) e[k] = V5_LDU16(pa[k]);
        float4 p[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) p[k] = V5_LDF4(e[k]);
        // separations along the (unnormalised) direction; the - side measures h - x_j
        float sp[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float *A = ax[k >> 1];
            const f2 dxy = add2(pk(p[k].x, p[k].y), nh[k]);
            const float dz = p[k].z - h[k][2];
            const float sv = fmaf(A[0], dxy.x, fmaf(A[1], dxy.y, A[2] * dz));
            sp[k] = (k & 1) ? -sv : sv;
        }
        if (sp[0] < Hk[0]) a[0] = pa[0];
        if (sp[1] < Hk[1]) a[1] = pa[1];
        if (sp[2] < Hk[2]) a[2] = pa[2];
        if (sp[3] < Hk[3]) a[3] = pa[3];
    }
    len[0] = (int)(amid[0] - a[0]) >> 1;
    len[1] = (int)(a[1] + 2u - amid[0]) >> 1;
    len[2] = (int)(amid[1] - a[2]) >> 1;
    len[3] = (int)(a[3] + 2u - amid[1]) >> 1;
}

#ifdef V5_STATS
__device__ unsigned long long g_v5dbg[16];   // profiling counters (scripts: exp builds only)
#endif

// One lane = one home particle of a staged tile (see density_v4.cuh for the tile geometry).
// lpos: first list entry of its home cell's block, qh: its staged column, yoff: its row.
template <bool COUNT, bool FRAMES>
__device__ __forceinline__ void v5_particle(const DevGrid &g, const DevCells &c, OutRec *orec, const V5Stage &S,
                                            unsigned qbase, bool active, int i, int yoff, int qh, int lpos, int hidx,
                                            unsigned cand[4], unsigned hits[4], unsigned &band)
{
    // The lane's stack column: V5_GUARD guard slots holding the drain padding, then the entries
    // (sQ = the first entry slot): a drain pops 2 NP entries unconditionally, and a lane holding
    // fewer reads padding -- no per-entry test.
    const unsigned sQg = qbase + 2u * (threadIdx.x & 31);
    const unsigned sQ = sQg + 64u * V5_GUARD;
    float x = 0.f, y = 0.f, z = 0.f, vx = 0.f, vy = 0.f, vz = 0.f, m = 0.f, H2 = -1.f, Hinv = 0.f, Hd = 0.f;
    if (active) {
        const float4 a = c.xyzh[i];
        const float4 b = c.vm[i];
        x = a.x; y = a.y; z = a.z;
        vx = b.x; vy = b.y; vz = b.z; m = b.w;
        const double H = (double)g.gamma * (double)a.w;   // exact product; H^2, 1/H rounded once
        H2 = (float)(H * H);
        Hinv = (float)(1.0 / H);
        Hd = (float)H + g.delta0;                          // + 2 max_dx of the neighbour cell, per segment
    }
    const float xs = x - g.boxf[0], ys = y - g.boxf[1], zs = z - g.boxf[2];   // exact where used (x >= L/2)
    const f2 nxy = pk(-x, -y);
    const f2 nHinv = bc2(-Hinv);
    auto scell = [&](int ox, int oy, int oz) { return ((ox + 1) * 4 + oy + yoff + 1) * S.nzs + qh + oz; };
    const int4 eh = S.tab[scell(0, 0, 0)];
    const int kh = active ? i - eh.z : -1;                // in-cell index of i

    Acc5 A;
    A.rho = A.wc = A.srt = A.st = A.Dq = A.Px = A.Nx = A.Py = A.Ny = A.Pz = A.Nz = zero2();
    unsigned qp = sQ;                                     // stack top (next free slot)
    int npop = 0;
    {
        const unsigned pad = FRAMES ? (S.pad - S.sb) >> 4 : S.pad;   // staged index V5_MS + 1, frame 0
#pragma unroll
        for (int k = 0; k < V5_GUARD; ++k) sts_u16_push(sQg + 64u * k, pad);
    }

    auto home_of = [&](unsigned fl, float &hx, float &hy, float &hz) {
        hx = (fl & 1u) ? xs : x;
        hy = (fl & 2u) ? ys : y;
        hz = (fl & 4u) ? zs : z;
    };
    // Stack entries: the staged particle's shared address (FRAMES: staged index | frame bits
    // << 12).  A drain pops up to 2 NP entries per lane (fewer on lanes holding fewer; the
    // missing ones are the far sentinel, whose terms are exactly 0) and evaluates them in NP
    // independent packed pairs.
    auto drain = [&](auto np_tag) {
        constexpr int NP = decltype(np_tag)::value;
        const unsigned n = (qp - sQ) >> 6;
        const unsigned take = min(n, 2u * NP);
        unsigned qv[2 * NP];
#pragma unroll
        for (int s2 = 0; s2 < 2 * NP; ++s2) qv[s2] = lds_u16(qp - 64u * (s2 + 1));   // below sQ: padding
        qp -= 64u * take;
        npop += (int)take;
#ifdef V5_STATS
        {   // [10] drain lane-slots, [11] popped entries (real)
            const unsigned tk = __reduce_add_sync(0xffffffffu, take);
            if ((threadIdx.x & 31) == 0) { atomicAdd(&g_v5dbg[10], 64ull); atomicAdd(&g_v5dbg[11], (unsigned long long)tk); }
        }
#endif
#pragma unroll
        for (int pr = 0; pr < NP; ++pr) {
            unsigned e[2];
            float hxv[2], hyv[2], hzv[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const unsigned qq = qv[2 * pr + k];
                hxv[k] = x; hyv[k] = y; hzv[k] = z;
                if (FRAMES) {
                    e[k] = S.sb + ((qq & 0xfffu) << 4);
                    home_of(qq >> 12, hxv[k], hyv[k], hzv[k]);
                } else {
                    e[k] = qq;
                }
            }
            const float4 p0 = ldsr_f4(e[0]), p1 = ldsr_f4(e[1]);
#if V5_STAGE_V
            const float4 v0 = ldsr_f4_at<V5_OFF_V>(e[0]), v1 = ldsr_f4_at<V5_OFF_V>(e[1]);
#else
            // (v, m) from global memory: the staged position's w holds the particle's slot
            const float4 v0 = __ldg(c.vm + __float_as_int(p0.w)), v1 = __ldg(c.vm + __float_as_int(p1.w));
#endif
            interact2(nHinv, pk(hxv[0] - p0.x, hxv[1] - p1.x), pk(hyv[0] - p0.y, hyv[1] - p1.y),
                      pk(hzv[0] - p0.z, hzv[1] - p1.z), pk(v0.w, v1.w), pk(v0.x - vx, v1.x - vx),
                      pk(v0.y - vy, v1.y - vy), pk(v0.z - vz, v1.z - vz), A);
        }
    };
    // keep every stack below V5_Q - V5_GUARD - V5_CHK entries (V5_CHK pushes follow before the next check); drain
    // four per lane when most lanes hold four
    // (one warp reduction: lanes holding >= 2 NP count 1, lanes near a full stack count 32, so
    // the sum reaches V5_TRIG <= 32 iff V5_TRIG lanes hold 2 NP or some stack is nearly full)
    static_assert(V5_TRIG <= 32 && V5_Q - V5_GUARD - V5_CHK >= 2 * V5_NP, "drain trigger encoding");
    static_assert(V5_GUARD >= 2 * V5_NP, "a drain may read 2 NP slots below an empty stack");
    static_assert(V5_MS + 1 < 4096, "the padding's staged index fits the 12-bit FRAMES field");
    auto drain_check = [&]() {
        for (;;) {
            const unsigned n = (qp - sQ) >> 6;
            const unsigned vote = (n >= 2 * V5_NP ? 1u : 0u) + (n >= V5_Q - V5_GUARD - V5_CHK ? 32u : 0u);
            if (__reduce_add_sync(0xffffffffu, vote) < (unsigned)V5_TRIG) break;
            drain(std::integral_constant<int, V5_NP>{});
        }
    };

    // ---- the self cell: all j != i of the home cell (staged contiguously) ----
    {
        const int total = active ? eh.y : 0;
        const int trip = __reduce_max_sync(0xffffffffu, total);
        const unsigned pa = S.sb + 16u * (unsigned)eh.x;
        auto sstep = [&](int t, auto n_tag) {
            constexpr int NU = decltype(n_tag)::value;
#pragma unroll
            for (int u = 0; u < NU; ++u) {
                const int tt = t + u;
                const bool ok = tt < total && tt != kh;
                const unsigned e = ok ? pa + 16u * (unsigned)tt : S.sent;
                const float4 p = ldsr_f4(e);
                const f2 dxy = add2(pk(p.x, p.y), nxy);          // (x_j - x_i, y_j - y_i): one FADD2
                const float dz = z - p.z;
                const float r2 = fmaf(dxy.x, dxy.x, fmaf(dxy.y, dxy.y, dz * dz));
                if (COUNT) {
                    cand[0] += ok ? 1u : 0u;
                    band += ok && fabsf(r2 - H2) < 1e-6f * H2 ? 1u : 0u;
                }
                if (r2 < H2) {                             // the sentinel never passes
                    sts_u16_push(qp, FRAMES ? (e - S.sb) >> 4 : e);
                    qp += 64u;
                    if (COUNT) ++hits[0];
                }
            }
        };
        for (int t = 0; t < trip; t += 8) {
#if V5_SELFTAIL
            if (t + 4 < trip)
                sstep(t, std::integral_constant<int, 8>{});
            else if (t + 2 < trip)
                sstep(t, std::integral_constant<int, 4>{});
            else
                sstep(t, std::integral_constant<int, 2>{});
#else
            sstep(t, std::integral_constant<int, 8>{});
#endif
            drain_check();
        }
    }

#if V5_CELLWIN
    // ---- 13 directions, cell-uniform windows (DESIGN.md §4.4 "v5, cell windows") ----
    // The tile setup stored, per (home cell, direction), the union over the cell's home
    // particles of their exact windows (W+ leading entries of the +d list, W- of the -d list,
    // the paper's Code 2 bound with the cell's h_max: P:94-100).  Every lane of a home
    // cell sweeps the same range L[mid - W+, mid + W-), so the lanes of one cell read the same
    // list entry and the same staged particle (shared-memory broadcasts); an entry outside the
    // lane's own window has projected separation >= H_i + delta, so r > H_i and the distance test
    // rejects it (R16).  COUNT counts exactly the lane's own Code 2 window (sep < H_i + delta).
    int pos = lpos + 1;                                   // after the home cell's leading sentinel
#pragma unroll 1
    for (int d = 0; d < 13; ++d) {
        const int4 dv = c_dirs[d];
        const int kind = dv.w;
        const int cp = scell(dv.x, dv.y, dv.z), cm = scell(-dv.x, -dv.y, -dv.z);
        const int4 ep = S.tab[cp];
        const int4 em = S.tab[cm];
        const int mid = pos + ep.y;                       // boundary between the two reversed segments
        const int sent = mid + em.y;                      // the sentinel slot after the -d segment
        pos = sent + 1;
        const unsigned wv = active ? S.win[hidx * 13 + d] : 0u;
        const int W0 = (int)(wv & 0xffffu), tot = W0 + (int)(wv >> 16);
        const unsigned fl0k = FRAMES ? (unsigned)ep.w & 7u : 0u, fl1k = FRAMES ? (unsigned)em.w & 7u : 0u;
        // COUNT only: the lane's exact window thresholds (as the per-lane bisection used them)
        float cax[3] = {0.f, 0.f, 0.f}, chp[3] = {0.f, 0.f, 0.f}, chm[3] = {0.f, 0.f, 0.f}, cHp = -3e38f, cHm = -3e38f;
        if (COUNT) {
            const float sk = kind == 1 ? 1.0f : (kind == 2 ? 1.41421356237309505f : 1.73205080756887729f);
            cax[0] = (float)dv.x; cax[1] = (float)dv.y; cax[2] = (float)dv.z;
            home_of(fl0k, chp[0], chp[1], chp[2]);
            home_of(fl1k, chm[0], chm[1], chm[2]);
            if (active) {
                cHp = fmaf(2.0f, S.tdx[cp], Hd) * sk;
                cHm = fmaf(2.0f, S.tdx[cm], Hd) * sk;
            }
        }
        const int trip = __reduce_max_sync(0xffffffffu, tot);
        const unsigned lb = S.sl + 2u * (unsigned)(mid - W0);
        const unsigned ls = S.sl + 2u * (unsigned)sent;
        auto step = [&](int t, auto n_tag) {
            constexpr int NU = decltype(n_tag)::value;
            unsigned e[NU];
#pragma unroll
            for (int u = 0; u < NU; ++u) e[u] = ldsr_u16(min(lb + 2u * (unsigned)(t + u), ls));
            float4 pp[NU];
#pragma unroll
            for (int u = 0; u < NU; ++u) pp[u] = ldsr_f4(e[u]);
#pragma unroll
            for (int u = 0; u < NU; ++u) {
                const float4 p = pp[u];
                unsigned fl = 0;
                float dx, dy, dz;
                if (FRAMES) {
                    float hx = x, hy = y, hz = z;
                    fl = t + u < W0 ? fl0k : fl1k;
                    home_of(fl, hx, hy, hz);
                    dx = hx - p.x; dy = hy - p.y; dz = hz - p.z;
                } else {
                    const f2 dxy = add2(pk(p.x, p.y), nxy);  // one FADD2; squares as before
                    dx = dxy.x; dy = dxy.y; dz = z - p.z;
                }
                const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                if (COUNT) {
                    const bool plus = t + u < W0;
                    const float *hh = plus ? chp : chm;
                    const f2 dxy = add2(pk(p.x, p.y), pk(-hh[0], -hh[1]));
                    const float sv = fmaf(cax[0], dxy.x, fmaf(cax[1], dxy.y, cax[2] * (p.z - hh[2])));
                    const bool inw = t + u < tot && (plus ? sv < cHp : -sv < cHm);
                    cand[kind] += inw ? 1u : 0u;
                    band += inw && fabsf(r2 - H2) < 1e-6f * H2 ? 1u : 0u;
                }
                if (r2 < H2) {                             // outside the lane's window: never (sep >= H + delta)
                    sts_u16_push(qp, FRAMES ? ((e[u] - S.sb) >> 4) | (fl << 12) : e[u]);
                    qp += 64u;
                    if (COUNT) ++hits[kind];
                }
            }
        };
        for (int t0 = 0; t0 < trip; t0 += V5_CHK) {
#pragma unroll 1
            for (int t = t0; t < min(t0 + V5_CHK, trip); t += 8) {
                if (t + 4 < trip)
                    step(t, std::integral_constant<int, 8>{});
#if V5_TAIL2
                else if (t + 2 < trip)                    // a tail of 3 or 4 candidates
                    step(t, std::integral_constant<int, 4>{});
                else                                      // a tail of 1 or 2
                    step(t, std::integral_constant<int, 2>{});
#else
                else                                      // a tail of <= 4 candidates
                    step(t, std::integral_constant<int, 4>{});
#endif
            }
            drain_check();
        }
    }
#else
    // ---- 13 directions: windows two directions at a time, then one sweep per direction ----
    int pos = lpos + 1;                                   // after the home cell's leading sentinel
    for (int d0 = 0; d0 < 13; d0 += 2) {
        const int nd = d0 + 1 < 13 ? 2 : 1;
        int mid[2] = {0, 0}, sent[2] = {0, 0};
        unsigned fl0v[2] = {0, 0}, fl1v[2] = {0, 0};
        unsigned amid[2] = {S.sl, S.sl}, lim[4] = {S.sl, S.sl, S.sl, S.sl};
        float hh[4][3];
        float Hkv[4] = {-3e38f, -3e38f, -3e38f, -3e38f};
        float axv[2][3] = {{0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f}};
        int nmax = 0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int d = d0 + k;
            hh[2 * k][0] = hh[2 * k + 1][0] = x;
            hh[2 * k][1] = hh[2 * k + 1][1] = y;
            hh[2 * k][2] = hh[2 * k + 1][2] = z;
            if (k < nd) {
                const int4 dv = c_dirs[d];
                const int kind = dv.w;
                const float sk = kind == 1 ? 1.0f : (kind == 2 ? 1.41421356237309505f : 1.73205080756887729f);
                const int a0 = dv.x, a1 = dv.y, a2 = dv.z;
                axv[k][0] = (float)a0;
                axv[k][1] = (float)a1;
                axv[k][2] = (float)a2;
                const int cp = scell(a0, a1, a2), cm = scell(-a0, -a1, -a2);
                const int4 ep = S.tab[cp];
                const int4 em = S.tab[cm];
                // window thresholds (H + delta + 2 max_dx(neighbour)) sqrt(kind): the stale list order
                // of a drifted cell is off by at most 2 max_dx
                Hkv[2 * k] = fmaf(2.0f, S.tdx[cp], Hd) * sk;
                Hkv[2 * k + 1] = fmaf(2.0f, S.tdx[cm], Hd) * sk;
                mid[k] = pos + ep.y;                      // boundary between the two reversed segments
                sent[k] = mid[k] + em.y;                  // the sentinel slot after the -d segment
                amid[k] = S.sl + 2u * (unsigned)mid[k];
                lim[2 * k] = S.sl + 2u * (unsigned)(pos - 1);   // the sentinel before the +d segment
                lim[2 * k + 1] = S.sl + 2u * (unsigned)sent[k];
                pos = sent[k] + 1;
                nmax = max(nmax, max(ep.y, em.y));
                if (FRAMES) {
                    fl0v[k] = (unsigned)ep.w & 7u;
                    fl1v[k] = (unsigned)em.w & 7u;
                    home_of(fl0v[k], hh[2 * k][0], hh[2 * k][1], hh[2 * k][2]);
                    home_of(fl1v[k], hh[2 * k + 1][0], hh[2 * k + 1][1], hh[2 * k + 1][2]);
                }
            }
        }
        if (!active) Hkv[0] = Hkv[1] = Hkv[2] = Hkv[3] = -3e38f;   // inactive lanes (position 0): empty windows
        nmax = __reduce_max_sync(0xffffffffu, nmax);
        const int top = nmax > 0 ? 1 << (31 - __clz(nmax)) : 0;
        int len[4] = {0, 0, 0, 0};
        v5_windows2(top, amid, lim, hh, axv, Hkv, len);
#pragma unroll 1
        for (int k = 0; k < nd; ++k) {
            const int kind = c_dirs[d0 + k].w;
            // (selects, not indexing: the loop is not unrolled, to keep one copy of the drains)
            const int len0 = k ? len[2] : len[0], tot = len0 + (k ? len[3] : len[1]);
            const unsigned fl0k = k ? fl0v[1] : fl0v[0], fl1k = k ? fl1v[1] : fl1v[0];
            const int trip = __reduce_max_sync(0xffffffffu, tot);
            const unsigned lb = S.sl + 2u * (unsigned)((k ? mid[1] : mid[0]) - len0);
            const unsigned ls = S.sl + 2u * (unsigned)(k ? sent[1] : sent[0]);
            auto step = [&](int t, auto n_tag) {
                constexpr int NU = decltype(n_tag)::value;
                unsigned e[NU];
#pragma unroll
                for (int u = 0; u < NU; ++u) e[u] = ldsr_u16(min(lb + 2u * (unsigned)(t + u), ls));
                float4 pp[NU];
#pragma unroll
                for (int u = 0; u < NU; ++u) pp[u] = ldsr_f4(e[u]);
#pragma unroll
                for (int u = 0; u < NU; ++u) {
                    const float4 p = pp[u];
                    unsigned fl = 0;
                    float dx, dy, dz;
                    if (FRAMES) {
                        float hx = x, hy = y, hz = z;
                        fl = t + u < len0 ? fl0k : fl1k;
                        home_of(fl, hx, hy, hz);
                        dx = hx - p.x; dy = hy - p.y; dz = hz - p.z;
                    } else {
                        const f2 dxy = add2(pk(p.x, p.y), nxy);  // one FADD2; squares as before
                        dx = dxy.x; dy = dxy.y; dz = z - p.z;
                    }
                    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                    if (COUNT) {
                        cand[kind] += t + u < tot ? 1u : 0u;
                        band += t + u < tot && fabsf(r2 - H2) < 1e-6f * H2 ? 1u : 0u;
                    }
                    if (r2 < H2) {                         // beyond the window: never (sep >= H + delta)
                        sts_u16_push(qp, FRAMES ? ((e[u] - S.sb) >> 4) | (fl << 12) : e[u]);
                        qp += 64u;
                        if (COUNT) ++hits[kind];
                    }
                }
            };
#ifdef V5_STATS
            {   // [12] sweep lane-slots, [13] window candidates, [14] final-drain rounds
                const unsigned tt = __reduce_add_sync(0xffffffffu, (unsigned)tot);
                if ((threadIdx.x & 31) == 0) {
                    atomicAdd(&g_v5dbg[12], 32ull * (unsigned long long)(((trip + 7) / 8) * 8 - ((trip % 8) && (trip % 8) <= 4 ? 4 : 0)));
                    atomicAdd(&g_v5dbg[13], (unsigned long long)tt);
                }
            }
#endif
            for (int t0 = 0; t0 < trip; t0 += V5_CHK) {
#pragma unroll 1
                for (int t = t0; t < min(t0 + V5_CHK, trip); t += 8) {
                    if (t + 4 < trip)
                        step(t, std::integral_constant<int, 8>{});
                    else                                  // a tail of <= 4 candidates
                        step(t, std::integral_constant<int, 4>{});
                }
                drain_check();
            }
        }
    }
#endif
#ifdef V5_STATS
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_v5dbg[9], 1ull);          // [9] warps
    {
        const unsigned left = __reduce_add_sync(0xffffffffu, (qp - sQ) >> 6);
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_v5dbg[15], (unsigned long long)left);   // [15] hits left for the final drain
    }
#endif
    while (__any_sync(0xffffffffu, qp != sQ)) drain(std::integral_constant<int, V5_NP>{});

    if (active) {
        // finalise: self term w(0) = 1/2, w(0) - 0 q = 1/2; K3 = 16/(pi H^3); rho_dh = -(K3 gamma/H) (3/2 m + 3 S_t);
        // div = -(K3/H)(-3) D/rho with D = sum m q/r (v_j - v_i).x_ij ... see DESIGN.md §4.4
        const float K3 = (16.0f / kPi) * Hinv * Hinv * Hinv;
        const float rho = K3 * fmaf(0.5f, m, sum2(A.rho));
        const float wc = K3 * (0.5f + sum2(A.wc));
        const float dh = -3.0f * K3 * g.gamma * Hinv;
        const float rho_dh = dh * fmaf(0.5f, m, sum2(A.srt));
        const float wc_dh = dh * (0.5f + sum2(A.st));
        const float gf = -3.0f * K3 * Hinv / rho;
        store_rec(orec, c.perm[i], rho, wc, rho_dh, wc_dh, gf * sum2(A.Dq), gf * (sum2(A.Px) - sum2(A.Nx)),
                  gf * (sum2(A.Py) - sum2(A.Ny)), gf * (sum2(A.Pz) - sum2(A.Nz)), npop);
    }
}

// Persistent CTAs over the k_v4_tiles list (same tiles and staging as v4; list block layout
// per home cell: for d = 0..12 the +d list reversed, the -d list reversed, one sentinel).
template <bool COUNT>
__global__ void __launch_bounds__(V5_TP, V5_CTAS) k_density_v5(DevGrid g, DevCells c, OutRec *orec, sph_stats *st,
                                                          const int4 *__restrict__ tiles,
                                                          const int *__restrict__ ntiles_p, int *tile_counter,
                                                          const unsigned *__restrict__ genp, unsigned *status)
{
    extern __shared__ __align__(16) unsigned char v5_smem[];
    float4 *P = reinterpret_cast<float4 *>(v5_smem);
    float4 *V = P + V5_MS + 2;
    int4 *tab = reinterpret_cast<int4 *>(V + (V5_STAGE_V ? V5_MS + 2 : 0));
    uint16_t *L = reinterpret_cast<uint16_t *>(tab + V4_MAXCELLS);
    int *hoff = reinterpret_cast<int *>(L + V5_MLA);
    uint16_t *queue = reinterpret_cast<uint16_t *>(hoff + V4_HOFF);
    int4 *seq = reinterpret_cast<int4 *>(queue + V5_WARPS * V5_Q * 32);
    float *tdx = reinterpret_cast<float *>(seq + V4_MAXZ);
    unsigned *win = reinterpret_cast<unsigned *>(tdx + V4_MAXCELLS);   // V5_CELLWIN only
    __shared__ int4 s_next;
    __shared__ int s_wsum[V5_WARPS];
    __shared__ __align__(8) unsigned long long s_mbar;
    const unsigned mbar = smem_addr(&s_mbar);
    unsigned mbar_phase = 0;

    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const RowPairs rp = row_pairs(g);
    const int ntiles = *ntiles_p;
    unsigned cand[4] = {0, 0, 0, 0}, hits[4] = {0, 0, 0, 0}, band = 0;
    const int4 kEnd = make_int4(-1, 0, 0, 0);
    const unsigned sb = smem_addr(P);
    // entries are 16-bit shared addresses of P: P must lie in the first 64 KiB of the window
    // (it does: P starts the dynamic shared memory, after ~1 KiB of static shared memory)
    if (sb + 16u * (V5_MS + 2) > 65536u) {
        if (threadIdx.x == 0) set_status(status, ST_EINVAL);
        return;
    }

    int pf_start[2] = {0, 0}, pf_end[2] = {0, 0}, pf_nh[2] = {0, 0};
    float pf_dx[2] = {0.0f, 0.0f};
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
                pf_dx[k] = c.cell_dx[cell];
            }
        }
    };
    if (threadIdx.x == 0) {
        const int t0 = atomicAdd(tile_counter, 1);
        s_next = t0 < ntiles ? tiles[t0] : kEnd;
        s_gen = *genp;
        // sentinels (never restaged).  P[V5_MS]: the list sentinel, NaN coordinates, so every
        // comparison with it is false (window probes on either side, distance tests).
        // P[V5_MS + 1]: the drain padding, far but finite (r^2 ~ 3e30) with (v, m) = 0, whose
        // terms evaluate to exactly 0 (x >> 1, q = w = 0).
        const float qnan = __int_as_float(0x7fc00000);
        P[V5_MS] = make_float4(qnan, qnan, qnan, 0.0f);
        if (V5_STAGE_V) V[V5_MS] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        P[V5_MS + 1] = make_float4(1e15f, 1e15f, 1e15f, 0.0f);
        if (V5_STAGE_V) V[V5_MS + 1] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int4 td = s_next;
    prefetch(td);

    while (td.x >= 0) {
        __syncthreads();                                  // s_next consumed, previous tile done
        if (threadIdx.x == 0) {
            const int t1 = atomicAdd(tile_counter, 1);
            s_next = t1 < ntiles ? tiles[t1] : kEnd;
        }
        const TileGeom T = tile_geom(g, rp, td);
        bool staged = T.staged;
        if (staged) {
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
                    ent[k] = make_int4(0, cnt2[k], pf_start[k], (int)fl | (pf_nh[k] << 8));
                }
            }
            if (2 * threadIdx.x < ncs) {
                tab[2 * threadIdx.x] = ent[0];
                tdx[2 * threadIdx.x] = pf_dx[0];
            }
            if (2 * threadIdx.x + 1 < ncs) {
                tab[2 * threadIdx.x + 1] = ent[1];
                tdx[2 * threadIdx.x + 1] = pf_dx[1];
            }
            __syncthreads();
            // direction blocks: (home cell h, direction d) -> n(+d) + n(-d) + 1 entries; two per thread
            const int ndseg = 13 * T.nh;
            int dsz[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int gs = 2 * threadIdx.x + j;
                dsz[j] = 0;
                if (gs < ndseg) {
                    const int h = gs / 13, d = gs % 13;
                    const int r = h / T.nzh, q = h % T.nzh + 1;
                    const int4 dv = c_dirs[d];
                    const int a0 = dv.x, a1 = dv.y, a2 = dv.z;
                    dsz[j] = tab[((a0 + 1) * 4 + a1 + r + 1) * T.nzs + q + a2].y +
                             tab[((-a0 + 1) * 4 - a1 + r + 1) * T.nzs + q - a2].y + 1 + (d == 0 ? 1 : 0);
                }
            }
            if (wl == V5_WARPS - 1) {
                int4 sl = make_int4(0, 0, 0, 0);
                int ns = 0;
                if (lane < T.nzh) {
                    const int4 ea = tab[5 * T.nzs + lane + 1];
                    const int4 eb = tab[6 * T.nzs + lane + 1];
                    sl = make_int4(ea.z, ea.w >> 8, eb.z, 0);
                    ns = (ea.w >> 8) + (T.hasB ? (eb.w >> 8) : 0);
                }
                int xx = ns;
#pragma unroll
                for (int o2 = 1; o2 < 32; o2 <<= 1) {
                    const int yv = __shfl_up_sync(0xffffffffu, xx, o2);
                    if (lane >= o2) xx += yv;
                }
                sl.w = xx - ns;
                if (lane < T.nzh) seq[lane] = sl;
            }
            int ptot;
            const int pp = block_exscan((cnt2[0] + cnt2[1]) | ((dsz[0] + dsz[1]) << 16), s_wsum, ptot);
            const int total = ptot & 0xffff, ltotal = ptot >> 16;
            const int pre = pp & 0xffff;
            int lpre = pp >> 16;
            if (2 * threadIdx.x < ncs) tab[2 * threadIdx.x].x = pre;
            if (2 * threadIdx.x + 1 < ncs) tab[2 * threadIdx.x + 1].x = pre + cnt2[0];
            int *segoff = reinterpret_cast<int *>(queue);        // scratch: the hit stacks are idle now
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int gs = 2 * threadIdx.x + j;
                if (gs < ndseg) {
                    segoff[gs] = lpre;
                    if (gs % 13 == 0) hoff[gs / 13] = lpre;
                }
                lpre += dsz[j];
            }
            if (total > V5_MS || ltotal > V5_ML || T.nh > V4_MAXH) staged = false;   // CTA-uniform
            __syncthreads();
            if (staged) {
                if (wl == 0) {
                    if (lane == 0) mbar_expect_tx(mbar, (unsigned)total * (V5_STAGE_V ? 32u : 16u));
                    __syncwarp();
                    const bool wlo = T.za == 0, whi = T.zb + 1 >= g.nz;
                    for (int job = lane; job < V4_ROWS * 3; job += 32) {
                        const int r = job / 3, piece = job % 3;
                        const int q0 = piece == 0 ? 0 : (piece == 1 ? (wlo ? 1 : 0) : T.nzs - 1);
                        const int q1 = piece == 0 ? (wlo ? 1 : 0) : (piece == 1 ? (whi ? T.nzs - 1 : T.nzs) : (whi ? T.nzs : T.nzs - 1));
                        if (q1 <= q0) continue;
                        const int4 ea = tab[r * T.nzs + q0];
                        const int4 eb = tab[r * T.nzs + q1 - 1];
                        const unsigned bytes = (unsigned)(eb.x + eb.y - ea.x) * 16u;
                        if (bytes == 0) continue;
                        bulk_g2s(smem_addr(P + ea.x), c.xyzh + ea.z, bytes, mbar);
                        if (V5_STAGE_V) bulk_g2s(smem_addr(V + ea.x), c.vm + ea.z, bytes, mbar);
                    }
                }
                // list segments (2 per direction block), entries turned into staged byte offsets
                const int nseg = 2 * ndseg;
                for (int gs2 = threadIdx.x; gs2 < nseg; gs2 += V5_TP) {
                    const int gs = gs2 >> 1, neg = gs2 & 1;
                    const int h = gs / 13, d = gs % 13, sg = neg ? -1 : 1;
                    const int r = h / T.nzh, q = h % T.nzh + 1;
                    const int4 dv = c_dirs[d];
                    const int a0 = dv.x, a1 = dv.y, a2 = dv.z;
                    const int4 ep = tab[((a0 + 1) * 4 + a1 + r + 1) * T.nzs + q + a2];
                    const int4 e = neg ? tab[((-a0 + 1) * 4 - a1 + r + 1) * T.nzs + q - a2] : ep;
                    const int mid = segoff[gs] + (d == 0 ? 1 : 0) + ep.y;
                    if (d == 0 && !neg) L[segoff[gs]] = (uint16_t)(sb + 16u * V5_MS);   // the home cell's leading sentinel
                    // +d reversed ends at mid - 1 (entry 0 at mid - 1); -d reversed starts at mid
                    // (its LAST list entry first); the sentinel after it
                    const int dst0 = neg ? mid + e.y - 1 : mid - 1;        // slot of list entry 0
                    if (neg) L[mid + e.y] = (uint16_t)(sb + 16u * V5_MS);
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
                            const int k = 8 * (w0 + u) - mis;
                            const unsigned wd[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                            for (int t = 0; t < 8; ++t) {
                                const unsigned qv = (t & 1) ? wd[t >> 1] >> 16 : wd[t >> 1] & 0xffffu;
                                if (k + t >= 0 && k + t < e.y) L[dst0 - k - t] = (uint16_t)(sb + 16u * (e.x + qv));
                            }
                        }
                    }
                }
                mbar_wait(mbar, mbar_phase);
                mbar_phase ^= 1u;
                if (!V5_STAGE_V || T.za == 0 || T.y0 == 0 || g.x_lo + T.xo == 0) {
                    // staged cells of a -L periodic image (flags 3-5): x_j - L, exact (x_j >= L/2);
                    // without staged (v, m): every staged position's w becomes its global slot
                    __syncthreads();
                    for (int sc = wl; sc < V4_ROWS * T.nzs; sc += V5_WARPS) {
                        const int4 e = tab[sc];
                        if (V5_STAGE_V && !(e.w & 56)) continue;
                        const float sx = (e.w & 8) ? g.boxf[0] : 0.0f;
                        const float sy = (e.w & 16) ? g.boxf[1] : 0.0f;
                        const float sz = (e.w & 32) ? g.boxf[2] : 0.0f;
                        for (int k = lane; k < e.y; k += 32) {
                            float4 qv = P[e.x + k];
                            qv.x -= sx;
                            qv.y -= sy;
                            qv.z -= sz;
                            if (!V5_STAGE_V) qv.w = __int_as_float(e.z + k);
                            P[e.x + k] = qv;
                        }
                    }
                }
                __syncthreads();
#if V5_CELLWIN
                // Cell windows: per (home cell h, direction d) the union over h's home particles k
                // of their exact windows, from a bound of the largest reach U+ = max_k (x_k.a + H_k
                // + delta + 2 max_dx(c+d)) |a| (frames: the home side shifted as the lanes do), and
                // U- the smallest; W+ = number of leading +d entries with x_j.a < U+, W- = leading
                // -d entries with x_j.a > U-, by bisection on the staged (sorted) lists.  The bounds
                // are widened by eps (fp32 rounding of the projections): a superset of every
                // lane's window is all the sweep needs (R16).
                {
                    const float eps = 0x1p-18f * (fabsf(g.boxf[0]) + fabsf(g.boxf[1]) + fabsf(g.boxf[2]));
                    const int njob = 13 * T.nh;
                    const int *segoff = reinterpret_cast<const int *>(queue);
                    for (int gs = threadIdx.x; gs < njob; gs += V5_TP) {
                        const int h = gs / 13, d = gs % 13;
                        const int r = h / T.nzh, q = h % T.nzh + 1;
                        const int4 dv = c_dirs[d];
                        const float a0 = (float)dv.x, a1 = (float)dv.y, a2 = (float)dv.z;
                        const float sk = dv.w == 1 ? 1.0f : (dv.w == 2 ? 1.41421356237309505f : 1.73205080756887729f);
                        const int4 eh = tab[(4 + r + 1) * T.nzs + q];
                        const int cp = ((dv.x + 1) * 4 + dv.y + r + 1) * T.nzs + q + dv.z;
                        const int cm = ((-dv.x + 1) * 4 - dv.y + r + 1) * T.nzs + q - dv.z;
                        const int4 ep = tab[cp], em = tab[cm];
                        const int nhome = eh.w >> 8;
                        float up = -3e38f, um = 3e38f;
                        for (int k = 0; k < nhome; ++k) {
                            const float4 p4 = P[eh.x + k];
                            const float sp = fmaf(a0, p4.x, fmaf(a1, p4.y, a2 * p4.z));
                            const float hb = fmaf(g.gamma, p4.w, g.delta0) * 1.000001f * sk;   // >= the lane's (H + delta) |a|
                            up = fmaxf(up, sp + hb);
                            um = fminf(um, sp - hb);
                        }
                        auto fshift = [&](unsigned fl) {                 // (x - L f) . a = x . a - fshift
                            return (fl & 1u ? g.boxf[0] * a0 : 0.0f) + (fl & 2u ? g.boxf[1] * a1 : 0.0f) +
                                   (fl & 4u ? g.boxf[2] * a2 : 0.0f);
                        };
                        const unsigned flp = T.frames ? (unsigned)ep.w & 7u : 0u, flm = T.frames ? (unsigned)em.w & 7u : 0u;
                        up = up - fshift(flp) + 2.0f * tdx[cp] * sk * 1.000001f + eps;
                        um = um - fshift(flm) - 2.0f * tdx[cm] * sk * 1.000001f - eps;
                        const int mid = segoff[gs] + (d == 0 ? 1 : 0) + ep.y;
                        int w0 = 0, w1 = 0;
                        if (nhome > 0) {
                            const unsigned lbase = smem_addr(L);
                            for (int st = ep.y > 0 ? 1 << (31 - __clz(ep.y)) : 0; st > 0; st >>= 1)
                                if (w0 + st <= ep.y) {
                                    const float4 pj = ldsr_f4(ldsr_u16(lbase + 2u * (unsigned)(mid - w0 - st)));
                                    if (fmaf(a0, pj.x, fmaf(a1, pj.y, a2 * pj.z)) < up) w0 += st;
                                }
                            for (int st = em.y > 0 ? 1 << (31 - __clz(em.y)) : 0; st > 0; st >>= 1)
                                if (w1 + st <= em.y) {
                                    const float4 pj = ldsr_f4(ldsr_u16(lbase + 2u * (unsigned)(mid + w1 + st - 1)));
                                    if (fmaf(a0, pj.x, fmaf(a1, pj.y, a2 * pj.z)) > um) w1 += st;
                                }
                        }
                        win[gs] = (unsigned)w0 | ((unsigned)w1 << 16);
                    }
                }
                __syncthreads();
#endif
            }
        }
        __syncthreads();
        const int4 td_next = s_next;
        prefetch(td_next);

        auto home_slot = [&](int h, int &slot, int &yo, int &tz) {
            const int qq = T.first + h;
            int lo = 0, hi = T.nzh - 1;
            while (lo < hi) {
                const int md = (lo + hi + 1) >> 1;
                if (seq[md].w <= qq) lo = md; else hi = md - 1;
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
            const V5Stage S{tab, tdx, T.nzs, sb, smem_addr(L), sb + 16u * V5_MS, sb + 16u * (V5_MS + 1), win};
            const unsigned qb = smem_addr(queue + wl * V5_Q * 32);
            if (wl * 32 < T.cnt) {
                if (T.frames)
                    v5_particle<COUNT, true>(g, c, orec, S, qb, active, i, yoff, tz + 1, lpos, yoff * T.nzh + tz, cand, hits, band);
                else
                    v5_particle<COUNT, false>(g, c, orec, S, qb, active, i, yoff, tz + 1, lpos, yoff * T.nzh + tz, cand, hits, band);
            }
        } else if (T.cnt > 0) {
            const long long rowA = ((long long)(T.xo + g.ghost_x) * g.ny + T.y0) * g.nz;
            const int ntot = T.cnt > 0 ? T.cnt : -T.cnt;
            for (int h = threadIdx.x; h < ntot; h += V5_TP) {
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
    flush_stats<COUNT>(st, cand, hits, band);
}

// sph_calibrate mode 3: the production interaction (interact2, two hits per lane with
// FFMA2/FMUL2/FADD2, exactly as the v5 drains evaluate them) on full masks: every thread is one
// i interacting with CALIB_NJ shared-memory neighbours per pass, no neighbour search (the
// Table 2 analogue, for the engine the bench runs).
__global__ void k_calib_interact2(float *out, int iters)
{
    constexpr int NJ = 256;
    __shared__ float4 sx[NJ], sv[NJ];
    for (int k = threadIdx.x; k < NJ; k += blockDim.x) {
        const float t = (float)k / NJ;
        sx[k] = make_float4(0.01f * t, 0.02f * (1.f - t), 0.005f * t, 0.f);
        sv[k] = make_float4(t, -t, 0.5f * t, 1e-3f);
    }
    __syncthreads();
    const float x = 0.0101f, y = 0.0102f, z = 0.0053f, vx = 0.3f, vy = -0.2f, vz = 0.1f;
    const f2 nHinv = bc2(-1.0f / 0.05f);
    Acc5 A;
    A.rho = A.wc = A.srt = A.st = A.Dq = A.Px = A.Nx = A.Py = A.Ny = A.Pz = A.Nz = zero2();
    for (int i = 0; i < iters; ++i)
        for (int k = 0; k < NJ; k += 2) {
            const float4 p0 = sx[k], p1 = sx[k + 1], v0 = sv[k], v1 = sv[k + 1];
            interact2(nHinv, pk(x - p0.x, x - p1.x), pk(y - p0.y, y - p1.y), pk(z - p0.z, z - p1.z), pk(v0.w, v1.w),
                      pk(v0.x - vx, v1.x - vx), pk(v0.y - vy, v1.y - vy), pk(v0.z - vz, v1.z - vz), A);
        }
    const float s = sum2(A.rho) + sum2(A.wc) + sum2(A.srt) + sum2(A.st) + sum2(A.Dq) + sum2(A.Px) + sum2(A.Nx) +
                    sum2(A.Py) + sum2(A.Ny) + sum2(A.Pz) + sum2(A.Nz);
    if (s == 123.456f) out[0] = s;
}

}  // namespace pvsph
