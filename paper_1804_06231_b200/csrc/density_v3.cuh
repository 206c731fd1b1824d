// density_v3.cuh -- the production sph_density_all engine.
//
// Same method and per-particle arithmetic as the reference engine (density.cuh),
// mapped onto the SIMT machine as follows:
//
//  * A warp owns 32 consecutive slots of the cell-sorted arrays (lane = particle
//    i), so lanes are filled across cell boundaries.
//  * The 27 cells are visited as the self cell plus 13 direction pairs: for the
//    sort direction d the lane's window in the +d neighbour (a prefix of its list
//    sorted along d) is followed by its window in the -d neighbour (a suffix of
//    the same-direction list).  The two lengths are anti-correlated (a particle
//    near the +d face sees much of +d and little of -d), so the per-lane total of
//    a pair varies far less than either window.
//  * Windows are exact: each lane binary-searches its bound on the sorted keys
//    (the bound of P:151-165 computed exactly instead of by the single pass of
//    the paper).  The warp then runs a loop of uniform trip count max(total); a
//    lane tests candidate t of its own concatenated window while t < total.
//    Lanes of one home cell read the same list region, so the loads stay
//    L1-friendly (no shared-memory staging: L1 keeps its full size).
//  * The candidate test computes r^2 only.  An in-range pair is pushed
//    into the lane's hit queue in shared memory; hit k is stored in half (k & 1)
//    of a packed pair slot, so a pop yields f32x2 operands directly and every
//    particle sums its hits in sweep order whatever the warp does (deterministic,
//    identical on any number of GPUs).  The left-packing of in-range candidates
//    of P:185 ("if (ANY(mask))") becomes this compaction.
//  * When most lanes hold a full pair (or a queue is nearly full) the warp pops
//    one pair per lane and evaluates both interactions with FFMA2/FADD2/FMUL2,
//    accumulating in registers; one writer per particle at the end.
#pragma once

#include "common.cuh"
#include "density.cuh"
#include "packed.cuh"

#include <type_traits>

namespace pvsph {

constexpr int V3_WARPS = 4;
constexpr int V3_QP = 4;                  // pair slots per lane (8 queued hits)
constexpr int V3_NC = 7;                  // queued components: dx dy dz m (vj-vi)x y z

// Packed accumulators; D and curl use v_j - v_i (= -v_ij) so the cross products
// need no negation: Dn = -sum fac (v_ij . x_ij); R = P - N.
struct Acc2 {
    f2 rho, wc, srt, st, Dn, Px, Nx, Py, Ny, Pz, Nz;
};

__device__ __forceinline__ void acc2_zero(Acc2 &A)
{
    A.rho = A.wc = A.srt = A.st = A.Dn = A.Px = A.Nx = A.Py = A.Ny = A.Pz = A.Nz = 0ull;
}

// Two interactions from one pair slot.  mk = (1, 1) or (1, 0) when the odd half is
// empty (its stale components are finite: the queue is zeroed at start).
// M4 in branch-free form: w(x) = u^3 - v^3/2, w'(x) = 3 (v^2 - u^2),
// u = 1 - x, v = max(0, 1 - 2x)   (equal to the two-branch form of R1).
__device__ __forceinline__ void interact_pair(f2 Hinv2, f2 dx, f2 dy, f2 dz, f2 m, f2 nvx, f2 nvy, f2 nvz, f2 mk,
                                              Acc2 &A)
{
    f2 r2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    float r2a, r2b;
    upk(r2, r2a, r2b);
    // r^2 = 0 (coincident particles): rinv stays finite, x = 0 and w'(0) = 0 make every gradient term 0
    f2 rinv = pk(rsqrt_fast(fmaxf(r2a, 1e-30f)), rsqrt_fast(fmaxf(r2b, 1e-30f)));
    f2 x = mul2(mul2(r2, rinv), Hinv2);
    f2 u = sub2(bc2(1.0f), x);
    f2 v = fma2(bc2(-2.0f), x, bc2(1.0f));
    float va, vb, xa, xb, ua, ub;
    upk(v, va, vb);
    upk(x, xa, xb);
    upk(u, ua, ub);
    v = pk(fmaxf(va, 0.0f), fmaxf(vb, 0.0f));
    const f2 mn = pk(fminf(xa, ua), fminf(xb, ub));   // u - v without cancellation: min(x, u)
    f2 uu = mul2(u, u), vv = mul2(v, v);
    f2 w = mul2(fma2(uu, u, mul2(bc2(-0.5f), mul2(vv, v))), mk);
    // w' = 3 (v^2 - u^2) = -3 (u - v)(u + v); the difference of squares would lose all
    // precision for x -> 0 (w' ~ -6x while v^2, u^2 ~ 1)
    f2 dw = mul2(mul2(bc2(-3.0f), mk), mul2(mn, add2(u, v)));
    m = mul2(m, mk);
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

__device__ __forceinline__ int image_code(const int sh[3])
{
    int c = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) c |= (sh[a] > 0 ? 1 : (sh[a] < 0 ? 2 : 0)) << (2 * a);
    return c;
}

__device__ __forceinline__ int kind_of_dir(int d)
{
    // faces (0,0,1) (0,1,0) (1,0,0); corners (1,-1,-1) (1,-1,1) (1,1,-1) (1,1,1); the rest edges
    return (d == 0 || d == 2 || d == 8) ? 1 : ((d == 4 || d == 6 || d == 10 || d == 12) ? 3 : 2);
}

// ---- traversal order: owned rows (ix, iy) in ROW_TILE x ROW_TILE tiles -----------
constexpr int ROW_TILE = 4;

__host__ __device__ __forceinline__ int row_tiles_y(const DevGrid &g) { return (g.ny + ROW_TILE - 1) / ROW_TILE; }

__host__ __device__ __forceinline__ long long row_nkeys(const DevGrid &g)
{
    const int nxo = g.x_hi - g.x_lo;
    return (long long)((nxo + ROW_TILE - 1) / ROW_TILE) * row_tiles_y(g) * ROW_TILE * ROW_TILE;
}

// key -> owned row (ix relative to x_lo, iy); may fall outside the grid (ragged tiles)
__device__ __forceinline__ void row_of_key(const DevGrid &g, int key, int &ix, int &iy)
{
    const int tile = key / (ROW_TILE * ROW_TILE), wi = key % (ROW_TILE * ROW_TILE);
    const int nty = row_tiles_y(g);
    ix = (tile / nty) * ROW_TILE + wi / ROW_TILE;
    iy = (tile % nty) * ROW_TILE + wi % ROW_TILE;
}

// chunks[key] = number of 32-slot chunks of the row (0 outside the grid)
__global__ void k_row_chunks(DevGrid g, const int *__restrict__ cell_start, int *__restrict__ chunks, int nkeys)
{
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nkeys; k += gridDim.x * blockDim.x) {
        int ix, iy;
        row_of_key(g, k, ix, iy);
        int nch = 0;
        if (ix < g.x_hi - g.x_lo && iy < g.ny) {
            const long long first = ((long long)(ix + g.ghost_x) * g.ny + iy) * g.nz;
            nch = (cell_start[first + g.nz] - cell_start[first] + 31) >> 5;
        }
        chunks[k] = nch;
    }
}

template <bool COUNT>
__global__ void __launch_bounds__(V3_WARPS * 32, 6) k_density_all_v3(DevGrid g, DevCells c, DevOut o, sph_stats *st,
                                                                       const int *row_prefix, int nkeys)
{
    __shared__ float2 qp[V3_WARPS][V3_QP][V3_NC][32];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const long long plane = (long long)g.ny * g.nz;
    // work unit of this warp: chunk w of the owned rows (ix, iy) taken in ROW_TILE x ROW_TILE
    // tiles (k_row_chunks), so that concurrently running warps share their neighbour
    // lists in L2; 32 consecutive slots of one row, lane = particle
    const int w = (int)((long long)blockIdx.x * V3_WARPS + wl);
    if (w >= row_prefix[nkeys]) return;                // whole warp idle (warp-uniform)
    int klo = 0, khi = nkeys;                          // row_prefix[klo] <= w < row_prefix[khi]
    while (khi - klo > 1) {
        const int mid = (klo + khi) >> 1;
        if (row_prefix[mid] <= w) klo = mid; else khi = mid;
    }
    int rix, riy;
    row_of_key(g, klo, rix, riy);
    const long long first_cell = ((long long)(rix + g.ghost_x) * g.ny + riy) * g.nz;
    const int slot_lo = c.cell_start[first_cell];
    const int slot_hi = c.cell_start[first_cell + g.nz];
    const int i = slot_lo + 32 * (w - row_prefix[klo]) + lane;
    const bool active = i < slot_hi;

#pragma unroll
    for (int s = 0; s < V3_QP; ++s)
#pragma unroll
        for (int cc = 0; cc < V3_NC; ++cc) qp[wl][s][cc][lane] = make_float2(0.0f, 0.0f);

    unsigned cand[4] = {0, 0, 0, 0}, hits[4] = {0, 0, 0, 0};
    HomeCell hc;
    IPart p;
    int home = 0;
    if (active) {
        home = c.slot_cell[i];
        hc = home_cell(g, home);
        p = load_i(g, c, i, hc.corner);
    } else {
        p.x = p.y = p.z = p.vx = p.vy = p.vz = p.m = p.h = 0.0f;
        p.H2 = -1.0f;
        p.Hinv = p.Hd = 0.0f;
        p.u0 = p.u1 = p.u2 = 0.0;
        p.slot = -1;
        hc.ixl = hc.iy = hc.iz = hc.ixg = 0;
    }
    const int isafe = active ? i : slot_lo;                            // a valid slot for dummy loads
    const f2 Hinv2 = bc2(p.Hinv);

    Acc2 A;
    acc2_zero(A);
    int nngb = 0;
    unsigned head = 0, tail = 0;                       // hit counters; head stays even
    float2 (*Q)[V3_NC][32] = qp[wl];

    // pop one pair slot per lane that holds a full pair (or, when final, any hit)
    auto drain = [&](bool final) {
        const unsigned n = tail - head;
        if (n >= 2 || (final && n == 1)) {
            const int s = (head >> 1) & (V3_QP - 1);
            const f2 mk = pk(1.0f, n >= 2 ? 1.0f : 0.0f);
            interact_pair(Hinv2, as_f2(Q[s][0][lane]), as_f2(Q[s][1][lane]), as_f2(Q[s][2][lane]),
                          as_f2(Q[s][3][lane]), as_f2(Q[s][4][lane]), as_f2(Q[s][5][lane]), as_f2(Q[s][6][lane]),
                          mk, A);
            head += n >= 2 ? 2u : 1u;
        }
    };

    // queue hit number `tail` in half (tail & 1) of its pair slot
    auto push = [&](float ddx, float ddy, float ddz, int j, int kd) {
        const float4 vj = c.vm[j];
        float *slot = &Q[(tail >> 1) & (V3_QP - 1)][0][lane].x + (tail & 1);
        slot[0 * 64] = ddx;
        slot[1 * 64] = ddy;
        slot[2 * 64] = ddz;
        slot[3 * 64] = vj.w;
        slot[4 * 64] = vj.x - p.vx;
        slot[5 * 64] = vj.y - p.vy;
        slot[6 * 64] = vj.z - p.vz;
        ++tail;
        ++nngb;
        if (COUNT) ++hits[kd];
    };

    for (int a = 0; a < 14; ++a) {
        // lane's two windows for this pass: a = 0 the self cell; a = 1 + d the +d, -d neighbours
        const int d = a == 0 ? 0 : a - 1;
        const float4 *L = reinterpret_cast<const float4 *>(c.pv) + (long long)d * c.cap;
        const int kind = a == 0 ? 0 : kind_of_dir(d);
        int qb0 = 0, len0 = 0, qb1 = 0, len1 = 0, code0 = 0, code1 = 0;
        if (active) {
            if (a == 0) {
                qb0 = c.cell_start[home];
                len0 = c.cell_start[home + 1] - qb0;
            } else {
                const int a0 = dir_component(d, 0), a1 = dir_component(d, 1), a2 = dir_component(d, 2);
                float ax, ay, az;
                dir_unit(d, ax, ay, az);
                // separation along the pair axis of x_j - x_i from exact differences;
                // sorted lists make it monotone in q, so the window is found by bisection
                auto sep_of = [&](int q, int code) {
                    const float4 e = L[q];
                    float xi = p.x, yi = p.y, zi = p.z, xj = e.x, yj = e.y, zj = e.z;
                    if (code & 1) xi -= g.boxf[0];
                    if (code & 2) xj -= g.boxf[0];
                    if (code & 4) yi -= g.boxf[1];
                    if (code & 8) yj -= g.boxf[1];
                    if (code & 16) zi -= g.boxf[2];
                    if (code & 32) zj -= g.boxf[2];
                    return fmaf(xj - xi, ax, fmaf(yj - yi, ay, (zj - zi) * az));
                };
                int cj, sh[3];
                if (neighbour(g, hc, a0, a1, a2, cj, sh)) {        // +d: prefix {sep < H + delta}
                    code0 = image_code(sh);
                    int lo = c.cell_start[cj], hi = c.cell_start[cj + 1];
                    qb0 = lo;
                    while (lo < hi) {
                        int mid = (lo + hi) >> 1;
                        if (sep_of(mid, code0) < p.Hd) lo = mid + 1; else hi = mid;
                    }
                    len0 = lo - qb0;
                }
                if (neighbour(g, hc, -a0, -a1, -a2, cj, sh)) {     // -d: suffix {-sep < H + delta}
                    code1 = image_code(sh);
                    int lo = c.cell_start[cj], hi = c.cell_start[cj + 1];
                    const int end = hi;
                    while (lo < hi) {
                        int mid = (lo + hi) >> 1;
                        if (-sep_of(mid, code1) < p.Hd) hi = mid; else lo = mid + 1;
                    }
                    qb1 = lo;
                    len1 = end - lo;
                }
            }
        }
        const int total = len0 + len1;
        const int trip = __reduce_max_sync(0xffffffffu, total);
        // warp-uniform: periodic-image arithmetic only in warps that need it
        const bool any_image = __any_sync(0xffffffffu, (code0 | code1) != 0);
        const bool selfpass = a == 0;
        // Two candidates per iteration: both loads issued first, the pair tested in f32x2.
        // slot of candidate t of the lane's concatenated window (i itself past the end: no load)
        // Candidates t, t+1 of the lane's concatenated window; two independent loads in
        // flight per iteration.  IMAGE (warp-uniform) selects the periodic-image variant.
        const float4 *const Lp = L;
        const float4 *const Ldummy = c.xyzh + isafe;      // valid address past the end
        auto sweep = [&](auto image_tag) {
            constexpr bool IMAGE = decltype(image_tag)::value;
            for (int t = 0; t < trip; t += 2) {
                const bool ok0 = t < total, ok1 = t + 1 < total;
                const bool f0 = t < len0, f1 = t + 1 < len0;
                const float4 ea = *(ok0 ? Lp + (f0 ? qb0 + t : qb1 + (t - len0)) : Ldummy);
                const float4 eb = *(ok1 ? Lp + (f1 ? qb0 + t + 1 : qb1 + (t + 1 - len0)) : Ldummy);
                float xia = p.x, yia = p.y, zia = p.z, xja = ea.x, yja = ea.y, zja = ea.z;
                float xib = p.x, yib = p.y, zib = p.z, xjb = eb.x, yjb = eb.y, zjb = eb.z;
                if constexpr (IMAGE) {                     // periodic image: exact differences (R4)
                    const int ca = f0 ? code0 : code1, cb = f1 ? code0 : code1;
                    if (ca & 1) xia -= g.boxf[0];
                    if (ca & 2) xja -= g.boxf[0];
                    if (ca & 4) yia -= g.boxf[1];
                    if (ca & 8) yja -= g.boxf[1];
                    if (ca & 16) zia -= g.boxf[2];
                    if (ca & 32) zja -= g.boxf[2];
                    if (cb & 1) xib -= g.boxf[0];
                    if (cb & 2) xjb -= g.boxf[0];
                    if (cb & 4) yib -= g.boxf[1];
                    if (cb & 8) yjb -= g.boxf[1];
                    if (cb & 16) zib -= g.boxf[2];
                    if (cb & 32) zjb -= g.boxf[2];
                }
                const float dxa = xia - xja, dya = yia - yja, dza = zia - zja;
                const float dxb = xib - xjb, dyb = yib - yjb, dzb = zib - zjb;
                const float r2a = fmaf(dxa, dxa, fmaf(dya, dya, dza * dza));
                const float r2b = fmaf(dxb, dxb, fmaf(dyb, dyb, dzb * dzb));
                const int j0 = __float_as_int(ea.w), j1 = __float_as_int(eb.w);
                const bool ca_ok = ok0 && (!selfpass || j0 != i), cb_ok = ok1 && (!selfpass || j1 != i);
                if (COUNT) cand[kind] += (unsigned)ca_ok + (unsigned)cb_ok;
                if (ca_ok && r2a < p.H2) push(dxa, dya, dza, j0, kind);
                if (cb_ok && r2b < p.H2) push(dxb, dyb, dzb, j1, kind);
                // two pushes per iteration: drain before a queue could overflow
                const unsigned n = tail - head;
                if (__popc(__ballot_sync(0xffffffffu, n >= 2)) >= 24 ||
                    __any_sync(0xffffffffu, n >= 2 * V3_QP - 2))
                    drain(false);
            }
        };
        if (any_image) sweep(std::true_type{}); else sweep(std::false_type{});
    }
    while (__any_sync(0xffffffffu, tail != head)) drain(true);

    if (active) {
        // finalise (self term w(0) = 1/2, t(0) = 3/2), as finalise() in density.cuh
        float Hinv = p.Hinv;
        float K3 = (16.0f / kPi) * Hinv * Hinv * Hinv;
        float rho = K3 * fmaf(0.5f, p.m, sum2(A.rho));
        float wc = K3 * (0.5f + sum2(A.wc));
        float dh = -K3 * g.gamma * Hinv;
        float rho_dh = dh * fmaf(1.5f, p.m, sum2(A.srt));
        float wc_dh = dh * (1.5f + sum2(A.st));
        float gf = K3 * Hinv;
        float rinv = 1.0f / rho;
        int out = c.perm[i];
        if (out < o.n_out) {
            o.rho[out] = rho;
            o.wcount[out] = wc;
            o.rho_dh[out] = rho_dh;
            o.wcount_dh[out] = wc_dh;
            o.div_v[out] = gf * sum2(A.Dn) * rinv;
            o.curl_v[out] = gf * (sum2(A.Px) - sum2(A.Nx)) * rinv;
            o.curl_v[o.n_out + out] = gf * (sum2(A.Py) - sum2(A.Ny)) * rinv;
            o.curl_v[2 * o.n_out + out] = gf * (sum2(A.Pz) - sum2(A.Nz)) * rinv;
            o.nngb[out] = nngb;
        }
    }
    flush_stats<COUNT>(st, cand, hits);
}

}  // namespace pvsph
