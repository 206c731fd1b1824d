// density_v2.cuh -- the production sph_density_all engine.
//
// Same method and per-particle arithmetic as the reference engine (density.cuh),
// mapped differently onto the SIMT machine:
//
//  * a warp owns 32 consecutive slots of the cell-sorted arrays (lane = i), so
//    lanes are filled across cell boundaries instead of idling in 21-particle
//    cells;
//  * the self cell and the 26 neighbour cells are swept warp-synchronously in a
//    fixed order; within a cell every lane walks its own pseudo-Verlet window
//    of the pair's sorted list, so lanes of one home cell read the
//    same list entries at the same time (broadcast-friendly loads);
//  * the candidate test only computes r^2 ("the most time-consuming part
//    of the neighbour search"); an in-range pair is compacted into the lane's
//    shared-memory hit queue (x_ij, m_j, v_j - v_i) instead of running the
//    interaction under divergence -- the GPU form of the paper's left-packed
//    masks ("if (ANY(mask))");
//  * interactions drain the queues two hits per lane at a time with packed
//    f32x2 arithmetic (FFMA2/FADD2/FMUL2), all lanes busy, accumulating in
//    registers; one writer per particle.
//
// Per particle the hits are accumulated in queue (= sweep) order, alternating
// between the two halves of the packed accumulators, so results do not depend
// on which other particles share the warp: deterministic, and identical on any
// number of GPUs.
#pragma once

#include "common.cuh"
#include "density.cuh"

namespace pvsph {

typedef unsigned long long f2;   // two fp32 lanes of one 64-bit register pair

__device__ __forceinline__ f2 pk(float a, float b)
{
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk(f2 v, float &a, float &b)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b)
{
    f2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b)
{
    f2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b)
{
    f2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c)
{
    f2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ float sum2(f2 v)
{
    float a, b;
    upk(v, a, b);
    return a + b;
}

constexpr int V2_WARPS = 4;
constexpr int V2_Q = 8;   // hit-queue entries per lane (power of two)

// Packed accumulators.  D and the curl use v_j - v_i (= -v_ij), so that the
// cross products need no negation: D' = -sum fac (v_ij . x_ij),
// R = P - N with P_x = sum f_z dy, N_x = sum f_y dz (f = fac (v_j - v_i)), etc.
struct Acc2 {
    f2 rho, wc, srt, st, Dn, Px, Nx, Py, Ny, Pz, Nz;
};

__device__ __forceinline__ void acc2_zero(Acc2 &A)
{
    A.rho = A.wc = A.srt = A.st = A.Dn = A.Px = A.Nx = A.Py = A.Ny = A.Pz = A.Nz = 0ull;
}

// Two queued hits (a = x_ij, m_j; b = v_j - v_i).  v0/v1 mark valid entries;
// invalid ones are zeroed so they contribute nothing (and no NaN).
__device__ __forceinline__ void interact2(float Hinv, float4 a0, float4 b0, float4 a1, float4 b1, bool v0, bool v1,
                                          Acc2 &A)
{
    const float z = 0.0f;
    if (!v0) { a0 = make_float4(z, z, z, z); b0 = a0; }
    if (!v1) { a1 = make_float4(z, z, z, z); b1 = a1; }
    f2 dx = pk(a0.x, a1.x), dy = pk(a0.y, a1.y), dz = pk(a0.z, a1.z), m = pk(a0.w, a1.w);
    f2 r2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    float r2a, r2b;
    upk(r2, r2a, r2b);
    f2 rinv = pk(r2a > 0.0f ? rsqrtf(r2a) : 0.0f, r2b > 0.0f ? rsqrtf(r2b) : 0.0f);
    f2 x = mul2(mul2(r2, rinv), pk(Hinv, Hinv));
    // both spline branches (w(x), w'(x)), then select per half
    f2 xx = mul2(x, x);
    f2 w_in = fma2(fma2(pk(3.0f, 3.0f), x, pk(-3.0f, -3.0f)), xx, pk(0.5f, 0.5f));
    f2 dw_in = mul2(x, fma2(pk(9.0f, 9.0f), x, pk(-6.0f, -6.0f)));
    f2 u = sub2(pk(1.0f, 1.0f), x);
    f2 uu = mul2(u, u);
    f2 w_out = mul2(uu, u);
    f2 dw_out = mul2(pk(-3.0f, -3.0f), uu);
    float xa, xb, wia, wib, woa, wob, dia, dib, doa, dob;
    upk(x, xa, xb);
    upk(w_in, wia, wib);
    upk(w_out, woa, wob);
    upk(dw_in, dia, dib);
    upk(dw_out, doa, dob);
    f2 w = pk(v0 ? (xa < 0.5f ? wia : woa) : 0.0f, v1 ? (xb < 0.5f ? wib : wob) : 0.0f);
    f2 dw = pk(xa < 0.5f ? dia : doa, xb < 0.5f ? dib : dob);
    A.rho = fma2(m, w, A.rho);
    A.wc = add2(A.wc, w);
    f2 t = fma2(x, dw, mul2(pk(3.0f, 3.0f), w));
    A.srt = fma2(m, t, A.srt);
    A.st = add2(A.st, t);
    f2 nvx = pk(b0.x, b1.x), nvy = pk(b0.y, b1.y), nvz = pk(b0.z, b1.z);
    f2 nvdx = fma2(nvx, dx, fma2(nvy, dy, mul2(nvz, dz)));
    f2 fac = mul2(mul2(m, dw), rinv);
    A.Dn = fma2(fac, nvdx, A.Dn);
    f2 fx = mul2(fac, nvx), fy = mul2(fac, nvy), fz = mul2(fac, nvz);
    A.Px = fma2(fz, dy, A.Px);
    A.Nx = fma2(fy, dz, A.Nx);
    A.Py = fma2(fx, dz, A.Py);
    A.Ny = fma2(fz, dx, A.Ny);
    A.Pz = fma2(fy, dx, A.Pz);
    A.Nz = fma2(fx, dy, A.Nz);
}

template <bool COUNT>
__global__ void __launch_bounds__(V2_WARPS * 32, 4) k_density_all_v2(DevGrid g, DevCells c, DevOut o, sph_stats *st)
{
    __shared__ float4 qa[V2_WARPS][V2_Q][32];
    __shared__ float4 qb[V2_WARPS][V2_Q][32];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const long long plane = (long long)g.ny * g.nz;
    const int slot_lo = c.cell_start[g.ghost_x ? plane : 0];
    const int slot_hi = c.cell_start[g.ghost_x ? (g.nxl - 1) * plane : g.ncell];
    const long long base = (long long)slot_lo + ((long long)blockIdx.x * V2_WARPS + wl) * 32;
    if (base >= slot_hi) return;                       // whole warp idle (warp-uniform)
    const int i = (int)base + lane;
    const bool active = i < slot_hi;

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
    Acc2 A;
    acc2_zero(A);
    int nngb = 0;
    unsigned head = 0, tail = 0;
    float4 (*QA)[32] = qa[wl];
    float4 (*QB)[32] = qb[wl];

    auto drain_step = [&]() {
        unsigned n = tail - head;
        bool v0 = n >= 1, v1 = n >= 2;
        unsigned h0 = head & (V2_Q - 1), h1 = (head + 1) & (V2_Q - 1);
        float4 a0 = QA[h0][lane], b0 = QB[h0][lane], a1 = QA[h1][lane], b1 = QB[h1][lane];
        interact2(p.Hinv, a0, b0, a1, b1, v0, v1, A);
        head += (v1 ? 2u : (v0 ? 1u : 0u));
    };

    for (int k = 0; k < 27; ++k) {
        // offset order: self cell first, then (ox, oy, oz) lexicographic
        int ox, oy, oz;
        if (k == 0) {
            ox = oy = oz = 0;
        } else {
            int e = k - 1 + (k - 1 >= 13 ? 1 : 0);   // skip (0,0,0) at lexicographic index 13
            ox = e / 9 - 1;
            oy = (e / 3) % 3 - 1;
            oz = e % 3 - 1;
        }
        const int kind = kind_of(ox, oy, oz);
        // this lane's list segment and window
        const sph_pv_entry *L = c.pv;
        int qbeg = 0, qend = 0, step = 1;
        float lim = 0.0f;
        float xi = p.x, yi = p.y, zi = p.z, sjx = 0.0f, sjy = 0.0f, sjz = 0.0f;
        bool more = false;
        if (active) {
            if (kind == 0) {
                qbeg = c.cell_start[home];
                qend = c.cell_start[home + 1];
                more = qbeg < qend;
                lim = __int_as_float(0x7f800000);   // +inf: no window in the self cell
            } else {
                int cj, sh[3];
                if (neighbour(g, hc, ox, oy, oz, cj, sh)) {
                    int s;
                    int d = canon_dir(ox, oy, oz, s);
                    float key_i = pv_key(p.u0, p.u1, p.u2, d);
                    float B = p.Hd - g.q[d];
                    L = c.pv + (long long)d * c.cap;
                    int s0 = c.cell_start[cj], s1 = c.cell_start[cj + 1];
                    if (s > 0) {
                        qbeg = s0; qend = s1; step = 1; lim = key_i + B;
                    } else {
                        qbeg = s1 - 1; qend = s0 - 1; step = -1; lim = -(key_i - B);
                    }
                    more = qbeg != qend;
                    xi = sh[0] > 0 ? p.x - g.boxf[0] : p.x;
                    yi = sh[1] > 0 ? p.y - g.boxf[1] : p.y;
                    zi = sh[2] > 0 ? p.z - g.boxf[2] : p.z;
                    sjx = sh[0] < 0 ? g.boxf[0] : 0.0f;
                    sjy = sh[1] < 0 ? g.boxf[1] : 0.0f;
                    sjz = sh[2] < 0 ? g.boxf[2] : 0.0f;
                }
            }
        }
        const float sgn = step > 0 ? 1.0f : -1.0f;
        int q = qbeg;
        while (__any_sync(0xffffffffu, more)) {
            if (more) {
                sph_pv_entry e = L[q];
                q += step;
                if (!(sgn * e.key < lim)) {
                    more = false;                      // sorted early exit (Code 2)
                } else {
                    if (q == qend) more = false;
                    if (e.j != i) {
                        float4 pj = c.xyzh[e.j];
                        float dx = xi - (pj.x - sjx), dy = yi - (pj.y - sjy), dz = zi - (pj.z - sjz);
                        float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                        if (COUNT) ++cand[kind];
                        if (r2 < p.H2) {
                            float4 vj = c.vm[e.j];
                            unsigned t = tail & (V2_Q - 1);
                            QA[t][lane] = make_float4(dx, dy, dz, vj.w);
                            QB[t][lane] = make_float4(vj.x - p.vx, vj.y - p.vy, vj.z - p.vz, 0.0f);
                            ++tail;
                            ++nngb;
                            if (COUNT) ++hits[kind];
                        }
                    }
                }
            }
            // drain when some queue is about to overflow, or every lane has two hits ready
            unsigned n = tail - head;
            if (__any_sync(0xffffffffu, n >= V2_Q - 1) || __all_sync(0xffffffffu, n >= 2 || !active)) drain_step();
        }
    }
    while (__any_sync(0xffffffffu, tail != head)) drain_step();

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
