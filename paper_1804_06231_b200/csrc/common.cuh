// common.cuh -- device-side definitions shared by the kernels of libpvsph.so.
// (CUDA path only; shares nothing with oracle/.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sph.h"

namespace pvsph {

// Status-word bits (mapped to SPH_E* codes by sph_status).
enum : unsigned {
    ST_EINVAL = 1u << 0,
    ST_EH_RANGE = 1u << 1,
    ST_ECAPACITY = 1u << 2,
    ST_EDOMAIN = 1u << 3,
};

// Flattened, by-value view of sph_grid plus derived constants.
struct DevGrid {
    int nc[3];
    int x_lo, x_hi, ghost_x;
    int nxl;             // local x planes
    int ny, nz;
    long long ncell;     // local cells
    long long n_owned_cells;
    double box[3];
    double cl[3];        // cell edges
    float boxf[3];
    float gamma;
    float h_home_min, h_home_max;   // level passes: home iff h_home_min < h <= h_home_max (max 0: all)
    float delta;         // window margin SPH_DELTA_FRAC * min(cl) + 4 skin (engines without per-cell max_dx)
    float delta0;        // the fp32 part alone, SPH_DELTA_FRAC * min(cl): k_density_v5 adds 2 max_dx(cj)
    float skin;          // list reuse: largest displacement since the build (sph_grid.skin)
    float q[SPH_NDIR];   // Q_d = sum_a |d_a| C_a / |d|: projection of the cell offset on axis d
};

struct DevCells {
    long long cap;
    const int *cell_start;
    const float4 *xyzh;
    const float4 *vm;
    const int *perm;
    const float *cell_hmax;
    const uint16_t *ord;    // sorted lists (include/sph.h), [SPH_NDIR][cap]
    const int *slot_cell;
    const int *cell_nhome;
    const float *cell_dx;   // per-cell max_dx since the build (sph_drift; workspace), or null
};

// Level passes: is a particle of smoothing length h a HOME particle of
// grid g (outputs computed here) or a neighbour source only?
__host__ __device__ __forceinline__ bool is_home(float h_home_min, float h_home_max, float h)
{
    return !(h_home_max > 0.0f) || (h > h_home_min && h <= h_home_max);
}

struct DevOut {
    long long n_out;
    float *rho, *rho_dh, *wcount, *wcount_dh, *div_v, *curl_v;
    int *nngb;
};

// The 13 directions as a constant table {a0, a1, a2, kind} (kind: 1 face, 2 edge, 3 corner),
// the values of dir_component below; one LDC instead of the index arithmetic in loops that
// run over d at run time (k_density_v5).
__constant__ int4 c_dirs[13] = {{0, 0, 1, 1},  {0, 1, -1, 2}, {0, 1, 0, 1},  {0, 1, 1, 2},  {1, -1, -1, 3},
                                {1, -1, 0, 2}, {1, -1, 1, 3}, {1, 0, -1, 2}, {1, 0, 0, 1},  {1, 0, 1, 2},
                                {1, 1, -1, 3}, {1, 1, 0, 2},  {1, 1, 1, 3}};

// The list along which k_density_dense orders a dense home cell's particles and sweeps the
// cell itself (direction 0 = (0,0,1)); level passes sort it for every cell with home particles.
constexpr int DENSE_SELF_DIR = 0;

// The 13 canonical sort directions: first nonzero component > 0,
// lexicographic order.  d = dir_index(canonical offset).
__host__ __device__ __forceinline__ int dir_component(int d, int a)
{
    // (0,0,1) (0,1,-1) (0,1,0) (0,1,1) then (1,b,c) for b,c in -1..1
    if (d == 0) return a == 2 ? 1 : 0;
    if (d <= 3) return a == 0 ? 0 : (a == 1 ? 1 : d - 2);
    int e = d - 4;
    return a == 0 ? 1 : (a == 1 ? e / 3 - 1 : e % 3 - 1);
}

__host__ __device__ __forceinline__ int dir_index(int a, int b, int c)
{
    return a == 1 ? 4 + (b + 1) * 3 + (c + 1) : (b == 1 ? 2 + c : 0);
}

// Canonicalise a neighbour offset o: returns d and sets s = +1 if o = +d_vec,
// -1 if o = -d_vec.
__host__ __device__ __forceinline__ int canon_dir(int ox, int oy, int oz, int &s)
{
    int first = ox != 0 ? ox : (oy != 0 ? oy : oz);
    s = first > 0 ? 1 : -1;
    return dir_index(ox * s, oy * s, oz * s);
}

// Cell-local projection key of local coordinates u (fp64) on unit axis d,
// rounded once to fp32.
__device__ __forceinline__ float pv_key(double ux, double uy, double uz, int d)
{
    int a = dir_component(d, 0), b = dir_component(d, 1), c = dir_component(d, 2);
    int kind = (a != 0) + (b != 0) + (c != 0);
    double inv = kind == 1 ? 1.0 : (kind == 2 ? 0.70710678118654752440 : 0.57735026918962576451);
    double s = (double)a * ux + (double)b * uy + (double)c * uz;
    return (float)(s * inv);
}

__device__ __forceinline__ int wrap_i(int a, int n)
{
    return a < 0 ? a + n : (a >= n ? a - n : a);
}

__device__ __forceinline__ void set_status(unsigned *status, unsigned bit)
{
    atomicOr(status, bit);
}

// Orderable 32-bit image of a float (ascending uint order == ascending float order).
__device__ __forceinline__ unsigned float_order(float f)
{
    unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

constexpr float kPi = 3.14159265358979323846f;

}  // namespace pvsph
