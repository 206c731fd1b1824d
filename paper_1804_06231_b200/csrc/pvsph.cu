// pvsph.cu -- C ABI of libpvsph.so (include/sph.h): argument checking,
// workspace layout and kernel launches.  One translation unit (the kernels
// live in the .cuh files) compiled for sm_100a only.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/sph_calib.h"
#include "build.cuh"
#include "calib.cuh"
#include "common.cuh"
#include "density.cuh"
#include "density_v4.cuh"
#include "density_v5.cuh"
#include "density_pair.cuh"
#include "density_dense.cuh"
#include "sort.cuh"

using namespace pvsph;

namespace {

thread_local char g_cuda_msg[256] = "CUDA error";

int cuda_fail(cudaError_t e)
{
    std::snprintf(g_cuda_msg, sizeof(g_cuda_msg), "CUDA error %d: %s", (int)e, cudaGetErrorString(e));
    return SPH_ECUDA;
}

// Per-device launch attributes (dynamic shared memory opt-ins, occupancy, SM count), set
// once per device on first use: cudaFuncSetAttribute applies to the current device only.
struct DevAttrs {
    int sms = 0, v4_blocks_per_sm = 1, v5_blocks_per_sm = 1;
};
constexpr int kMaxDevices = 64;
DevAttrs g_dev_attrs[kMaxDevices];
std::once_flag g_dev_once[kMaxDevices];

const DevAttrs &dev_attrs(int dev)
{
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    std::call_once(g_dev_once[dev], [dev]() {
        DevAttrs &a = g_dev_attrs[dev];
        cudaDeviceGetAttribute(&a.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_density_v4<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)V4_SMEM);
        cudaFuncSetAttribute(k_density_v4<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)V4_SMEM);
        cudaFuncSetAttribute(k_density_v5<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)V5_SMEM);
        cudaFuncSetAttribute(k_density_v5<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)V5_SMEM);
        cudaFuncSetAttribute(k_density_dense<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DENSE_SMEM);
        cudaFuncSetAttribute(k_density_dense<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DENSE_SMEM);
        cudaFuncSetAttribute(k_stable_radix<STABLE_BT_MAX, STABLE_BT_T, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, stable_radix_smem(STABLE_BT_MAX, STABLE_BT_T));
        cudaFuncSetAttribute(k_sort_radix<65535, SORT_GIANT_T, false, true, 2>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, radix_smem_global(SORT_GIANT_T));
        cudaFuncSetAttribute(k_sort_radix<SORT_HUGE_MAX, SORT_HUGE_T, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, radix_smem(SORT_HUGE_MAX, SORT_HUGE_T));
        cudaFuncSetAttribute(k_density_pair_staged<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PAIR_SMEM);
        cudaFuncSetAttribute(k_density_pair_staged<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PAIR_SMEM);
        cudaFuncSetAttribute(k_density_pair_sym<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SYM_SMEM);
        cudaFuncSetAttribute(k_density_pair_sym<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SYM_SMEM);
        cudaFuncSetAttribute(k_density_pair_sym<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SYM_SMEM);
        cudaFuncSetAttribute(k_density_pair_sym<true, true, SYMW_MAXN, 1, SYMW_WARPS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SYMW_SMEM);
        cudaFuncSetAttribute(k_density_pair_sym<false, true, SYMW_MAXN, 1, SYMW_WARPS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SYMW_SMEM);
        cudaFuncSetAttribute(k_density_pair_sym<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SYM_SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a.v4_blocks_per_sm, k_density_v4<false>, V4_TP, V4_SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a.v5_blocks_per_sm, k_density_v5<false>, V5_TP, V5_SMEM);
        if (a.v4_blocks_per_sm < 1) a.v4_blocks_per_sm = 1;
        if (a.v5_blocks_per_sm < 1) a.v5_blocks_per_sm = 1;
        if (a.sms < 1) a.sms = 148;
        cudaGetLastError();
    });
    return g_dev_attrs[dev];
}

// the attributes of the current device (set on first use)
int ensure_attrs()
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e);
    dev_attrs(dev);
    return SPH_OK;
}

int check_launch()
{
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SPH_OK : cuda_fail(e);
}

int make_grid(const sph_grid *gr, DevGrid &g)
{
    if (!gr) return SPH_EINVAL;
    for (int k = 0; k < 3; ++k)
        if (gr->nc[k] < 3 || !(gr->box[k] > 0.0) || !std::isfinite(gr->box[k])) return SPH_EINVAL;
    if (gr->ghost_x != 0 && gr->ghost_x != 1) return SPH_EINVAL;
    if (gr->x_lo < 0 || gr->x_hi > gr->nc[0] || gr->x_lo >= gr->x_hi) return SPH_EINVAL;
    if (!gr->ghost_x && (gr->x_lo != 0 || gr->x_hi != gr->nc[0])) return SPH_EINVAL;
    if (gr->ghost_x && gr->nc[0] - (gr->x_hi - gr->x_lo) == 1) return SPH_EINVAL;  // ghost planes coincide
    if (!(gr->gamma > 0.0f) || !std::isfinite(gr->gamma)) return SPH_EINVAL;
    std::memset(&g, 0, sizeof(g));
    for (int k = 0; k < 3; ++k) {
        g.nc[k] = gr->nc[k];
        g.box[k] = gr->box[k];
        g.boxf[k] = (float)gr->box[k];
        g.cl[k] = gr->box[k] / gr->nc[k];
    }
    g.x_lo = gr->x_lo;
    g.x_hi = gr->x_hi;
    g.ghost_x = gr->ghost_x;
    g.nxl = (gr->x_hi - gr->x_lo) + 2 * gr->ghost_x;
    g.ny = gr->nc[1];
    g.nz = gr->nc[2];
    g.ncell = (long long)g.nxl * g.ny * g.nz;
    g.n_owned_cells = (long long)(gr->x_hi - gr->x_lo) * g.ny * g.nz;
    if (g.ncell >= (1LL << 31) - 1) return SPH_EINVAL;
    g.gamma = gr->gamma;
    if (gr->reserved != 0 || !(gr->skin >= 0.0f) || !std::isfinite(gr->skin)) return SPH_EINVAL;
    if (!(gr->h_home_max >= 0.0f) || !(gr->h_home_min >= 0.0f) || !std::isfinite(gr->h_home_max) ||
        (gr->h_home_max > 0.0f && !(gr->h_home_min < gr->h_home_max)))
        return SPH_EINVAL;
    g.h_home_min = gr->h_home_min;
    g.h_home_max = gr->h_home_max;
    double clmin = std::fmin(g.cl[0], std::fmin(g.cl[1], g.cl[2]));
    g.skin = gr->skin;
    // window margin: the fp32 margin of §4.2 plus 4 skin (stale sort order after drifts, §4.6)
    g.delta = (float)(SPH_DELTA_FRAC * clmin + 4.0 * (double)gr->skin);
    g.delta0 = (float)(SPH_DELTA_FRAC * clmin);
    if (gr->skin > 0.0f && !(2.0 * (double)gr->skin < clmin)) return SPH_EINVAL;
    for (int d = 0; d < SPH_NDIR; ++d) {
        int nz = 0;
        double q = 0.0;
        for (int a = 0; a < 3; ++a) {
            int c = dir_component(d, a);
            nz += c != 0;
            q += (c != 0 ? 1.0 : 0.0) * g.cl[a];
        }
        g.q[d] = (float)(q / std::sqrt((double)nz));
    }
    return SPH_OK;
}

bool cells_ok(const sph_cells *c)
{
    return c && c->cell_start && c->xyzh && c->vm && c->perm && c->cell_hmax && c->order && c->slot_cell && c->cell_nhome &&
           c->disp && c->cell_dx &&
           c->capacity >= 0 &&
           c->capacity < (1LL << 31) && ((uintptr_t)c->xyzh % 16 == 0) && ((uintptr_t)c->vm % 16 == 0) &&
           ((uintptr_t)c->order % 2 == 0);
}

DevCells dev_cells(const sph_cells *c)
{
    DevCells d;
    d.cap = c->capacity;
    d.cell_start = c->cell_start;
    d.xyzh = reinterpret_cast<const float4 *>(c->xyzh);
    d.vm = reinterpret_cast<const float4 *>(c->vm);
    d.perm = c->perm;
    d.cell_hmax = c->cell_hmax;
    d.ord = c->order;
    d.slot_cell = c->slot_cell;
    d.cell_nhome = c->cell_nhome;
    d.cell_dx = c->cell_dx;
    return d;
}

bool out_ok(const sph_out *o)
{
    return o && o->n_out >= 0 && o->rho && o->rho_dh && o->wcount && o->wcount_dh && o->div_v && o->curl_v &&
           o->nngb;
}

DevOut dev_out(const sph_out *o)
{
    DevOut d;
    d.n_out = o->n_out;
    d.rho = o->rho;
    d.rho_dh = o->rho_dh;
    d.wcount = o->wcount;
    d.wcount_dh = o->wcount_dh;
    d.div_v = o->div_v;
    d.curl_v = o->curl_v;
    d.nngb = o->nngb;
    return d;
}

// ---- workspace layout --------------------------------------------------------
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Ws {
    size_t status, cell_of, rank, rec, orec, count, tile_sum, big_count, big_items, huge_count,
        huge_items, mid_items, w256_items, rows, rows_sum, tiles, counter, gen, gtiles, gcount, row_home, total;
    long long tile_cap, huge_cap;
};

Ws ws_layout(const DevGrid &g, long long n)
{
    const long long ncell = g.ncell;
    Ws w;
    size_t o = 0;
    w.status = o;
    o = align_up(o + 4, 256);
    w.cell_of = o;
    o = align_up(o + 4 * (size_t)(n > 0 ? n : 1), 256);
    w.rank = o;
    o = align_up(o + 4 * (size_t)(n > 0 ? n : 1), 256);
    w.rec = o;
    o = align_up(o + sizeof(ParticleRec) * (size_t)(n > 0 ? n : 1), 256);
    w.orec = o;
    o = align_up(o + sizeof(OutRec) * (size_t)(n > 0 ? n : 1), 256);
    w.count = o;
    o = align_up(o + 4 * (size_t)(ncell + 1), 256);
    long long ntiles = (ncell + SCAN_TILE - 1) / SCAN_TILE;
    w.tile_sum = o;
    o = align_up(o + 4 * (size_t)(ntiles + 1), 256);
    w.big_count = o;
    o = align_up(o + 4, 256);
    w.big_items = o;                     // (cell, chunk) items: cells of > 32 particles, chunks of 256
    o = align_up(o + 8 * (size_t)(n / 32 + 64), 256);
    w.huge_count = o;                    // [medium, huge, mid (k_sort_mid), w256 (k_sort_warp256)]
    o = align_up(o + 16, 256);
    w.huge_items = o;                    // cells of > SORT_MED particles (medium from the front, huge from the back)
    w.huge_cap = n / SORT_MED + 64;
    o = align_up(o + 4 * (size_t)w.huge_cap, 256);
    w.mid_items = o;                     // cells of SORT_SMALL < n <= SORT_MED particles
    o = align_up(o + 4 * (size_t)(n / (SORT_SMALL + 1) + 64), 256);
    w.w256_items = o;                    // cells of SORT_MED < n <= SORT_W256 particles
    o = align_up(o + 4 * (size_t)(n / (SORT_MED + 1) + 64), 256);
    const long long nkeys = row_pairs(g).nkeys;
    w.rows = o;
    o = align_up(o + 4 * (size_t)(nkeys + 1), 256);
    w.rows_sum = o;
    o = align_up(o + 4 * (size_t)((nkeys + SCAN_TILE - 1) / SCAN_TILE + 1), 256);
    w.tile_cap = v4_tile_capacity(g, n);
    w.tiles = o;
    o = align_up(o + 16 * (size_t)w.tile_cap, 256);
    w.counter = o;
    o = align_up(o + 4, 256);
    w.gen = o;                           // sph_density_all call counter: tags the output records
    o = align_up(o + 4, 256);
    w.gtiles = o;                        // tiles k_v4_tiles could not stage (k_density_dense)
    o = align_up(o + 4 * (size_t)w.tile_cap, 256);
    w.gcount = o;                        // [listed, claimed]
    o = align_up(o + 8, 256);
    w.row_home = o;                      // per local (x, y) row: any home particle (build -> k_v4_tiles)
    o = align_up(o + 4 * (size_t)g.nxl * g.ny, 256);
    w.total = o;
    return w;
}

template <typename T>
T *at(void *ws, size_t off)
{
    return reinterpret_cast<T *>(static_cast<char *>(ws) + off);
}

int grid_blocks(long long work, int per_block, int cap)
{
    long long b = (work + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (int)b;
}

}  // namespace

extern "C" {

int sph_abi_version(void) { return SPH_ABI_VERSION; }

int64_t sph_ncell(const sph_grid *grid)
{
    DevGrid g;
    if (make_grid(grid, g) != SPH_OK) return -1;
    return g.ncell;
}

size_t sph_workspace_bytes(const sph_grid *grid, int64_t n_total)
{
    DevGrid g;
    if (make_grid(grid, g) != SPH_OK || n_total < 0) return 0;
    return ws_layout(g, n_total).total;
}

int sph_status_reset(void *ws, void *stream)
{
    if (!ws) return SPH_EINVAL;
    cudaError_t e = cudaMemsetAsync(ws, 0, 4, (cudaStream_t)stream);
    return e == cudaSuccess ? SPH_OK : cuda_fail(e);
}

}  // extern "C"

namespace {

// sph_build_cells; FUSE_SORT: the small cells' lists too (sph_build_sort_cells)
int build_impl(const sph_grid *grid, int64_t n_own, int64_t n_ghost, const float *xyzh_in, const float *vm_in,
               sph_cells *cells, void *ws, size_t ws_bytes, void *stream, bool fuse_sort)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (n_own < 0 || n_ghost < 0 || !cells_ok(cells) || !ws) return SPH_EINVAL;
    if (n_ghost > 0 && !g.ghost_x) return SPH_EINVAL;
    long long n = n_own + n_ghost;
    if (n > 0 && (!xyzh_in || !vm_in)) return SPH_EINVAL;
    if (((uintptr_t)xyzh_in % 16) || ((uintptr_t)vm_in % 16)) return SPH_EINVAL;
    if (n > cells->capacity) return SPH_ECAPACITY;
    Ws w = ws_layout(g, cells->capacity);
    if (ws_bytes < w.total) return SPH_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    if ((e = cudaMemsetAsync(at<unsigned>(ws, w.status), 0, 4, s)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMemsetAsync(at<int>(ws, w.count), 0, 4 * (size_t)g.ncell, s)) != cudaSuccess) return cuda_fail(e);
    unsigned *status = at<unsigned>(ws, w.status);
    int *cell_of = at<int>(ws, w.cell_of), *rank = at<int>(ws, w.rank), *count = at<int>(ws, w.count);
    int *tile_sum = at<int>(ws, w.tile_sum);
    const float4 *xin = reinterpret_cast<const float4 *>(xyzh_in);
    const float4 *vin = reinterpret_cast<const float4 *>(vm_in);
    if (n > 0) {
        k_bin<<<grid_blocks(n, 256, 148 * 32), 256, 0, s>>>(g, n_own, n, xin, vin, cell_of, rank, count,
                                                            status);
    }
    long long ntiles = (g.ncell + SCAN_TILE - 1) / SCAN_TILE;
    k_scan_tiles<<<(int)ntiles, SCAN_T, 0, s>>>(count, g.ncell, cells->cell_start, tile_sum, status);
    k_scan_sums<<<1, SCAN_T, 0, s>>>(tile_sum, ntiles, cells->cell_start, g.ncell);
    k_scan_add<<<(int)ntiles, SCAN_T, 0, s>>>(cells->cell_start, g.ncell, tile_sum);
    int *big_count = at<int>(ws, w.big_count);
    int2 *big_items = at<int2>(ws, w.big_items);
    if ((e = cudaMemsetAsync(big_count, 0, 4, s)) != cudaSuccess) return cuda_fail(e);
    if (n > 0) {
        ParticleRec *rec = at<ParticleRec>(ws, w.rec);
        k_scatter_rec<<<grid_blocks(n, 256, 148 * 32), 256, 0, s>>>(g, n, cell_of, rank, cells->cell_start, xin,
                                                                    vin, rec);
        float4 *xs = reinterpret_cast<float4 *>(cells->xyzh), *vs = reinterpret_cast<float4 *>(cells->vm);
        int *bt_items = at<int>(ws, w.huge_items), *bt_count = at<int>(ws, w.huge_count);
        int *row_home = at<int>(ws, w.row_home);
        if ((e = cudaMemsetAsync(bt_count, 0, 8, s)) != cudaSuccess) return cuda_fail(e);
        if ((e = cudaMemsetAsync(row_home, 0, 4 * (size_t)g.nxl * g.ny, s)) != cudaSuccess) return cuda_fail(e);
        // a fresh build: no displacement since it (list reuse, sph_drift)
        if ((e = cudaMemsetAsync(cells->disp, 0, 4 * (size_t)n, s)) != cudaSuccess) return cuda_fail(e);
        if ((e = cudaMemsetAsync(cells->cell_dx, 0, 4 * (size_t)g.ncell, s)) != cudaSuccess) return cuda_fail(e);
        if (fuse_sort)
            k_stable_small<true><<<grid_blocks(g.ncell, STABLE_WARPS, 148 * 64), STABLE_WARPS * 32, 0, s>>>(
                g.ncell, cells->cell_start, rec, xs, vs, cells->perm, cells->slot_cell, cells->cell_nhome,
                cells->cell_hmax, row_home, g.nz, big_items, big_count, bt_items, bt_count, (int)w.huge_cap, g,
                cells->order, cells->capacity);
        else
            k_stable_small<false><<<grid_blocks(g.ncell, STABLE_WARPS, 148 * 64), STABLE_WARPS * 32, 0, s>>>(
                g.ncell, cells->cell_start, rec, xs, vs, cells->perm, cells->slot_cell, cells->cell_nhome,
                cells->cell_hmax, row_home, g.nz, big_items, big_count, bt_items, bt_count, (int)w.huge_cap, g,
                cells->order, cells->capacity);
        if ((rc = ensure_attrs()) != SPH_OK) return rc;
        k_stable_radix<STABLE_MED_MAX, STABLE_MED_T, false>
            <<<148 * 8, STABLE_MED_T, stable_radix_smem(STABLE_MED_MAX, STABLE_MED_T), s>>>(
                cells->cell_start, rec, xs, vs, cells->perm, bt_items, bt_count, (int)w.huge_cap);
        k_stable_radix<STABLE_BT_MAX, STABLE_BT_T, true><<<148, STABLE_BT_T, stable_radix_smem(STABLE_BT_MAX, STABLE_BT_T), s>>>(
            cells->cell_start, rec, xs, vs, cells->perm, bt_items, bt_count + 1, (int)w.huge_cap);
        k_stable_big<<<148 * 4, STABLE_BIG_CHUNK, 0, s>>>(cells->cell_start, rec, xs, vs, cells->perm, big_items,
                                                          big_count);
    }
    if (n == 0 && (e = cudaMemsetAsync(cells->cell_nhome, 0, 4 * (size_t)g.ncell, s)) != cudaSuccess)
        return cuda_fail(e);
    if (n == 0 && (e = cudaMemsetAsync(cells->cell_hmax, 0, 4 * (size_t)g.ncell, s)) != cudaSuccess)
        return cuda_fail(e);
    if (n == 0 && (e = cudaMemsetAsync(cells->cell_dx, 0, 4 * (size_t)g.ncell, s)) != cudaSuccess)
        return cuda_fail(e);
    cells->n = n;
    return check_launch();
}

// sph_sort_cells; SMALL_DONE: cells of <= SORT_SMALL particles already have their lists
int sort_impl(const sph_grid *grid, const sph_cells *cells, int64_t cell_begin, int64_t cell_end, void *ws,
              size_t ws_bytes, void *stream, bool small_done)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (!cells_ok(cells) || !ws) return SPH_EINVAL;
    if (cell_end < 0) cell_end = g.ncell;
    if (cell_begin < 0 || cell_begin > cell_end || cell_end > g.ncell) return SPH_EINVAL;
    Ws w = ws_layout(g, cells->capacity);
    if (ws_bytes < w.total) return SPH_EINVAL;
    if (cell_end == cell_begin) return SPH_OK;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    int *big_count = at<int>(ws, w.big_count);
    int2 *big_items = at<int2>(ws, w.big_items);
    int *huge_count = at<int>(ws, w.huge_count);
    int *huge_items = at<int>(ws, w.huge_items);
    if ((e = cudaMemsetAsync(big_count, 0, 4, s)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaMemsetAsync(huge_count, 0, 16, s)) != cudaSuccess) return cuda_fail(e);
    int *mid_items = at<int>(ws, w.mid_items), *w256_items = at<int>(ws, w.w256_items);
    DevCells c = dev_cells(cells);
    int *need = nullptr;
    if (g.h_home_max > 0.0f) {                 // level pass: sort only cells next to home particles
        need = at<int>(ws, w.count);           // (the build's count array, free after the build)
        if ((e = cudaMemsetAsync(need, 0, 4 * (size_t)g.ncell, s)) != cudaSuccess) return cuda_fail(e);
        k_mark_needed<<<grid_blocks(g.ncell, 256, 148 * 32), 256, 0, s>>>(g, cells->cell_nhome, need);
    }
    // huge cells' directions in groups over several CTAs (item = cell | group << 28)
    const int huge_ngrp = g.ncell < (1ll << 28) ? SORT_DIR_GROUPS : 1;
    static_assert(sizeof(ParticleRec) >= 12 * SORT_DIR_GROUPS, "giant-tier scratch stripes fit the record region");
    k_sort_small<<<grid_blocks(cell_end - cell_begin, SORT_WARPS, 148 * 64), SORT_WARPS * 32, 0, s>>>(
        g, c, cells->order, cell_begin, cell_end, big_items, big_count, huge_items, huge_count, (int)w.huge_cap,
        mid_items, huge_count + 2, w256_items, huge_count + 3, need, small_done, huge_ngrp);
    k_sort_mid<<<148 * 8, SORT_WARPS * 32, 0, s>>>(g, c, cells->order, mid_items, huge_count + 2, need);
    k_sort_warp256<<<148 * 4, SORT_WARPS * 32, 0, s>>>(g, c, cells->order, w256_items, huge_count + 3, need);
    if ((rc = ensure_attrs()) != SPH_OK) return rc;
    // cells above SORT_HUGE_MAX: key/index buffers in the build's record region (free after it)
    k_sort_radix<65535, SORT_GIANT_T, false, true, 2><<<148, SORT_GIANT_T, radix_smem_global(SORT_GIANT_T), s>>>(
        g, c, cells->order, reinterpret_cast<const int *>(big_items), big_count, 0, need,
        at<unsigned>(ws, w.rec), SORT_DIR_GROUPS);
    k_sort_radix<SORT_MED_MAX, SORT_MED_T, false><<<148 * 8, SORT_MED_T, radix_smem(SORT_MED_MAX, SORT_MED_T), s>>>(
        g, c, cells->order, huge_items, huge_count, (int)w.huge_cap, need);
    k_sort_radix<SORT_HUGE_MAX, SORT_HUGE_T, true><<<148, SORT_HUGE_T, radix_smem(SORT_HUGE_MAX, SORT_HUGE_T), s>>>(
        g, c, cells->order, huge_items, huge_count + 1, (int)w.huge_cap, need, nullptr, huge_ngrp);
    return check_launch();
}

}  // namespace

extern "C" {

int sph_build_cells(const sph_grid *grid, int64_t n_own, int64_t n_ghost, const float *xyzh_in, const float *vm_in,
                    sph_cells *cells, void *ws, size_t ws_bytes, void *stream)
{
    return build_impl(grid, n_own, n_ghost, xyzh_in, vm_in, cells, ws, ws_bytes, stream, false);
}

int sph_sort_cells(const sph_grid *grid, const sph_cells *cells, int64_t cell_begin, int64_t cell_end, void *ws,
                   size_t ws_bytes, void *stream)
{
    return sort_impl(grid, cells, cell_begin, cell_end, ws, ws_bytes, stream, false);
}

int sph_build_sort_cells(const sph_grid *grid, int64_t n_own, int64_t n_ghost, const float *xyzh_in,
                         const float *vm_in, sph_cells *cells, void *ws, size_t ws_bytes, void *stream)
{
    // level grids sort only the cells next to home particles (known after the build): unfused
    const bool fuse = grid && !(grid->h_home_max > 0.0f);
    int rc = build_impl(grid, n_own, n_ghost, xyzh_in, vm_in, cells, ws, ws_bytes, stream, fuse);
    if (rc) return rc;
    return sort_impl(grid, cells, 0, -1, ws, ws_bytes, stream, fuse);
}

int sph_density_self(const sph_grid *grid, const sph_cells *cells, const int32_t *cell_list, int64_t ncells_list,
                     sph_out *acc, sph_stats *stats, void *ws, size_t ws_bytes, void *stream)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (!cells_ok(cells) || !out_ok(acc) || !ws || ncells_list < 0 || (ncells_list > 0 && !cell_list)) return SPH_EINVAL;
    if (ws_bytes < 4) return SPH_EINVAL;
    if (ncells_list == 0) return SPH_OK;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned *status = at<unsigned>(ws, 0);
    int blocks = grid_blocks(ncells_list, API_WARPS, 1 << 30);
    if (stats)
        k_density_self<true><<<blocks, API_WARPS * 32, 0, s>>>(g, dev_cells(cells), dev_out(acc), cell_list,
                                                               ncells_list, stats, status);
    else
        k_density_self<false><<<blocks, API_WARPS * 32, 0, s>>>(g, dev_cells(cells), dev_out(acc), cell_list,
                                                                ncells_list, nullptr, status);
    return check_launch();
}

int sph_density_pair(const sph_grid *grid, const sph_cells *cells, const int32_t *pairs, int64_t npairs, sph_out *acc,
                     sph_stats *stats, void *ws, size_t ws_bytes, void *stream)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (!cells_ok(cells) || !out_ok(acc) || !ws || npairs < 0 || (npairs > 0 && !pairs)) return SPH_EINVAL;
    if (((uintptr_t)pairs % 8) || ws_bytes < 4) return SPH_EINVAL;
    if (npairs == 0) return SPH_OK;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned *status = at<unsigned>(ws, 0);
    const int2 *pr = reinterpret_cast<const int2 *>(pairs);
    if ((rc = ensure_attrs()) != SPH_OK) return rc;
    const int blocks = grid_blocks(npairs, 1, 148 * 8);
    if (stats)
        k_density_pair_staged<true><<<blocks, PAIR_WARPS * 32, PAIR_SMEM, s>>>(g, dev_cells(cells), dev_out(acc), pr,
                                                                            npairs, stats, status);
    else
        k_density_pair_staged<false><<<blocks, PAIR_WARPS * 32, PAIR_SMEM, s>>>(g, dev_cells(cells), dev_out(acc), pr,
                                                                             npairs, nullptr, status);
    return check_launch();
}

int sph_density_pair_sym(const sph_grid *grid, const sph_cells *cells, const int32_t *pairs, int64_t npairs,
                         sph_out *acc, sph_stats *stats, void *ws, size_t ws_bytes, void *stream)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (!cells_ok(cells) || !out_ok(acc) || !ws || npairs < 0 || (npairs > 0 && !pairs)) return SPH_EINVAL;
    if (((uintptr_t)pairs % 8) || ws_bytes < 4) return SPH_EINVAL;
    if (npairs == 0) return SPH_OK;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned *status = at<unsigned>(ws, 0);
    const int2 *pr = reinterpret_cast<const int2 *>(pairs);
    if ((rc = ensure_attrs()) != SPH_OK) return rc;
    const int blocks = grid_blocks(npairs, 1, 148 * 12);
    if (stats)
        k_density_pair_sym<true><<<blocks, SYM_WARPS * 32, SYM_SMEM, s>>>(g, dev_cells(cells), dev_out(acc), pr, npairs,
                                                                        stats, status);
    else
        k_density_pair_sym<false><<<blocks, SYM_WARPS * 32, SYM_SMEM, s>>>(g, dev_cells(cells), dev_out(acc), pr,
                                                                         npairs, nullptr, status);
    return check_launch();
}

int sph_drift(const sph_grid *grid, sph_cells *cells, float dt, float *max_disp, void *stream)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (!cells_ok(cells) || !std::isfinite(dt)) return SPH_EINVAL;
    if (cells->n <= 0) return SPH_OK;
    k_drift<<<grid_blocks(cells->n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<float4 *>(cells->xyzh), reinterpret_cast<const float4 *>(cells->vm),
        cells->cell_start + g.ncell, dt, cells->disp, cells->slot_cell, cells->cell_dx, max_disp);
    return check_launch();
}

int sph_gather_positions(const sph_grid *grid, const sph_cells *cells, float *xyzh_out, int64_t n_out, void *stream)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (!cells_ok(cells) || n_out < 0 || (n_out > 0 && !xyzh_out) || ((uintptr_t)xyzh_out % 16)) return SPH_EINVAL;
    if (cells->n <= 0 || n_out == 0) return SPH_OK;
    k_gather_positions<<<grid_blocks(cells->n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float4 *>(cells->xyzh), cells->perm, cells->cell_start + g.ncell, n_out, g.boxf[0],
        g.boxf[1], g.boxf[2], reinterpret_cast<float4 *>(xyzh_out));
    return check_launch();
}

__global__ void k_mask_ghost_rows(float4 *x, float4 *v, long long cap, const long long *__restrict__ counts,
                                  float4 dx, float4 dv)
{
    const long long n0 = counts[0], n1 = counts[1];
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < 2 * cap;
         r += (long long)gridDim.x * blockDim.x) {
        const long long k = r >= cap, row = r - k * cap;
        if (row >= (k ? n1 : n0)) {
            x[r] = dx;
            v[r] = dv;
        }
    }
}

int sph_mask_ghost_rows(float *xyzh, float *vm, int64_t cap, const int64_t *counts, const float dead_xyzh[4],
                        const float dead_vm[4], void *stream)
{
    if (cap < 0 || !counts || !dead_xyzh || !dead_vm || (cap > 0 && (!xyzh || !vm))) return SPH_EINVAL;
    if (((uintptr_t)xyzh % 16) || ((uintptr_t)vm % 16)) return SPH_EINVAL;
    if (cap == 0) return SPH_OK;
    const float4 dx = make_float4(dead_xyzh[0], dead_xyzh[1], dead_xyzh[2], dead_xyzh[3]);
    const float4 dv = make_float4(dead_vm[0], dead_vm[1], dead_vm[2], dead_vm[3]);
    k_mask_ghost_rows<<<grid_blocks(2 * cap, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<float4 *>(xyzh), reinterpret_cast<float4 *>(vm), cap,
        reinterpret_cast<const long long *>(counts), dx, dv);
    return check_launch();
}

int sph_select_planes(const sph_grid *grid, int64_t n_own, const float *xyzh_in, const float *vm_in,
                      float *sel_xyzh, float *sel_vm, int64_t cap, int64_t *counts, void *ws, size_t ws_bytes,
                      void *stream)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (n_own < 0 || cap < 0 || !counts || !ws || (n_own > 0 && (!xyzh_in || !vm_in))) return SPH_EINVAL;
    if (cap > 0 && (!sel_xyzh || !sel_vm)) return SPH_EINVAL;
    if (((uintptr_t)xyzh_in % 16) || ((uintptr_t)vm_in % 16) || ((uintptr_t)sel_xyzh % 16) || ((uintptr_t)sel_vm % 16))
        return SPH_EINVAL;
    // scratch in the build's cell_of region: it starts at a fixed offset for any capacity and
    // is written only inside sph_build_cells (the call counter and other state are untouched)
    Ws w = ws_layout(g, n_own);
    const long long nblk = (n_own + SEL_B - 1) / SEL_B, nk = 2 * nblk;
    const size_t blk_off = w.cell_of, sum_off = align_up(blk_off + 4 * (size_t)(nk + 1), 16);
    if (ws_bytes < w.total || sum_off + 4 * (size_t)((nk + SCAN_TILE - 1) / SCAN_TILE + 1) > w.rank)
        return SPH_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    if (n_own == 0) {
        if ((e = cudaMemsetAsync(counts, 0, 16, s)) != cudaSuccess) return cuda_fail(e);
        return SPH_OK;
    }
    int *blk = at<int>(ws, blk_off), *sum = at<int>(ws, sum_off);
    unsigned *status = at<unsigned>(ws, w.status);
    const float4 *x = reinterpret_cast<const float4 *>(xyzh_in), *v = reinterpret_cast<const float4 *>(vm_in);
    k_sel_count<<<(int)nblk, SEL_B, 0, s>>>(g, n_own, x, blk, nblk);
    const long long nt = (nk + SCAN_TILE - 1) / SCAN_TILE;
    k_scan_tiles<<<(int)nt, SCAN_T, 0, s>>>(blk, nk, blk, sum, status, SEL_B);
    k_scan_sums<<<1, SCAN_T, 0, s>>>(sum, nt, blk, nk);
    k_scan_add<<<(int)nt, SCAN_T, 0, s>>>(blk, nk, sum);
    k_sel_write<<<(int)nblk, SEL_B, 0, s>>>(g, n_own, x, v, blk, nblk, reinterpret_cast<float4 *>(sel_xyzh),
                                             reinterpret_cast<float4 *>(sel_vm), cap,
                                             reinterpret_cast<long long *>(counts), status);
    return check_launch();
}

int sph_partition_migrants(const sph_grid *grid, int64_t n, const float *xyzh, const float *vm, const int64_t *gid,
                           float *lo_xyzh, float *lo_vm, int64_t *lo_gid, int64_t cap_lo, float *hi_xyzh,
                           float *hi_vm, int64_t *hi_gid, int64_t cap_hi, float *keep_xyzh, float *keep_vm,
                           int64_t *keep_gid, int64_t cap_keep, int64_t *counts, void *ws, size_t ws_bytes,
                           void *stream)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (n < 0 || cap_lo < 0 || cap_hi < 0 || cap_keep < 0 || !counts || !ws) return SPH_EINVAL;
    if (n > 0 && (!xyzh || !vm || !gid)) return SPH_EINVAL;
    const float *outs[6] = {lo_xyzh, lo_vm, hi_xyzh, hi_vm, keep_xyzh, keep_vm};
    const int64_t caps[3] = {cap_lo, cap_hi, cap_keep};
    const int64_t *gids[3] = {lo_gid, hi_gid, keep_gid};
    for (int k = 0; k < 3; ++k)
        if (caps[k] > 0 && (!outs[2 * k] || !outs[2 * k + 1] || !gids[k])) return SPH_EINVAL;
    const float *aligned[8] = {xyzh, vm, lo_xyzh, lo_vm, hi_xyzh, hi_vm, keep_xyzh, keep_vm};
    for (const float *q : aligned)
        if ((uintptr_t)q % 16) return SPH_EINVAL;
    // scratch: the build's cell_of region, as sph_select_planes
    Ws w = ws_layout(g, n);
    const long long nblk = (n + SEL_B - 1) / SEL_B, nk = 3 * nblk;
    const size_t blk_off = w.cell_of, sum_off = align_up(blk_off + 4 * (size_t)(nk + 1), 16);
    if (ws_bytes < w.total || sum_off + 4 * (size_t)((nk + SCAN_TILE - 1) / SCAN_TILE + 1) > w.rank)
        return SPH_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    if (n == 0) {
        if ((e = cudaMemsetAsync(counts, 0, 24, s)) != cudaSuccess) return cuda_fail(e);
        return SPH_OK;
    }
    int *blk = at<int>(ws, blk_off), *sum = at<int>(ws, sum_off);
    unsigned *status = at<unsigned>(ws, w.status);
    const float4 *x = reinterpret_cast<const float4 *>(xyzh), *v = reinterpret_cast<const float4 *>(vm);
    MigOut o;
    for (int k = 0; k < 3; ++k) {
        o.x[k] = reinterpret_cast<float4 *>(const_cast<float *>(outs[2 * k]));
        o.v[k] = reinterpret_cast<float4 *>(const_cast<float *>(outs[2 * k + 1]));
        o.g[k] = reinterpret_cast<long long *>(const_cast<int64_t *>(gids[k]));
        o.cap[k] = caps[k];
    }
    k_mig_count<<<(int)nblk, SEL_B, 0, s>>>(g, n, x, blk, nblk);
    const long long nt = (nk + SCAN_TILE - 1) / SCAN_TILE;
    k_scan_tiles<<<(int)nt, SCAN_T, 0, s>>>(blk, nk, blk, sum, status, SEL_B);
    k_scan_sums<<<1, SCAN_T, 0, s>>>(sum, nt, blk, nk);
    k_scan_add<<<(int)nt, SCAN_T, 0, s>>>(blk, nk, sum);
    k_mig_write<<<(int)nblk, SEL_B, 0, s>>>(g, n, x, v, reinterpret_cast<const long long *>(gid), blk, nblk, o,
                                             reinterpret_cast<long long *>(counts), status);
    return check_launch();
}

int sph_merge_by_id(int64_t na, const float *a_xyzh, const float *a_vm, const int64_t *a_gid, int64_t nb,
                    const float *b_xyzh, const float *b_vm, const int64_t *b_gid, int64_t nc, const float *c_xyzh,
                    const float *c_vm, const int64_t *c_gid, float *out_xyzh, float *out_vm, int64_t *out_gid,
                    void *stream)
{
    const int64_t ns[3] = {na, nb, nc};
    const float *xs[3] = {a_xyzh, b_xyzh, c_xyzh}, *vs[3] = {a_vm, b_vm, c_vm};
    const int64_t *gs[3] = {a_gid, b_gid, c_gid};
    MergeIn in;
    for (int k = 0; k < 3; ++k) {
        if (ns[k] < 0 || (ns[k] > 0 && (!xs[k] || !vs[k] || !gs[k]))) return SPH_EINVAL;
        if (((uintptr_t)xs[k] % 16) || ((uintptr_t)vs[k] % 16)) return SPH_EINVAL;
        in.x[k] = reinterpret_cast<const float4 *>(xs[k]);
        in.v[k] = reinterpret_cast<const float4 *>(vs[k]);
        in.g[k] = reinterpret_cast<const long long *>(gs[k]);
        in.n[k] = ns[k];
    }
    const long long total = na + nb + nc;
    if (total == 0) return SPH_OK;
    if (!out_xyzh || !out_vm || !out_gid || ((uintptr_t)out_xyzh % 16) || ((uintptr_t)out_vm % 16))
        return SPH_EINVAL;
    k_merge_by_id<<<grid_blocks(total, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
        in, reinterpret_cast<float4 *>(out_xyzh), reinterpret_cast<float4 *>(out_vm),
        reinterpret_cast<long long *>(out_gid));
    return check_launch();
}

__global__ void k_max_speed(const float4 *__restrict__ vm, long long n, unsigned long long *out)
{
    double m = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float4 v = vm[i];
        m = fmax(m, sqrt((double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z));
    }
    // non-negative doubles order like their bit patterns
    unsigned long long b = (unsigned long long)__double_as_longlong(m);
    for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, b);
}

int sph_max_speed(const float *vm, int64_t n, double *out, void *stream)
{
    if (n < 0 || !out || (n > 0 && !vm) || ((uintptr_t)vm % 16)) return SPH_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(out, 0, 8, s);
    if (e != cudaSuccess) return cuda_fail(e);
    if (n == 0) return SPH_OK;
    k_max_speed<<<grid_blocks(n, 256, 148 * 8), 256, 0, s>>>(reinterpret_cast<const float4 *>(vm), n,
                                                             reinterpret_cast<unsigned long long *>(out));
    return check_launch();
}

int sph_density_finalize(sph_out *acc, int64_t n, void *stream)
{
    if (!out_ok(acc) || n < 0 || n > acc->n_out) return SPH_EINVAL;
    if (n == 0) return SPH_OK;
    k_finalize<<<grid_blocks(n, 256, 148 * 32), 256, 0, (cudaStream_t)stream>>>(dev_out(acc), n);
    return check_launch();
}

int sph_density_all(const sph_grid *grid, const sph_cells *cells, sph_out *out, sph_stats *stats, void *ws,
                    size_t ws_bytes, void *stream)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (!cells_ok(cells) || !out_ok(out) || !ws || ws_bytes < 4) return SPH_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const char *eng = std::getenv("PVSPH_ENGINE");   // "v1": reference engine (validation only)
    if (eng && eng[0] == 'v' && eng[1] == '1') {
        int blocks = grid_blocks(g.n_owned_cells, V1_WARPS, 1 << 30);
        if (stats)
            k_density_all_v1<true><<<blocks, V1_WARPS * 32, 0, s>>>(g, dev_cells(cells), dev_out(out), stats);
        else
            k_density_all_v1<false><<<blocks, V1_WARPS * 32, 0, s>>>(g, dev_cells(cells), dev_out(out), nullptr);
        return check_launch();
    }
    Ws w = ws_layout(g, cells->capacity);
    if (ws_bytes < w.total) return SPH_EINVAL;
    // tile list (k_v4_tiles): count per row pair -> exclusive scan -> write
    const long long nkeys = row_pairs(g).nkeys;
    int *rows = at<int>(ws, w.rows), *rows_sum = at<int>(ws, w.rows_sum);
    unsigned *status = at<unsigned>(ws, w.status);
    int4 *tiles = at<int4>(ws, w.tiles);
    int *counter = at<int>(ws, w.counter);
    const DevCells dc = dev_cells(cells);
    unsigned *gen = at<unsigned>(ws, w.gen);
    int *gtiles = at<int>(ws, w.gtiles), *gcount = at<int>(ws, w.gcount);
    k_row_home<<<grid_blocks((long long)g.nxl * g.ny * 32, 256, 148 * 16), 256, 0, s>>>((long long)g.nxl * g.ny, g.nz,
                                                                                      dc.cell_nhome,
                                                                                      at<int>(ws, w.row_home));
    k_v4_tiles<false><<<grid_blocks(nkeys, 256, 148 * 8), 256, 0, s>>>(g, dc.cell_start, dc.cell_nhome, rows, tiles,
                                                                       w.tile_cap, status, gen, gtiles, gcount,
                                                                       at<int>(ws, w.row_home));
    const long long ntiles_scan = (nkeys + SCAN_TILE - 1) / SCAN_TILE;
    k_scan_tiles<<<(int)ntiles_scan, SCAN_T, 0, s>>>(rows, nkeys, rows, rows_sum, status, 0x7fffffff);
    k_scan_sums<<<1, SCAN_T, 0, s>>>(rows_sum, ntiles_scan, rows, nkeys);
    k_scan_add<<<(int)ntiles_scan, SCAN_T, 0, s>>>(rows, nkeys, rows_sum);
    cudaError_t e;
    if ((e = cudaMemsetAsync(gcount, 0, 8, s)) != cudaSuccess) return cuda_fail(e);
    k_v4_tiles<true><<<grid_blocks(nkeys, 256, 148 * 8), 256, 0, s>>>(g, dc.cell_start, dc.cell_nhome, rows, tiles,
                                                                      w.tile_cap, status, gen, gtiles, gcount,
                                                                      at<int>(ws, w.row_home));
    if ((e = cudaMemsetAsync(counter, 0, 4, s)) != cudaSuccess) return cuda_fail(e);
    const bool v4 = eng && eng[0] == 'v' && eng[1] == '4';   // round-1 engine (comparison only)
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return cuda_fail(e);
    const DevAttrs &da = dev_attrs(dev);
    const int blocks = da.sms * (v4 ? da.v4_blocks_per_sm : da.v5_blocks_per_sm);
    OutRec *orec = at<OutRec>(ws, w.orec);
    if (v4) {
        if (stats)
            k_density_v4<true><<<blocks, V4_TP, V4_SMEM, s>>>(g, dc, orec, stats, tiles, rows + nkeys, counter, gen);
        else
            k_density_v4<false><<<blocks, V4_TP, V4_SMEM, s>>>(g, dc, orec, nullptr, tiles, rows + nkeys, counter, gen);
    } else {
        if (stats)
            k_density_v5<true><<<blocks, V5_TP, V5_SMEM, s>>>(g, dc, orec, stats, tiles, rows + nkeys, counter, gen, status);
        else
            k_density_v5<false><<<blocks, V5_TP, V5_SMEM, s>>>(g, dc, orec, nullptr, tiles, rows + nkeys, counter, gen,
                                                              status);
    }
    const int sms = da.sms;
    // the slices k_v4_tiles could not stage (dense clustered cells): warp-level engine
    if (stats)
        k_density_dense<true><<<sms * 2, DENSE_WARPS * 32, DENSE_SMEM, s>>>(g, dc, orec, stats, tiles, gtiles, gcount,
                                                                         gcount + 1, gen);
    else
        k_density_dense<false><<<sms * 2, DENSE_WARPS * 32, DENSE_SMEM, s>>>(g, dc, orec, nullptr, tiles, gtiles,
                                                                          gcount, gcount + 1, gen);
    if (out->n_out > 0)
        k_unpermute<<<grid_blocks(out->n_out, 256, 148 * 16), 256, 0, s>>>(dev_out(out), orec, gen);
    return check_launch();
}

int sph_density_all_sym(const sph_grid *grid, const sph_cells *cells, sph_out *out, sph_stats *stats, void *ws,
                        size_t ws_bytes, void *stream)
{
    DevGrid g;
    int rc = make_grid(grid, g);
    if (rc) return rc;
    if (!cells_ok(cells) || !out_ok(out) || !ws) return SPH_EINVAL;
    Ws w = ws_layout(g, cells->capacity);
    if (ws_bytes < w.total) return SPH_EINVAL;
    if ((rc = ensure_attrs()) != SPH_OK) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    const DevOut o = dev_out(out);
    const size_t nb = 4 * (size_t)out->n_out;
    for (float *a : {out->rho, out->rho_dh, out->wcount, out->wcount_dh, out->div_v})
        if (nb && (e = cudaMemsetAsync(a, 0, nb, s)) != cudaSuccess) return cuda_fail(e);
    if (nb && (e = cudaMemsetAsync(out->curl_v, 0, 3 * nb, s)) != cudaSuccess) return cuda_fail(e);
    if (nb && (e = cudaMemsetAsync(out->nngb, 0, nb, s)) != cudaSuccess) return cuda_fail(e);
    const DevCells dc = dev_cells(cells);
    unsigned *status = at<unsigned>(ws, w.status);
    // scratch: the phase's pair list in the build's record region, its count in big_count
    int2 *pairs = at<int2>(ws, w.rec);
    int *count = at<int>(ws, w.big_count);
    // a phase lists at most one pair per non-empty cell, so at most min(ncell, capacity) pairs:
    // two such lists (the phase's pairs, the deferred large ones) = 16 B per stored slot, inside
    // the 64 B per slot of the record region
    const long long maxp = std::min<long long>(g.ncell, cells->capacity > 0 ? cells->capacity : 1);
    static_assert(sizeof(ParticleRec) >= 16, "two int2 pair lists per stored slot");
    const int gen_blocks = grid_blocks(g.n_owned_cells, 256, 148 * 8);
    // self cells (every ordered pair i != j and the self term): one warp per cell, exclusive
    if ((e = cudaMemsetAsync(count, 0, 4, s)) != cudaSuccess) return cuda_fail(e);
    k_sym_phase_pairs<<<gen_blocks, 256, 0, s>>>(g, dc.cell_start, -1, 0, pairs, count);
    // (the self kernel takes a cell list: the first int of each (c, c) record is the cell)
    {
        const int blocks = grid_blocks(g.n_owned_cells, API_WARPS, 1 << 30);
        if (stats)
            k_density_self<true><<<blocks, API_WARPS * 32, 0, s>>>(g, dc, o, reinterpret_cast<const int *>(pairs),
                                                                   -2, stats, status, count);
        else
            k_density_self<false><<<blocks, API_WARPS * 32, 0, s>>>(g, dc, o, reinterpret_cast<const int *>(pairs),
                                                                    -2, nullptr, status, count);
    }
    // the 13 directions x colours: symmetric pairs, no atomics
    // pairs with a cell above SYMW_MAXN: deferred to the CTA form (list after the phase's pairs,
    // count in big_count + 1)
    int2 *big = pairs + maxp;
    int *big_n = count + 1;
    // per-slot accumulators in the output-record region (SlotAcc = sizeof(OutRec) per slot)
    static_assert(sizeof(SlotAcc) == sizeof(OutRec), "slot accumulators reuse the output-record region");
    SlotAcc *sacc = at<SlotAcc>(ws, w.orec);
    if ((e = cudaMemsetAsync(sacc, 0, sizeof(SlotAcc) * (size_t)(cells->capacity > 0 ? cells->capacity : 1), s)) !=
        cudaSuccess)
        return cuda_fail(e);
    for (int d = 0; d < SPH_NDIR; ++d)
        for (int col = 0; col < sym_dir_colours(g, d); ++col) {
            if ((e = cudaMemsetAsync(count, 0, 8, s)) != cudaSuccess) return cuda_fail(e);
            k_sym_phase_pairs<<<gen_blocks, 256, 0, s>>>(g, dc.cell_start, d, col, pairs, count);
            const int wblocks = 148 * 2;
            if (stats)
                k_density_pair_sym<true, true, SYMW_MAXN, 1, SYMW_WARPS><<<wblocks, SYMW_WARPS * 32, SYMW_SMEM, s>>>(
                    g, dc, o, pairs, maxp, stats, status, count, big, big_n, sacc);
            else
                k_density_pair_sym<false, true, SYMW_MAXN, 1, SYMW_WARPS><<<wblocks, SYMW_WARPS * 32, SYMW_SMEM, s>>>(
                    g, dc, o, pairs, maxp, nullptr, status, count, big, big_n, sacc);
            const int blocks = 148 * 3;
            if (stats)
                k_density_pair_sym<true, true><<<blocks, SYM_WARPS * 32, SYM_SMEM, s>>>(
                    g, dc, o, big, maxp, stats, status, big_n, nullptr, nullptr, sacc);
            else
                k_density_pair_sym<false, true><<<blocks, SYM_WARPS * 32, SYM_SMEM, s>>>(
                    g, dc, o, big, maxp, nullptr, status, big_n, nullptr, nullptr, sacc);
        }
    k_sym_merge<<<grid_blocks(cells->capacity, 256, 148 * 16), 256, 0, s>>>(o, sacc, dc.perm, dc.cell_start + g.ncell);
    return check_launch();
}

int sph_status(void *ws, void *stream)
{
    if (!ws) return SPH_EINVAL;
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e);
    unsigned st = 0;
    e = cudaMemcpy(&st, ws, 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e);
    if (st & ST_EINVAL) return SPH_EINVAL;
    if (st & ST_EDOMAIN) return SPH_EDOMAIN;
    if (st & ST_EH_RANGE) return SPH_EH_RANGE;
    if (st & ST_ECAPACITY) return SPH_ECAPACITY;
    return SPH_OK;
}

#ifdef PVSPH_PHASE_TIMING
int sph_debug_phase_cycles(unsigned long long *out8, int reset)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out8, g_phase_cycles, 12 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
    }
    return SPH_OK;
}
#endif

#if defined(V5_CHECK_BISECT) || defined(V5_STATS)
int sph_debug_v5(unsigned long long *out16)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out16, g_v5dbg, 16 * sizeof(unsigned long long));
    return SPH_OK;
}
#endif

int sph_calibrate(int mode, int blocks, int threads, int iters, float *out, void *stream)
{
    if (mode < 0 || mode > 3 || blocks <= 0 || threads <= 0 || threads > 1024 || iters <= 0 || !out) return SPH_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    if (mode == 0) k_calib_ffma<<<blocks, threads, 0, s>>>(out, iters);
    else if (mode == 1) k_calib_ffma2<<<blocks, threads, 0, s>>>(out, iters);
    else if (mode == 2) k_calib_interact<<<blocks, threads, 0, s>>>(out, iters);
    else k_calib_interact2<<<blocks, threads, 0, s>>>(out, iters);
    return check_launch();
}

const char *sph_strerror(int code)
{
    switch (code) {
    case SPH_OK: return "ok";
    case SPH_EINVAL: return "invalid argument (null pointer, bad size or grid, workspace too small, bad cell list)";
    case SPH_EH_RANGE: return "smoothing length or mass out of range (h <= 0, m <= 0 or gamma*h > cell edge)";
    case SPH_ECAPACITY: return "capacity exceeded (cell occupancy > SPH_MAX_CELL or particle arrays too small)";
    case SPH_EDOMAIN: return "position not finite or outside the box / the rank's slab";
    case SPH_ECUDA: return g_cuda_msg;
    default: return "unknown error";
    }
}

}  // extern "C"
