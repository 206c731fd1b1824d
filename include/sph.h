/*
 * sph.h -- C ABI of libpvsph.so: the pseudo-Verlet SPH density loop of
 * Willis, Schaller, Gonnet, Bower & Draper, "An Efficient SIMD Implementation
 * of Pseudo-Verlet Lists for Neighbour Interactions in Particle-Based Codes"
 * (arXiv:1804.06231), on NVIDIA B200 (sm_100a).
 *
 * Citations "P:n" are lines of the paper text (reference PAPER.md).
 *
 * Problem statement:
 *   N particles with positions x_i, per-particle smoothing length h_i,
 *   velocity v_i and mass m_i in a periodic box.  The cut-off radius of
 *   particle i is H_i = gamma * h_i (the paper's "h_i"); j is a neighbour of
 *   i iff j != i and |x_i - x_j|^2 < H_i^2 (minimum image; gather on h_i).
 *   The box is decomposed into cells of edge C_l >= max H, particles
 *   of a cell are stored together, and for each of the 13 symmetry-reduced
 *   cell-pair directions every cell keeps its particles sorted by
 *   their projection on the unit axis ("dist" and "index").  For each
 *   pair of neighbouring cells only the particles of the neighbour whose
 *   projected separation is below H_i are tested (Code 2).
 *   For every particle the library computes, with the M4 cubic spline
 *   W(r,h) = (16/pi) H^-3 w(r/H) (support H = gamma h):
 *     rho       = m_i W(0,h_i) + sum_j m_j W(r_ij,h_i)
 *     wcount    =     W(0,h_i) + sum_j     W(r_ij,h_i)
 *     rho_dh    = d rho / d h_i,   wcount_dh = d wcount / d h_i
 *     div_v     = -(1/rho) sum_j m_j (v_ij . x_ij) W'(r_ij)/r_ij
 *     curl_v    =  (1/rho) sum_j m_j (v_ij x x_ij) W'(r_ij)/r_ij
 *     nngb      = number of neighbours (self excluded)
 *
 * Conventions for every call:
 *   - All array pointers are DEVICE pointers unless stated otherwise; the
 *     caller allocates and owns all memory (inputs, sph_cells arrays,
 *     outputs, workspace).  The library allocates nothing; its only global
 *     state is one-time kernel attribute setup (first call) and the text of
 *     the last CUDA error (sph_strerror).  Calls on different streams with
 *     disjoint outputs and workspaces may run concurrently (after a first
 *     call of each entry point from one thread).
 *   - The workspace (sph_workspace_bytes) is zero-filled by the caller once
 *     after allocation; afterwards the calls own its contents (it carries
 *     the status word and a sph_density_all call counter that tags output
 *     records, so one workspace serves one grid at a time).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *     Calls are asynchronous: argument errors are returned at once,
 *     data-dependent errors set the device status word in the workspace,
 *     read by sph_status() (one stream synchronisation).
 *   - Return codes: SPH_OK, SPH_EINVAL (null pointer, bad size or grid,
 *     workspace too small), SPH_EH_RANGE (h <= 0, m <= 0, or gamma*h +
 *     2*skin > C_l for a home particle),
 *     SPH_ECAPACITY (a cell holds more than SPH_MAX_CELL particles, or the
 *     particle arrays are too small), SPH_EDOMAIN (non-finite value, or a
 *     position outside [0, box) / outside the rank's slab), SPH_ECUDA (a
 *     CUDA launch failed; sph_strerror(SPH_ECUDA) gives the CUDA message).
 */
#ifndef PVSPH_SPH_H
#define PVSPH_SPH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPH_ABI_VERSION 7

#define SPH_OK 0
#define SPH_EINVAL 1
#define SPH_EH_RANGE 2
#define SPH_ECAPACITY 3
#define SPH_EDOMAIN 4
#define SPH_ECUDA 5

/* Largest number of particles one cell may hold. */
#define SPH_MAX_CELL 65535

/* Number of sort directions and the window margin: a candidate is
 * swept when its projected separation is below H_i + SPH_DELTA_FRAC * C_l
 * + 4 * skin (reading R5: covers fp32 rounding of the keys; the
 * skin term covers drifts since the lists were built, §4.6). */
#define SPH_NDIR 13
#define SPH_DELTA_FRAC (1.0 / 65536.0)

/* Cell grid of one rank.  Cells are numbered x-major on the LOCAL grid:
 *   cell = (ixl * nc[1] + iy) * nc[2] + iz,  ixl = ix - x_lo + ghost_x,
 * whose x extent is nx_local = (x_hi - x_lo) + 2 * ghost_x planes.  With
 * ghost_x = 0 the rank must own every plane (x_lo = 0, x_hi = nc[0]) and x
 * is periodic like y and z; with ghost_x = 1 planes x_lo-1 and x_hi (mod
 * nc[0]) are read-only ghost planes (x-slab decomposition). */
typedef struct sph_grid {
    int32_t nc[3];      /* global cells per dimension, each >= 3            */
    int32_t x_lo, x_hi; /* owned x planes [x_lo, x_hi)                      */
    int32_t ghost_x;    /* 0 or 1                                           */
    int32_t reserved;   /* must be 0                                        */
    double box[3];      /* periodic box lengths (> 0)                       */
    float gamma;        /* support / smoothing length (1.825742)            */
    float h_home_min;   /* level passes: if h_home_max > 0, */
    float h_home_max;   /*   only particles with h_home_min < h <= h_home_max */
                        /*   are HOME (outputs computed) on this grid; the  */
                        /*   others are binned as neighbour sources only    */
                        /*   and may have gamma*h > C_l.  0, 0: all home.   */
    float skin;         /* list reuse: the      */
                        /*   largest displacement any particle may have had */
                        /*   since the cells and lists were built (moved by */
                        /*   sph_drift); 0 = none.  The build then requires */
                        /*   gamma*h + 2*skin <= C_l for home particles.    */
                        /*   sph_density_all widens the window in a neighbour */
                        /*   cell c by 2*cells->cell_dx[c] (the per-cell    */
                        /*   max_dx of P:102); the other density calls by   */
                        /*   4*skin.                       */
} sph_grid;

/* Per-direction sorted lists ("index" of P:92).  For cell c and direction
 * d, order[d * capacity + cell_start[c] + k] is the IN-CELL index (0 ..
 * n_c - 1, uint16: SPH_MAX_CELL bounds the occupancy) of the particle of
 * rank k when the cell's particles are ascending in the projection of their
 * position on the unit axis of d, key = (x - cell corner) . d/|d| computed in
 * fp64; keys closer than 2^-25 * 2 sqrt(3) C_l (far below the window margin
 * delta) may be ordered by input index instead.  The projected distances
 * ("dist" of P:92) are not stored: the density sweeps recompute projected
 * separations (x_j - x_i) . d from exact coordinate differences
 * (DESIGN.md §4.2), so a list costs 2 bytes per particle and direction. */
#define SPH_ORDER_BYTES 2

/* Cell-sorted particle storage (caller-allocated device arrays).
 *   cell_start[ncell + 1]   first slot of each local cell (written by build)
 *   xyzh[4 * capacity]      x, y, z, h  in cell order (float4 per particle)
 *   vm[4 * capacity]        vx, vy, vz, m in cell order
 *   perm[capacity]          slot -> input index
 *   cell_hmax[ncell]        max h in each cell
 *   slot_cell[capacity]     local cell of each slot (written by build)
 *   cell_nhome[ncell]       home particles of each cell; they occupy the first
 *                           cell_nhome[c] slots of the cell (written by build)
 *   order[SPH_NDIR * capacity] sorted lists (uint16 in-cell indices):
 *                           direction d, cell c at
 *                           order[d * capacity + cell_start[c] ...];
 *                           16-byte aligned, readable up to the next 16-byte
 *                           boundary past its end (the density kernel reads
 *                           it in aligned 16-byte words; cudaMalloc
 *                           allocations satisfy this)
 *   disp[capacity]          list reuse: per slot, an upper bound of
 *                           |x - x_build| (0 after sph_build_cells,
 *                           accumulated by sph_drift)
 *   cell_dx[ncell]          per cell, the largest disp of its particles: the
 *                           paper's max_dx (0 after a build); sph_density_all
 *                           widens a window in neighbour cell c by 2*cell_dx[c]
 * n is written by sph_build_cells: the inputs it was given (owned + ghosts), an
 * upper bound of the stored particles; the exact stored count is
 * cell_start[ncell] (rejected inputs, e.g. ghosts outside the ghost planes,
 * get no slot).  16-byte alignment
 * is required for xyzh and vm. */
typedef struct sph_cells {
    int64_t capacity;
    int64_t n;
    int32_t *cell_start;
    float *xyzh;
    float *vm;
    int32_t *perm;
    float *cell_hmax;
    uint16_t *order;
    int32_t *slot_cell;
    int32_t *cell_nhome;
    float *disp;
    float *cell_dx;
} sph_cells;

/* Outputs, each an array of n_out elements indexed by INPUT index (only
 * owned particles are written); curl_v is [3][n_out] (x, y, z planes). */
typedef struct sph_out {
    int64_t n_out;
    float *rho, *rho_dh, *wcount, *wcount_dh, *div_v, *curl_v;
    int32_t *nngb;
} sph_out;

/* Optional device-side counters (pass NULL to skip; counting costs time).
 * Index k: 0 self cell, 1 face, 2 edge, 3 corner neighbour cells.
 * cand = candidate distance evaluations (the pseudo-Verlet windows of Code 2,
 * P:94-100), hits = in-range pairs, band = candidate pairs with
 * |r^2 - H_i^2| < 1e-6 H_i^2 evaluated in fp32 (BASELINE north_star: pairs in
 * that band are "counted and reported"; sph_density_all's engines count it,
 * the accumulating API kernels leave it 0). */
typedef struct sph_stats {
    unsigned long long cand[4];
    unsigned long long hits[4];
    unsigned long long band;
} sph_stats;

/* Number of local cells of `grid` (< 0 on a bad grid). */
int64_t sph_ncell(const sph_grid *grid);

/* Bytes of workspace the calls need for up to n_total stored particles. */
size_t sph_workspace_bytes(const sph_grid *grid, int64_t n_total);

/* Bin particles into cells and write the cell-sorted SoA
 * arrays, perm, cell_start, cell_hmax, cell_nhome and cells->n =
 * n_own + n_ghost.  Within a cell, home particles come first, each group in
 * input order.
 * Inputs xyzh_in/vm_in hold n_own owned particles followed by n_ghost
 * ghost particles (float4 each, device).  Owned particles must lie in the
 * rank's owned planes (n_ghost > 0 needs ghost_x = 1); ghosts outside the
 * ghost planes are dropped (not stored: a finer level grid keeps only its
 * own ghost planes of the coarse ghosts), so cells->n is an upper bound and
 * cell_start[ncell] the stored count.  Resets the status word, then reports SPH_EDOMAIN /
 * SPH_EH_RANGE / SPH_ECAPACITY through it.  Cell bins use fp64:
 * ix = floor(x * nc / box), clamped to [0, nc-1]. */
int sph_build_cells(const sph_grid *grid, int64_t n_own, int64_t n_ghost, const float *xyzh_in,
                    const float *vm_in, sph_cells *cells, void *ws, size_t ws_bytes, void *stream);

/* Sort every cell of [cell_begin, cell_end) along the 13 directions (P:92,
 * P:102): fills cells->order for those cells.  cell_end = -1 means all.
 * With a home range (level pass) only cells within one cell of a home
 * particle are sorted: the others' lists are never read by sph_density_all. */
int sph_sort_cells(const sph_grid *grid, const sph_cells *cells, int64_t cell_begin, int64_t cell_end,
                   void *ws, size_t ws_bytes, void *stream);

/* sph_build_cells followed by sph_sort_cells over all cells, with identical
 * results (P:65, P:80 binning; P:92, P:102 the 13 sorted lists) and the same
 * arguments, errors and workspace as sph_build_cells.  On a single grid
 * (h_home_max <= 0) the lists of cells of up to 32 particles are computed
 * inside the build's in-cell placement pass (the records are already in the
 * warp), so the memory-bound placement and the issue-bound ranking overlap;
 * level grids run the two calls unfused.  (ABI v7) */
int sph_build_sort_cells(const sph_grid *grid, int64_t n_own, int64_t n_ghost, const float *xyzh_in,
                         const float *vm_in, sph_cells *cells, void *ws, size_t ws_bytes, void *stream);

/* (sph_density_self / sph_density_pair treat every particle of a listed cell
 * as home, whatever the grid's home range.)
 * Self-cell interactions of each listed cell (device int32 list): every
 * ordered pair i != j in the cell plus the self term of i.  ACCUMULATES
 * with atomics into acc (caller zeroes it first): rho, wcount, rho_dh,
 * wcount_dh and nngb receive their final contributions, div_v and curl_v
 * receive rho-weighted sums (rho*div, rho*curl); see sph_density_finalize. */
int sph_density_self(const sph_grid *grid, const sph_cells *cells, const int32_t *cell_list, int64_t ncells_list,
                     sph_out *acc, sph_stats *stats, void *ws, size_t ws_bytes, void *stream);

/* One-sided pseudo-Verlet pair sweeps: for each
 * device pair (ci, cj) of `pairs` ([npairs][2] int32), particles of ci
 * gather from cj, which must be one of the 26 neighbours of ci.  One CTA
 * per cell pair; accumulates like sph_density_self.  The paper's symmetric
 * pair is the two calls (ci, cj) and (cj, ci). */
int sph_density_pair(const sph_grid *grid, const sph_cells *cells, const int32_t *pairs, int64_t npairs,
                     sph_out *acc, sph_stats *stats, void *ws, size_t ws_bytes, void *stream);

/* Symmetric pair sweeps: for each device pair
 * (ci, cj) of `pairs` ([npairs][2] int32, cj one of the 26 neighbours of
 * ci, each unordered pair listed once), every candidate distance of the
 * pair is evaluated once and BOTH particles accumulate: i when r < H_i, j
 * when r < H_j (the window in cj's list uses max(H_i, gamma * hmax(cj)) +
 * delta).  Equals sph_density_pair on (ci, cj) plus (cj, ci) within fp32
 * summation order; accumulates like sph_density_self (atomics; finalize
 * with sph_density_finalize).  j in a ghost cell (slabs) is not updated. */
int sph_density_pair_sym(const sph_grid *grid, const sph_cells *cells, const int32_t *pairs, int64_t npairs,
                         sph_out *acc, sph_stats *stats, void *ws, size_t ws_bytes, void *stream);

/* The symmetric sweep over the whole pass ("computing interactions
 * symmetrically"): every unordered candidate pair is
 * evaluated once and both particles accumulate, with the ownership made
 * conflict-free by colouring instead of atomics: the self cells first, then
 * for each of the 13 directions d and each colour of d's first nonzero axis
 * (parity, a third colour for the last cell of an odd periodic axis) one
 * launch over the pairs (c, c + d) of that colour -- two pairs of one
 * direction share a cell only if their cells are neighbours on that axis,
 * so a launch writes disjoint particles (plain read-modify-writes into
 * per-slot accumulators in the workspace, merged into the outputs at the
 * end; each j sums its hits in ascending i: deterministic; a j hit by more
 * than 32 i of one pair falls back to an atomic add).  Outputs final (as
 * sph_density_all), zeroed first.  Same cells/workspace contract as
 * sph_density_all (the workspace's record regions hold the phase pair lists
 * and the accumulators). */
int sph_density_all_sym(const sph_grid *grid, const sph_cells *cells, sph_out *out, sph_stats *stats, void *ws,
                        size_t ws_bytes, void *stream);

/* div_v /= rho and curl_v /= rho for the first n elements (after the self
 * and pair calls). */
int sph_density_finalize(sph_out *acc, int64_t n, void *stream);

/* The fused hot path: every owned HOME particle gathers from its own cell
 * and the 26 neighbour cells with pseudo-Verlet windows, one writer per
 * particle, no atomics, deterministic; writes FINAL values in input order
 * (outputs of non-home particles are left untouched: a level pass). */
int sph_density_all(const sph_grid *grid, const sph_cells *cells, sph_out *out, sph_stats *stats, void *ws,
                    size_t ws_bytes, void *stream);

/* Synchronises `stream`, returns the status word's error code (SPH_OK if
 * none), or SPH_ECUDA if the stream reports a CUDA error. */
int sph_status(void *ws, void *stream);

/* Clears the status word (asynchronous). */
int sph_status_reset(void *ws, void *stream);

/* Static description of an error code (the last CUDA error text for
 * SPH_ECUDA). */
const char *sph_strerror(int code);

/* List reuse ("max_dx"): move every stored
 * particle of `cells` by its velocity, x <- fp32(x + fp32(v * dt)) per
 * component (two roundings), keeping cells, order and lists as they are.
 * Each slot's disp grows by the norm of its stored increment (rounded up),
 * so disp bounds |x - x_build|; cell_dx[c] becomes the largest disp of cell
 * c (the paper's max_dx).  Positions may leave [0, box) by up to the skin.
 * If max_disp (device float, caller-initialised) is not NULL it receives
 * the largest disp (atomic max).  The caller rebuilds (sph_gather_positions,
 * sph_build_cells, sph_sort_cells) before it exceeds the grid's skin; the
 * density calls on the same cells are then exact. */
int sph_drift(const sph_grid *grid, sph_cells *cells, float dt, float *max_disp, void *stream);

/* The stored (possibly drifted) positions and h back in INPUT order,
 * xyzh_out[4 * n_out] (device, 16-byte aligned), every coordinate wrapped
 * into [0, box): the input of the next sph_build_cells when a reuse loop
 * rebuilds.  Slots whose input index is >= n_out (ghosts)
 * are skipped. */
int sph_gather_positions(const sph_grid *grid, const sph_cells *cells, float *xyzh_out, int64_t n_out,
                         void *stream);

/* Ghost exchange helper (x-slabs): after a fixed-capacity
 * exchange, rows [counts[k], cap) of received block k (k = 0, 1; block k at
 * xyzh/vm + 4 * k * cap floats, device, 16-byte aligned) become the "dead"
 * particle (dead_xyzh, dead_vm: 4 floats each, host values passed by value
 * as arrays): a position in the receiver's own middle plane, which every
 * level grid's sph_build_cells drops as a ghost outside its ghost planes.
 * counts: device int64[2], read on the device (no host synchronisation). */
int sph_mask_ghost_rows(float *xyzh, float *vm, int64_t cap, const int64_t *counts, const float dead_xyzh[4],
                        const float dead_vm[4], void *stream);

/* max_i |v_i| (fp64 norms of the fp32 velocities vm[4 * i .. + 2], device,
 * 16-byte aligned) into out (device double): the speed bound of a list-reuse
 * loop's displacement check.  0 for n = 0. */
int sph_max_speed(const float *vm, int64_t n, double *out, void *stream);

/* Slab migration on a list-reuse rebuild: a stable three-way
 * partition of the owned particles (xyzh/vm float4, gid int64; device, n;
 * positions already wrapped into the box, in ascending gid) by x plane --
 * list "lo": the left neighbour's last plane x_lo - 1 (mod nc), list "hi":
 * the right neighbour's first plane x_hi (mod nc), list "keep": the rest --
 * each in input order, into the caller's buffers (capacities cap_*).
 * counts: device int64[3] (lo, hi, keep).  A list longer than its capacity
 * sets SPH_ECAPACITY in the status word (the copy is truncated).  Planes by
 * the binning rule of sph_build_cells.  Workspace as for sph_build_cells
 * with n_total >= n. */
int sph_partition_migrants(const sph_grid *grid, int64_t n, const float *xyzh, const float *vm, const int64_t *gid,
                           float *lo_xyzh, float *lo_vm, int64_t *lo_gid, int64_t cap_lo, float *hi_xyzh,
                           float *hi_vm, int64_t *hi_gid, int64_t cap_hi, float *keep_xyzh, float *keep_vm,
                           int64_t *keep_gid, int64_t cap_keep, int64_t *counts, void *ws, size_t ws_bytes,
                           void *stream);

/* Merge of three particle lists (xyzh/vm float4, id int64; device), each
 * ascending in id, ids distinct across the lists, into one ascending list
 * out_* of na + nb + nc particles (must not alias the inputs).  The counts
 * are host values. */
int sph_merge_by_id(int64_t na, const float *a_xyzh, const float *a_vm, const int64_t *a_gid, int64_t nb,
                    const float *b_xyzh, const float *b_vm, const int64_t *b_gid, int64_t nc, const float *c_xyzh,
                    const float *c_vm, const int64_t *c_gid, float *out_xyzh, float *out_vm, int64_t *out_gid,
                    void *stream);

/* Ghost exchange helper (x-slabs): copies the owned
 * particles (xyzh_in/vm_in, n_own, device) whose x plane is the rank's
 * first plane x_lo (list 0) or last plane x_hi - 1 (list 1), in input
 * order, to sel_xyzh/sel_vm (float4 each): list k at [k * cap, k * cap +
 * counts[k]).  counts: device int64[2].  Planes are found by the binning
 * rule of sph_build_cells.  A list longer than cap sets SPH_ECAPACITY in the
 * status word (the copy is truncated).  Workspace as for sph_build_cells
 * with n_total >= n_own. */
int sph_select_planes(const sph_grid *grid, int64_t n_own, const float *xyzh_in, const float *vm_in,
                      float *sel_xyzh, float *sel_vm, int64_t cap, int64_t *counts, void *ws, size_t ws_bytes,
                      void *stream);

/* SPH_ABI_VERSION of the loaded library. */
int sph_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PVSPH_SPH_H */
