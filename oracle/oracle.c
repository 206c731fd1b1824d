/*
 * oracle/oracle.c -- CPU fp64 oracle for the SPH density loop of
 * Willis et al., "An Efficient SIMD Implementation of Pseudo-Verlet Lists for
 * Neighbour Interactions in Particle-Based Codes" (arXiv:1804.06231).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_1804_06231_b200/csrc), and never includes or links it.
 *
 * What it computes is the plain definition (DESIGN.md §2 readings R1-R8):
 *   for every target particle i, with H_i = gamma*h_i and the strict
 *   predicate  j in N_i  <=>  j != i  and  r_ij^2 < H_i^2     (PAPER.md l.86,
 *   l.98, l.185 "r < h";  l.116 "||p_i - p_j|| < h_i^(a)", gather on h_i),
 *   minimum-image separations in the periodic box,
 *     rho_i       = m_i W(0,h_i) + sum_j m_j W(r_ij,h_i)
 *     wcount_i    =     W(0,h_i) + sum_j     W(r_ij,h_i)
 *     rho_dh_i    = m_i dW/dh(0) + sum_j m_j dW/dh(r_ij,h_i)
 *     wcount_dh_i =     dW/dh(0) + sum_j     dW/dh(r_ij,h_i)
 *     div_i       = -(1/rho_i) sum_j m_j (v_ij . x_ij) (dW/dr)/r_ij
 *     curl_i      =  (1/rho_i) sum_j m_j (v_ij x x_ij) (dW/dr)/r_ij
 *     nngb_i      = |N_i|
 *   with the M4 cubic spline of support H = gamma*h (reading R1):
 *     W(r,h) = (16/pi) H^-3 w(r/H),  w(x) = 3x^3 - 3x^2 + 1/2  (x < 1/2)
 *                                          = (1-x)^3           (1/2 <= x < 1)
 *                                          = 0                 (x >= 1).
 *   Scales for the signed outputs (readings R13, R14): A = sum of |terms|,
 *   C = sum of |terms| * (|x w''(x)/w'(x)| + 1), the first-order change of
 *   the div/curl sums under a unit relative perturbation of every x = r/H.
 *   The neighbour list of each i is sorted by j and summed in that order in
 *   fp64 (reading R6), so the brute-force (O1) and cell-list (O2) variants
 *   give bitwise identical results.
 *
 * Two searches, differing only in how candidates j are enumerated:
 *   O1 oracle_bruteforce : all j (the naive O(N^2) loop);
 *   O2 oracle_celllist   : cells of edge C_l = L/nc >= H_max, candidates from
 *                          the 27 surrounding cells, every particle of every
 *                          cell tested (Code 1 l.82-88).
 * plus
 *   oracle_pv_counts     : the pseudo-Verlet candidate count of Code 2
 *                           evaluated as a count per
 *                          orientation (self/face/edge/corner), with the
 *                          projections onto the unit cell-pair axis in fp64;
 *   oracle_bin_cells     : the cell of every particle and the stable
 *                          cell-sorted order ("particles
 *                          corresponding to each cell are stored together");
 *   oracle_cell_keys     : the cell-local projections onto the 13 sort axes
 *                          (PAPER.md l.92, l.102).
 *
 * Parity pins: tests/test_oracle_pins.py (closed forms, the worked example
 * in tests/golden/, lattice sums, invariances, the paper's 16 % / 68 %).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_NOUT 16
enum {
    O_RHO = 0, O_WCOUNT, O_RHO_DH, O_WCOUNT_DH, O_DIV, O_CURLX, O_CURLY, O_CURLZ,
    O_NNGB, O_BAND, O_A_RHODH, O_A_WDH, O_A_DIV, O_A_CURL, O_C_DIV, O_C_CURL
};

static const double ORC_PI = 3.14159265358979323846264338327950288;
static const double ORC_BAND = 1e-6;   /* band: |r^2 - H^2| < 1e-6 H^2 (BASELINE north_star) */

int oracle_nout(void) { return ORC_NOUT; }

/* ---- kernel (reading R1) ------------------------------------------------ */
static double w_m4(double x)
{
    if (x < 0.5) return 3.0 * x * x * x - 3.0 * x * x + 0.5;
    if (x < 1.0) { double u = 1.0 - x; return u * u * u; }
    return 0.0;
}

static double dw_m4(double x)
{
    if (x < 0.5) return 9.0 * x * x - 6.0 * x;
    if (x < 1.0) { double u = 1.0 - x; return -3.0 * u * u; }
    return 0.0;
}

static double d2w_m4(double x)
{
    if (x < 0.5) return 18.0 * x - 6.0;
    if (x < 1.0) return 6.0 * (1.0 - x);
    return 0.0;
}

/* Condition factor of a gradient term m (v.x_ij) W'(r)/r ~ w'(x) (v . unit vector)
 * under a relative perturbation of x = r/H (reading R14): |x w''/w'| + 1. */
static double kappa_m4(double x)
{
    double dw = dw_m4(x);
    return dw != 0.0 ? fabs(x * d2w_m4(x) / dw) + 1.0 : 1.0;
}

/* W(r,h), dW/dr and dW/dh for support H = gamma*h.
 * W = (16/pi) H^-3 w(x), x = r/H;  dW/dr = (16/pi) H^-4 w'(x);
 * dW/dh = -(16/pi) gamma H^-4 (3 w(x) + x w'(x))   (d/dh at fixed r). */
void oracle_kernel(double r, double h, double gamma, double *W, double *dWdr, double *dWdh)
{
    double H = gamma * h;
    double x = r / H;
    double c3 = 16.0 / (ORC_PI * H * H * H);
    double w = w_m4(x), dw = dw_m4(x);
    *W = c3 * w;
    *dWdr = c3 / H * dw;
    *dWdh = -(c3 * gamma / H) * (3.0 * w + x * dw);
}

/* ---- helpers ------------------------------------------------------------ */
static double min_image(double d, double L)
{
    return d - L * nearbyint(d / L);
}

static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* Sum the outputs of target i over its neighbour list nb[0..k) (ascending j). */
static void accumulate(int64_t i, const float *xyzh, const float *vm, double L, double gamma,
                       const int64_t *nb, int64_t k, int64_t band, double *out)
{
    double xi = xyzh[4 * i + 0], yi = xyzh[4 * i + 1], zi = xyzh[4 * i + 2], hi = xyzh[4 * i + 3];
    double vxi = vm[4 * i + 0], vyi = vm[4 * i + 1], vzi = vm[4 * i + 2], mi = vm[4 * i + 3];
    double W0, dW0, dWh0;
    oracle_kernel(0.0, hi, gamma, &W0, &dW0, &dWh0);
    double rho = mi * W0, wc = W0, rho_dh = mi * dWh0, wc_dh = dWh0;
    double a_rdh = fabs(mi * dWh0), a_wdh = fabs(dWh0);
    double D = 0.0, Rx = 0.0, Ry = 0.0, Rz = 0.0, a_div = 0.0, a_curl = 0.0, c_div = 0.0, c_curl = 0.0;
    for (int64_t q = 0; q < k; ++q) {
        int64_t j = nb[q];
        double dx = min_image(xi - (double)xyzh[4 * j + 0], L);
        double dy = min_image(yi - (double)xyzh[4 * j + 1], L);
        double dz = min_image(zi - (double)xyzh[4 * j + 2], L);
        double r2 = dx * dx + dy * dy + dz * dz;
        double r = sqrt(r2);
        double mj = vm[4 * j + 3];
        double W, dWdr, dWdh;
        oracle_kernel(r, hi, gamma, &W, &dWdr, &dWdh);
        rho += mj * W;
        wc += W;
        rho_dh += mj * dWdh;
        wc_dh += dWdh;
        a_rdh += fabs(mj * dWdh);
        a_wdh += fabs(dWdh);
        if (r2 > 0.0) {                       /* reading R7: gradient term 0 at r = 0 */
            double f = mj * dWdr / r;
            double vx = vxi - (double)vm[4 * j + 0];
            double vy = vyi - (double)vm[4 * j + 1];
            double vz = vzi - (double)vm[4 * j + 2];
            double vdx = vx * dx + vy * dy + vz * dz;
            D += f * vdx;
            Rx += f * (vy * dz - vz * dy);
            Ry += f * (vz * dx - vx * dz);
            Rz += f * (vx * dy - vy * dx);
            a_div += fabs(f * vdx);
            a_curl += fabs(f) * sqrt(vx * vx + vy * vy + vz * vz) * r;
            double kap = kappa_m4(r / (gamma * hi));
            c_div += fabs(f * vdx) * kap;
            c_curl += fabs(f) * sqrt(vx * vx + vy * vy + vz * vz) * r * kap;
        }
    }
    out[O_RHO] = rho;
    out[O_WCOUNT] = wc;
    out[O_RHO_DH] = rho_dh;
    out[O_WCOUNT_DH] = wc_dh;
    out[O_DIV] = -D / rho;
    out[O_CURLX] = Rx / rho;
    out[O_CURLY] = Ry / rho;
    out[O_CURLZ] = Rz / rho;
    out[O_NNGB] = (double)k;
    out[O_BAND] = (double)band;
    out[O_A_RHODH] = a_rdh;
    out[O_A_WDH] = a_wdh;
    out[O_A_DIV] = a_div / rho;
    out[O_A_CURL] = a_curl / rho;
    out[O_C_DIV] = c_div / rho;
    out[O_C_CURL] = c_curl / rho;
}

/* Test candidate j for target i: push to nb if in range, count band. */
static inline void test_pair(int64_t i, int64_t j, const float *xyzh, double L, double xi, double yi,
                             double zi, double H2, int64_t *nb, int64_t *k, int64_t *band)
{
    if (j == i) return;
    double dx = min_image(xi - (double)xyzh[4 * j + 0], L);
    double dy = min_image(yi - (double)xyzh[4 * j + 1], L);
    double dz = min_image(zi - (double)xyzh[4 * j + 2], L);
    double r2 = dx * dx + dy * dy + dz * dz;
    if (fabs(r2 - H2) < ORC_BAND * H2) ++*band;
    if (r2 < H2) nb[(*k)++] = j;
}

static int valid_targets(int64_t n, const int64_t *targets, int64_t nt)
{
    for (int64_t t = 0; t < nt; ++t)
        if (targets[t] < 0 || targets[t] >= n) return 0;
    return 1;
}

/* ---- O1: brute force ----------------------------------------------------- */
/* targets: indices of the particles to evaluate (NULL = all, nt ignored).
 * out: (nt or n) x ORC_NOUT doubles.  Returns 0, or -1 on bad arguments. */
int oracle_bruteforce(int64_t n, const float *xyzh, const float *vm, double L, double gamma,
                      const int64_t *targets, int64_t nt, double *out)
{
    if (n < 0 || !xyzh || !vm || !out || L <= 0.0) return -1;
    if (!targets) nt = n;
    else if (!valid_targets(n, targets, nt)) return -1;
    int err = 0;
#pragma omp parallel
    {
        int64_t *nb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
        if (!nb) {
#pragma omp atomic write
            err = 1;
        }
#pragma omp for schedule(dynamic, 16)
        for (int64_t t = 0; t < nt; ++t) {
            if (!nb) continue;
            int64_t i = targets ? targets[t] : t;
            double xi = xyzh[4 * i], yi = xyzh[4 * i + 1], zi = xyzh[4 * i + 2];
            double H = gamma * (double)xyzh[4 * i + 3];
            double H2 = H * H;
            int64_t k = 0, band = 0;
            for (int64_t j = 0; j < n; ++j)
                test_pair(i, j, xyzh, L, xi, yi, zi, H2, nb, &k, &band);
            accumulate(i, xyzh, vm, L, gamma, nb, k, band, out + (size_t)t * ORC_NOUT);
        }
        free(nb);
    }
    return err ? -2 : 0;
}

/* ---- cell binning (shared by O2 and the pV counts) ---------------------- */
static int64_t cell_coord(double x, int nc, double L)
{
    int64_t c = (int64_t)floor(x * (double)nc / L);
    if (c < 0) c = 0;
    if (c > nc - 1) c = nc - 1;
    return c;
}

/* cell_of[i] = (ix*nc + iy)*nc + iz; order = particles sorted by cell, stable
 * (input order inside a cell); start[ncell+1] = first slot of each cell. */
int oracle_bin_cells(int64_t n, const float *xyzh, double L, int nc, int64_t *cell_of,
                     int64_t *order, int64_t *start)
{
    if (n < 0 || nc < 1 || !xyzh || !cell_of || !order || !start) return -1;
    int64_t ncell = (int64_t)nc * nc * nc;
    for (int64_t c = 0; c <= ncell; ++c) start[c] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t ix = cell_coord(xyzh[4 * i + 0], nc, L);
        int64_t iy = cell_coord(xyzh[4 * i + 1], nc, L);
        int64_t iz = cell_coord(xyzh[4 * i + 2], nc, L);
        cell_of[i] = (ix * nc + iy) * nc + iz;
        start[cell_of[i] + 1]++;
    }
    for (int64_t c = 0; c < ncell; ++c) start[c + 1] += start[c];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncell + 1));
    if (!fill) return -2;
    memcpy(fill, start, sizeof(int64_t) * (size_t)(ncell + 1));
    for (int64_t i = 0; i < n; ++i) order[fill[cell_of[i]]++] = i;
    free(fill);
    return 0;
}

typedef struct {
    int nc;
    int64_t ncell;
    int64_t *cell_of, *order, *start;
    int64_t maxocc;
} orc_cells;

static int cells_build(orc_cells *c, int64_t n, const float *xyzh, double L, int nc)
{
    c->nc = nc;
    c->ncell = (int64_t)nc * nc * nc;
    c->cell_of = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    c->order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    c->start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(c->ncell + 1));
    if (!c->cell_of || !c->order || !c->start) return -2;
    if (oracle_bin_cells(n, xyzh, L, nc, c->cell_of, c->order, c->start)) return -2;
    c->maxocc = 0;
    for (int64_t q = 0; q < c->ncell; ++q)
        if (c->start[q + 1] - c->start[q] > c->maxocc) c->maxocc = c->start[q + 1] - c->start[q];
    return 0;
}

static void cells_free(orc_cells *c)
{
    free(c->cell_of);
    free(c->order);
    free(c->start);
}

static int64_t wrapi(int64_t a, int nc) { return ((a % nc) + nc) % nc; }

/* ---- O2: plain cell list, Code 1 over the 27-cell block ----------------- */
int oracle_celllist(int64_t n, const float *xyzh, const float *vm, double L, double gamma, int nc,
                    const int64_t *targets, int64_t nt, double *out)
{
    if (n < 0 || !xyzh || !vm || !out || L <= 0.0 || nc < 3) return -1;
    if (!targets) nt = n;
    else if (!valid_targets(n, targets, nt)) return -1;
    orc_cells C;
    if (cells_build(&C, n, xyzh, L, nc)) { cells_free(&C); return -2; }
    int err = 0;
#pragma omp parallel
    {
        int64_t cap = 27 * C.maxocc + 1;
        int64_t *nb = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
        if (!nb) {
#pragma omp atomic write
            err = 1;
        }
#pragma omp for schedule(dynamic, 64)
        for (int64_t t = 0; t < nt; ++t) {
            if (!nb) continue;
            int64_t i = targets ? targets[t] : t;
            double xi = xyzh[4 * i], yi = xyzh[4 * i + 1], zi = xyzh[4 * i + 2];
            double H = gamma * (double)xyzh[4 * i + 3];
            double H2 = H * H;
            int64_t ci = C.cell_of[i];
            int64_t ix = ci / ((int64_t)nc * nc), iy = (ci / nc) % nc, iz = ci % nc;
            int64_t k = 0, band = 0;
            for (int ox = -1; ox <= 1; ++ox)
                for (int oy = -1; oy <= 1; ++oy)
                    for (int oz = -1; oz <= 1; ++oz) {
                        int64_t cj = (wrapi(ix + ox, nc) * nc + wrapi(iy + oy, nc)) * nc + wrapi(iz + oz, nc);
                        for (int64_t s = C.start[cj]; s < C.start[cj + 1]; ++s)
                            test_pair(i, C.order[s], xyzh, L, xi, yi, zi, H2, nb, &k, &band);
                    }
            qsort(nb, (size_t)k, sizeof(int64_t), cmp_i64);
            accumulate(i, xyzh, vm, L, gamma, nb, k, band, out + (size_t)t * ORC_NOUT);
        }
        free(nb);
    }
    cells_free(&C);
    return err ? -2 : 0;
}

/* ---- the 13 sort directions ----------------------------
 * One representative per +/- pair of the 26 neighbour offsets: the one whose
 * first nonzero component is positive, listed in lexicographic order. */
static void orc_direction(int d, int o[3])
{
    int idx = 0;
    for (int a = -1; a <= 1; ++a)
        for (int b = -1; b <= 1; ++b)
            for (int c = -1; c <= 1; ++c) {
                int first = a != 0 ? a : (b != 0 ? b : c);
                if (first <= 0) continue;   /* skips (0,0,0) and the negative half */
                if (idx == d) { o[0] = a; o[1] = b; o[2] = c; return; }
                ++idx;
            }
    o[0] = o[1] = o[2] = 0;
}

int oracle_directions(int *offsets /* 13 x 3 */)
{
    for (int d = 0; d < 13; ++d) orc_direction(d, offsets + 3 * d);
    return 13;
}

/* keys[d*n + i] = (x_i - corner(cell(i))) . o_d/|o_d|, fp64. */
int oracle_cell_keys(int64_t n, const float *xyzh, double L, int nc, double *keys)
{
    if (n < 0 || !xyzh || !keys || nc < 1) return -1;
    double Cl = L / nc;
    for (int d = 0; d < 13; ++d) {
        int o[3];
        orc_direction(d, o);
        double nrm = sqrt((double)(o[0] * o[0] + o[1] * o[1] + o[2] * o[2]));
        for (int64_t i = 0; i < n; ++i) {
            double s = 0.0;
            for (int a = 0; a < 3; ++a) {
                double x = xyzh[4 * i + a];
                double u = x - (double)cell_coord(x, nc, L) * Cl;
                s += u * (double)o[a] / nrm;
            }
            keys[(size_t)d * n + i] = s;
        }
    }
    return 0;
}

/* ---- pseudo-Verlet candidate counts (Code 2 as a count) -----------------
 * For every target i and each of the 26 neighbour cells cj = ci + o:
 *   sep_ij = (x_j^img - x_i) . o/|o|, x_j^img the image of x_j inside the
 *   unwrapped cell ci+o; j is a pV candidate iff sep_ij < H_i + delta
 *   ("dist_b[j] < dist_a[i] + h", with the per-particle h of
 *   l.156 and the margin delta of reading R5).  The self cell contributes its
 *   n_c - 1 other particles.  out per target, 4 kinds (self, face, edge,
 *   corner) x 3 counts (naive candidates, pV candidates, in-range hits):
 *   out[t*12 + kind*3 + {0,1,2}].  Also returns (via *unsafe) the number of
 *   in-range pairs that fall outside their pV window (must be 0). */
int oracle_pv_counts(int64_t n, const float *xyzh, double L, double gamma, int nc, double delta,
                     const int64_t *targets, int64_t nt, int64_t *out, int64_t *unsafe)
{
    if (n < 0 || !xyzh || !out || L <= 0.0 || nc < 3) return -1;
    if (!targets) nt = n;
    else if (!valid_targets(n, targets, nt)) return -1;
    orc_cells C;
    if (cells_build(&C, n, xyzh, L, nc)) { cells_free(&C); return -2; }
    int64_t bad = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : bad)
    for (int64_t t = 0; t < nt; ++t) {
        int64_t i = targets ? targets[t] : t;
        int64_t *o12 = out + (size_t)t * 12;
        for (int q = 0; q < 12; ++q) o12[q] = 0;
        double xi[3] = {xyzh[4 * i], xyzh[4 * i + 1], xyzh[4 * i + 2]};
        double H = gamma * (double)xyzh[4 * i + 3];
        double H2 = H * H;
        int64_t ci = C.cell_of[i];
        int64_t cix[3] = {ci / ((int64_t)nc * nc), (ci / nc) % nc, ci % nc};
        for (int ox = -1; ox <= 1; ++ox)
            for (int oy = -1; oy <= 1; ++oy)
                for (int oz = -1; oz <= 1; ++oz) {
                    int o[3] = {ox, oy, oz};
                    int kind = (ox != 0) + (oy != 0) + (oz != 0);
                    double nrm = sqrt((double)kind);
                    int64_t cj = 0;
                    double shift[3];
                    for (int a = 0; a < 3; ++a) {
                        int64_t u = cix[a] + o[a];
                        shift[a] = u < 0 ? -L : (u >= nc ? L : 0.0);
                        cj = cj * nc + wrapi(u, nc);
                    }
                    for (int64_t s = C.start[cj]; s < C.start[cj + 1]; ++s) {
                        int64_t j = C.order[s];
                        if (j == i) continue;
                        double d[3], r2 = 0.0, sep = 0.0;
                        for (int a = 0; a < 3; ++a) {
                            d[a] = ((double)xyzh[4 * j + a] + shift[a]) - xi[a];
                            r2 += d[a] * d[a];
                            sep += kind ? d[a] * (double)o[a] / nrm : 0.0;
                        }
                        int in_window = kind == 0 ? 1 : (sep < H + delta);
                        int hit = r2 < H2;
                        o12[kind * 3 + 0] += 1;
                        o12[kind * 3 + 1] += in_window;
                        o12[kind * 3 + 2] += hit;
                        if (hit && !in_window) bad += 1;
                    }
                }
    }
    if (unsafe) *unsafe = bad;
    cells_free(&C);
    return 0;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
