/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the SIMP
 * mesh-independency filter of Gupta et al., "A 55-line code for large-scale
 * parallel topology optimization in 2D and 3D" (arXiv 2012.08208).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (libtopofilt, paper_2012_08208_b200/) never links, imports or calls it, and it
 * shares no code, header, table or helper with the CUDA path.
 *
 * Single-threaded C99, compiled with -O2 -ffp-contract=off (no FMA contraction,
 * no fast-math) so every expression below rounds exactly as written.
 *
 * What it computes (the plain definition, sec. 3.2.2 and 4.5):
 *   Weight (Eq. filter_cond; listing PAPER.md:442-445):
 *       W_ij = max(0, rmin - |c_i - c_j|),  stored for pairs with d^2 < rmin^2,
 *       d^2 = (dx*dx + dy*dy) + dz*dz   (direct difference, fixed order;
 *       DESIGN.md reading R2/R3 -- not the EDM expansion of PAPER.md:393).
 *   Row sums (listing PAPER.md:445, distance_sum = distance_mat.sum(1)):
 *       Hs_i = sum_j W_ij, accumulated in ascending j.
 *   Sensitivity filter (Eq. filter, Eq. filter_mat PAPER.md:401-439,
 *   listing PAPER.md:447, plus the max(1e-3, x) floor of BASELINE.json north_star):
 *       out_i = (sum_j W_ij * (x_j*dc_j)) / (Hs_i * max(1e-3, x_i))
 *   Density filter (BASELINE.json north_star only; not in the paper -- parity
 *   for its *definition* is unpinned by the paper):
 *       out_i = (sum_j W_ij * x_j) / Hs_i
 *
 * Functions:
 *   O1 or_bf_*          brute force over all j for each i (N^2 tests).
 *   O2 or_cl_*          plain uniform cell list with bin side s >= rmin*(1+1e-6),
 *                       3^dim neighbour bins, identical pair test and formula,
 *                       candidates sorted by j before accumulation.
 *   O3 or_apply_*       row loops of the two filters over a CSR.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ pair test */

/* d^2 between centroid i and j, fixed order (dx*dx + dy*dy) + dz*dz. */
static double pair_d2(const double *c, int dim, int64_t i, int64_t j)
{
    double dx = c[i * dim + 0] - c[j * dim + 0];
    double dy = c[i * dim + 1] - c[j * dim + 1];
    double d2 = dx * dx + dy * dy;
    if (dim == 3) {
        double dz = c[i * dim + 2] - c[j * dim + 2];
        d2 = d2 + dz * dz;
    }
    return d2;
}

/* W = max(0, rmin - sqrt(d2))  (Eq. filter_cond; listing clips negatives) */
static double weight(double rmin, double d2)
{
    double w = rmin - sqrt(d2);
    if (w < 0.0) w = 0.0;
    return w;
}

/* ------------------------------------------------------------------ O1 brute force */

/* rowptr[0..n] of the brute-force CSR. Returns nnz. */
int64_t or_bf_rowptr(const double *c, int64_t n, int dim, double rmin, int64_t *rowptr)
{
    double r2 = rmin * rmin;
    rowptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t cnt = 0;
        for (int64_t j = 0; j < n; ++j)
            if (pair_d2(c, dim, i, j) < r2) ++cnt;
        rowptr[i + 1] = rowptr[i] + cnt;
    }
    return rowptr[n];
}

/* Fill cols/vals (ascending j) and Hs given rowptr from or_bf_rowptr. */
void or_bf_fill(const double *c, int64_t n, int dim, double rmin, const int64_t *rowptr,
                int32_t *cols, double *vals, double *hs)
{
    double r2 = rmin * rmin;
    for (int64_t i = 0; i < n; ++i) {
        int64_t k = rowptr[i];
        double sum = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            double d2 = pair_d2(c, dim, i, j);
            if (d2 < r2) {
                double w = weight(rmin, d2);
                cols[k] = (int32_t)j;
                vals[k] = w;
                sum = sum + w;
                ++k;
            }
        }
        hs[i] = sum;
    }
}

/* O1 on a subset of rows ("random rows of configs 3/4/5 over all N"): output row r
 * is global row rows[r], tested against all n points in ascending j -- the same loop as
 * or_bf_rowptr / or_bf_fill restricted to the listed rows. */
int64_t or_bf_rows_rowptr(const double *c, int64_t n, int dim, double rmin, const int64_t *rows, int64_t m,
                          int64_t *rowptr)
{
    double r2 = rmin * rmin;
    rowptr[0] = 0;
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = rows[r], cnt = 0;
        for (int64_t j = 0; j < n; ++j)
            if (pair_d2(c, dim, i, j) < r2) ++cnt;
        rowptr[r + 1] = rowptr[r] + cnt;
    }
    return rowptr[m];
}

void or_bf_rows_fill(const double *c, int64_t n, int dim, double rmin, const int64_t *rows, int64_t m,
                     const int64_t *rowptr, int32_t *cols, double *vals, double *hs)
{
    double r2 = rmin * rmin;
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = rows[r], k = rowptr[r];
        double sum = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            double d2 = pair_d2(c, dim, i, j);
            if (d2 < r2) {
                double w = weight(rmin, d2);
                cols[k] = (int32_t)j;
                vals[k] = w;
                sum = sum + w;
                ++k;
            }
        }
        hs[r] = sum;
    }
}

/* ------------------------------------------------------------------ O2 cell list */

typedef struct {
    const double *c;
    int64_t n;
    int dim;
    double rmin, s;
    double lo[3];
    int64_t nb[3];       /* bins per dimension (nb[2] = 1 in 2D) */
    int64_t nbins;
    int64_t *start;      /* [nbins+1] first slot of each bin in `pts` */
    int64_t *pts;        /* point ids grouped by bin, ascending id inside a bin */
    int64_t *bin_of;     /* bin index of each point */
    int64_t *bin3;       /* per point: 3 integer bin coordinates */
} or_cl;

static int64_t bin_coord(double v, double lo, double s, int64_t nb)
{
    int64_t k = (int64_t)floor((v - lo) / s);
    if (k < 0) k = 0;
    if (k > nb - 1) k = nb - 1;
    return k;
}

/* Build a cell list with bin side s = rmin*(1+1e-6)*bin_factor (bin_factor >= 1).
 * The side is doubled while the bin count exceeds 8n+64 (still >= rmin).
 * Completeness of the 3^dim search for s >= rmin*(1+1e-6): DESIGN.md reading R5. */
or_cl *or_cl_create(const double *c, int64_t n, int dim, double rmin, double bin_factor)
{
    if (n < 1 || (dim != 2 && dim != 3) || !(rmin > 0.0) || !(bin_factor >= 1.0)) return NULL;
    or_cl *h = (or_cl *)calloc(1, sizeof(or_cl));
    h->c = c; h->n = n; h->dim = dim; h->rmin = rmin;
    double hi[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) { h->lo[d] = c[d]; hi[d] = c[d]; }
    for (int64_t i = 0; i < n; ++i)
        for (int d = 0; d < dim; ++d) {
            double v = c[i * dim + d];
            if (v < h->lo[d]) h->lo[d] = v;
            if (v > hi[d]) hi[d] = v;
        }
    h->s = rmin * (1.0 + 1e-6) * bin_factor;
    for (;;) {
        double total = 1.0;
        for (int d = 0; d < 3; ++d) h->nb[d] = 1;
        for (int d = 0; d < dim; ++d) {
            h->nb[d] = (int64_t)floor((hi[d] - h->lo[d]) / h->s) + 1;
            total *= (double)h->nb[d];
        }
        if (total <= 8.0 * (double)n + 64.0) break;
        h->s *= 2.0;
    }
    h->nbins = h->nb[0] * h->nb[1] * h->nb[2];
    h->start = (int64_t *)calloc((size_t)h->nbins + 1, sizeof(int64_t));
    h->pts = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    h->bin_of = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    h->bin3 = (int64_t *)calloc((size_t)n * 3, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        int64_t k[3] = {0, 0, 0};
        for (int d = 0; d < dim; ++d) k[d] = bin_coord(c[i * dim + d], h->lo[d], h->s, h->nb[d]);
        for (int d = 0; d < 3; ++d) h->bin3[i * 3 + d] = k[d];
        h->bin_of[i] = (k[2] * h->nb[1] + k[1]) * h->nb[0] + k[0];
        h->start[h->bin_of[i] + 1] += 1;
    }
    for (int64_t b = 0; b < h->nbins; ++b) h->start[b + 1] += h->start[b];
    int64_t *fillpos = (int64_t *)malloc((size_t)h->nbins * sizeof(int64_t));
    memcpy(fillpos, h->start, (size_t)h->nbins * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) h->pts[fillpos[h->bin_of[i]]++] = i; /* ascending i */
    free(fillpos);
    return h;
}

void or_cl_free(or_cl *h)
{
    if (!h) return;
    free(h->start); free(h->pts); free(h->bin_of); free(h->bin3); free(h);
}

double or_cl_binside(const or_cl *h) { return h->s; }
int64_t or_cl_nbins(const or_cl *h) { return h->nbins; }

static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* Accepted columns of row i, ascending. `buf` must hold n entries. Returns count. */
static int64_t cl_row_cols(const or_cl *h, int64_t i, int64_t *buf)
{
    double r2 = h->rmin * h->rmin;
    int64_t cnt = 0;
    int64_t k0 = h->bin3[i * 3 + 0], k1 = h->bin3[i * 3 + 1], k2 = h->bin3[i * 3 + 2];
    int64_t zlo = (h->dim == 3) ? -1 : 0, zhi = (h->dim == 3) ? 1 : 0;
    for (int64_t dz = zlo; dz <= zhi; ++dz) {
        int64_t bz = k2 + dz;
        if (bz < 0 || bz >= h->nb[2]) continue;
        for (int64_t dy = -1; dy <= 1; ++dy) {
            int64_t by = k1 + dy;
            if (by < 0 || by >= h->nb[1]) continue;
            for (int64_t dx = -1; dx <= 1; ++dx) {
                int64_t bx = k0 + dx;
                if (bx < 0 || bx >= h->nb[0]) continue;
                int64_t b = (bz * h->nb[1] + by) * h->nb[0] + bx;
                for (int64_t p = h->start[b]; p < h->start[b + 1]; ++p) {
                    int64_t j = h->pts[p];
                    if (pair_d2(h->c, h->dim, i, j) < r2) buf[cnt++] = j;
                }
            }
        }
    }
    qsort(buf, (size_t)cnt, sizeof(int64_t), cmp_i64);
    return cnt;
}

/* Row lengths for rows[0..m-1] (rows == NULL means all n rows, m = n);
 * rowptr[0..m]. Returns total nnz. */
int64_t or_cl_rowptr(const or_cl *h, const int64_t *rows, int64_t m, int64_t *rowptr)
{
    int64_t *buf = (int64_t *)malloc((size_t)h->n * sizeof(int64_t));
    rowptr[0] = 0;
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = rows ? rows[r] : r;
        rowptr[r + 1] = rowptr[r] + cl_row_cols(h, i, buf);
    }
    free(buf);
    return rowptr[m];
}

/* cols (ascending), vals and hs (accumulated in ascending j) for rows[0..m-1]. */
void or_cl_fill(const or_cl *h, const int64_t *rows, int64_t m, const int64_t *rowptr,
                int32_t *cols, double *vals, double *hs)
{
    int64_t *buf = (int64_t *)malloc((size_t)h->n * sizeof(int64_t));
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = rows ? rows[r] : r;
        int64_t cnt = cl_row_cols(h, i, buf);
        int64_t k = rowptr[r];
        double sum = 0.0;
        for (int64_t t = 0; t < cnt; ++t) {
            double w = weight(h->rmin, pair_d2(h->c, h->dim, i, buf[t]));
            cols[k + t] = (int32_t)buf[t];
            vals[k + t] = w;
            sum = sum + w;
        }
        hs[r] = sum;
    }
    free(buf);
}

/* ------------------------------------------------------------------ O3 apply */

/* Sensitivity filter (Eq. filter_mat / listing PAPER.md:447 with the max(1e-3,x)
 * floor): one division by the product Hs_i * max(1e-3, x_i), as in
 * np.divide(num, np.multiply(d, distance_sum)).
 * rows[r] is the global index of CSR row r (NULL: identity). */
void or_apply_sensitivity(int64_t m, const int64_t *rows, const int64_t *rowptr,
                          const int32_t *cols, const double *vals, const double *hs,
                          const double *x, const double *dc, double *out)
{
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = rows ? rows[r] : r;
        double acc = 0.0;
        for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
            int64_t j = cols[k];
            double t = x[j] * dc[j];
            acc = acc + vals[k] * t;
        }
        double xi = x[i];
        double floor_x = fmax(1e-3, xi);
        double den = hs[r] * floor_x;
        out[r] = acc / den;
    }
}

/* Density filter x~ = Hx/Hs (BASELINE.json north_star). */
void or_apply_density(int64_t m, const int64_t *rows, const int64_t *rowptr,
                      const int32_t *cols, const double *vals, const double *hs,
                      const double *x, double *out)
{
    (void)rows;
    for (int64_t r = 0; r < m; ++r) {
        double acc = 0.0;
        for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) acc = acc + vals[k] * x[cols[k]];
        out[r] = acc / hs[r];
    }
}

/* ------------------------------------------------------------------ NEXT-1: OC update
 *
 * Optimality-criteria update with bisection on the Lagrange multiplier (Eq. update,
 * PAPER.md:218-228; bisection PAPER.md:229-234; listing PAPER.md:380-385):
 *
 *   l1, l2, move = 0, 100000, 0.2
 *   while l2 - l1 > 1e-4:
 *       l_mid = 0.5 * (l2 + l1)
 *       density_new = max(0.001, max(d - move, min(1.0, min(d + move, d * sqrt(-dc / l_mid)))))
 *       l1, l2 = (l_mid, l2) if sum(density_new) - volfrac * N > 0 else (l1, l_mid)
 *
 * Reading R15: the branch compares the EXACT sum with volfrac*N. Every
 * density_new lies in [0.001, 1], so it is an integer multiple of 2^-62; the sum is
 * accumulated exactly as 128-bit integers in units of 2^-62 (order-independent), and the
 * target volfrac*N (one fp64 rounding, as in the listing) is converted exactly.
 * Preconditions (as for the listing): d in [0, 1], dc <= 0 (filtered compliance sensitivities).
 * max/min propagate NaN like numpy's maximum/minimum. Returns the number of iterations;
 * *lmid_out = the last l_mid evaluated; xnew = density_new at that l_mid.
 */
static double np_max(double a, double b) { return (a != a || b != b) ? (a != a ? a : b) : (a > b ? a : b); }
static double np_min(double a, double b) { return (a != a || b != b) ? (a != a ? a : b) : (a < b ? a : b); }

static double oc_value(double d, double dc, double lmid, double move)
{
    double s = sqrt(-dc / lmid);
    return np_max(0.001, np_max(d - move, np_min(1.0, np_min(d + move, d * s))));
}

/* exact value*2^62 as an integer (value in [0.001, 1], a multiple of 2^-62) */
static unsigned __int128 oc_units(double v) { return (unsigned __int128)ldexp(v, 62); }

/* Reading R23: the listing's loop runs while l2 - l1 > tol; when tol is below the fp64
 * spacing near l_mid, l_mid rounds to l1 or l2 and the bracket stops shrinking, so the loop also
 * stops there (and after 4096 steps). *flags_out: bit 0 = every step moved l1 up (the volume still
 * exceeds the target at l2: bracket exhausted), bit 1 = stopped without reaching tol. */
int or_oc_update(int64_t n, const double *d, const double *dc, double volfrac, double move,
                 double l1, double l2, double tol, double *xnew, double *lmid_out, int *flags_out)
{
    const double target = volfrac * (double)n;
    const unsigned __int128 T = oc_units(target);  /* target*2^62 is an integer for target >= 2^-10 */
    int iters = 0, all_up = 1, stalled = 0;
    double lmid = 0.5 * (l2 + l1);
    while (l2 - l1 > tol) {
        lmid = 0.5 * (l2 + l1);
        if (lmid == l1 || lmid == l2 || iters >= 4096) { stalled = 1; break; }
        unsigned __int128 S = 0;
        int nan = 0;
        for (int64_t i = 0; i < n; ++i) {
            double v = oc_value(d[i], dc[i], lmid, move);
            if (v != v) nan = 1;          /* numpy: NaN sum, NaN > 0 is False */
            else S += oc_units(v);
        }
        if (!nan && S > T) l1 = lmid;
        else { l2 = lmid; all_up = 0; }
        ++iters;
    }
    for (int64_t i = 0; i < n; ++i) xnew[i] = oc_value(d[i], dc[i], lmid, move);
    *lmid_out = lmid;
    if (flags_out) *flags_out = ((iters > 0 && all_up) ? 1 : 0) | (stalled ? 2 : 0);
    return iters;
}

/* NEXT-2: compliance sensitivity (listing PAPER.md:376, numpy order):
 *   sensitivity = -penal * density ** (penal - 1) * U   ==  ((-penal) * pow(x, penal-1)) * U */
void or_compliance_sensitivity(int64_t n, const double *x, const double *U, double penal, double *dc)
{
    for (int64_t i = 0; i < n; ++i) dc[i] = (-penal * pow(x[i], penal - 1.0)) * U[i];
}
