/*
 * topofilt.h -- C ABI of libtopofilt, the B200 (sm_100a) mesh-independency filter of
 * Gupta et al., "A 55-line code for large-scale parallel topology optimization in
 * 2D and 3D" (arXiv 2012.08208).
 *
 * The operations (PAPER.md = the paper's LaTeX source):
 *   build   W_ij = max(0, rmin - |c_i - c_j|) over cell-midpoint pairs within rmin
 *           (Eq. filter_cond; listing PAPER.md:442-444) and the
 *           row sums Hs_i = sum_j W_ij. Built once, outside the
 *           optimisation loop. Stored as CSR: pairs with d^2 < rmin^2,
 *           d^2 = (dx*dx + dy*dy) + dz*dz in fp64, no FMA contraction; columns
 *           ascending; weights fp64 (readings R1-R4).
 *   sensitivity filter   dc~_i = (sum_j W_ij x_j dc_j) / (Hs_i * max(1e-3, x_i))
 *           (Eq. filter, Eq. filter_mat PAPER.md:401-439,
 *           listing PAPER.md:447; the max(1e-3, .) floor is BASELINE.json's).
 *   density filter       x~_i = (sum_j W_ij x_j) / Hs_i   (BASELINE.json north_star;
 *           not in the paper).
 *
 * Conventions for every call:
 *   - Array arguments are CUDA DEVICE pointers unless the name ends in _host.
 *     Device arrays are contiguous, 8-byte aligned, and owned by the caller.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Work is stream-ordered; apply calls are asynchronous (no host sync).
 *   - A handle is bound to the CUDA device that was current when it was built; calls on it
 *     must be made with that device current (TF_ERR_INVALID otherwise); tf_free works from any
 *     device. Device pointers must belong to the current device (TF_ERR_INVALID otherwise).
 *   - Every call returns tf_status; nothing throws or aborts across the ABI.
 *     On a non-OK status tf_last_error() returns a thread-local message.
 *   - Sizes: 1 <= n < 2^31 - 1 (int32 column indices); nnz < 2^63.
 */
#ifndef TOPOFILT_H
#define TOPOFILT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TOPOFILT_VERSION 1

#if defined(__GNUC__)
#define TF_API __attribute__((visibility("default")))
#else
#define TF_API
#endif

typedef struct tf_filter_s *tf_filter; /* opaque; owns rowptr/cols/vals/hs; immutable after build */

typedef enum {
    TF_OK = 0,
    TF_ERR_INVALID = 1,  /* bad argument: dim not 2/3, n out of range, rmin <= 0 / NaN / Inf,
                            NULL pointer, host pointer where a device pointer is required,
                            non-finite centroid, out aliasing x or dc */
    TF_ERR_NOMEM = 2,    /* device allocation failed (message states the bytes and nnz) */
    TF_ERR_CUDA = 3,     /* any CUDA runtime error (message carries cudaGetErrorString) */
    TF_ERR_OVERFLOW = 4  /* nnz does not fit the index types */
} tf_status;

/* Borrowed device views of a built filter; valid until tf_free(h). */
typedef struct {
    int64_t n;            /* rows = columns = number of cells */
    int64_t nnz;          /* stored entries (pairs with d^2 < rmin^2, incl. the diagonal) */
    int32_t dim;          /* 2 or 3 */
    double rmin;          /* filter radius */
    const int64_t *rowptr;/* [n+1], rowptr[0] = 0, rowptr[n] = nnz */
    const int32_t *cols;  /* [nnz], strictly ascending inside each row */
    const double *vals;   /* [nnz], W_ij in [0, rmin]; W_ii = rmin */
    const double *hs;     /* [n], Hs_i = sum_j W_ij */
} tf_view;

/* Which build path produced a handle (tf_build_info.path). */
#define TF_PATH_CELL_LIST 0      /* uniform cell list + radix sort + count/fill (any centroids) */
#define TF_PATH_LATTICE_TESTED 1 /* lattice-ordered centroids: per-type candidate table, every
                                    candidate decided by the exact fp64 pair test */
#define TF_PATH_LATTICE_EXACT 2  /* lattice-ordered centroids exactly on a dyadic grid: the pair
                                    test and weight of each table entry are position-independent
                                    and evaluated once on the host (R22) */
#define TF_PATH_DENSE 3          /* ablation (TF_BUILD_DENSE): every pair (i, j) visited, the
                                    paper's own all-pairs method */

/* Build statistics (diagnostics; all host values). For lattice-path builds, bins = cubes per
 * axis, nbins = cubes, max_candidates = the largest per-type table, bin_side = 0. */
typedef struct {
    double bin_side;      /* cell-list bin side s >= rmin*(1+1e-6) */
    int64_t bins[3];      /* bins per dimension (bins[2] = 1 in 2D) */
    int64_t nbins;
    int64_t max_candidates; /* largest 3^dim neighbourhood (points) of any bin */
    int64_t large_rows;   /* rows whose bin neighbourhood exceeded the shared-memory path
                             (built unsorted, then sorted by the row-sort kernel) */
    int32_t radix_passes;
    int32_t path;         /* TF_PATH_* */
    int64_t groups;       /* cell-list path: query groups of the group kernels;
                             0 = the per-bin kernels ran */
} tf_build_info;

/*
 * tf_build_filter -- build W (CSR) and Hs from cell centroids.
 *   centroids: device fp64, row-major [n x dim] (cell midpoints).
 *   n:         number of cells, 1 <= n < 2^31 - 1.
 *   dim:       2 or 3.
 *   rmin:      filter radius, finite and > 0 (rmin <= 0 is invalid).
 *   stream:    cudaStream_t; the call synchronises this stream a few times (lattice
 *              detection, bounding box, nnz readback) and returns a complete handle.
 *   out:       receives the handle (set to NULL on failure).
 * Errors: TF_ERR_INVALID (arguments, non-finite centroid), TF_ERR_NOMEM, TF_ERR_CUDA,
 *         TF_ERR_OVERFLOW.
 */
TF_API tf_status tf_build_filter(const double *centroids, int64_t n, int dim, double rmin,
                          void *stream, tf_filter *out);

/*
 * tf_build_filter_ex -- tf_build_filter with a path choice (the result is the same CSR and Hs
 * on every path: same pairs, bitwise the same weights; Hs within rounding of the order).
 *   flags = TF_BUILD_AUTO: tf_build_filter's behaviour. Centroids ordered as a cube lattice --
 *     cell T*((k*ny + j)*nx + i) + t (1 <= T <= 8 cells per cube, x fastest; FEniCS
 *     BoxMesh/RectangleMesh order) -- within 5% of the spacing of
 *     c[t] + (i hx, j hy, k hz) are detected from a prefix and verified on the device over every
 *     centroid; their rows are then built from a per-type offset table (no cell list, no sort):
 *     TF_PATH_LATTICE_EXACT when every coordinate is exactly on the lattice and on a dyadic grid,
 *     else TF_PATH_LATTICE_TESTED. Anything else takes the cell list (TF_PATH_CELL_LIST).
 *     Detection costs a few small device-to-host copies (synchronising `stream`).
 *   flags = TF_BUILD_CELL_LIST: always the cell list.
 *   flags = TF_BUILD_LATTICE: the lattice path or TF_ERR_INVALID (tests, benchmarks).
 *   flags = TF_BUILD_CELL_LIST_BINS: the cell list with its per-bin kernels (tests, benchmarks).
 *   flags = TF_BUILD_DENSE: ABLATION, O(n^2): the paper's own all-pairs build (its Euclidean
 *     distance matrix, PAPER.md:390-396 and listing PAPER.md:442-445) as tiled kernels that visit
 *     every pair with the same exact pair expression; no cell list. Same CSR; Hs bitwise the
 *     ascending-column sum. For measuring what the cell list buys (tools/dense_probe.py); refuses
 *     n > 4,000,000 (TF_ERR_INVALID).
 * Other arguments and errors as tf_build_filter; TF_ERR_INVALID for unknown flags.
 */
/*
 * tf_lattice_detect_host -- the detection step of the lattice path alone, on a HOST array (no
 * CUDA calls; test hook and diagnostics). Reads a prefix and a few probe rows of `centroids_host`
 * [n x dim] and proposes the lattice model: *ntypes = T (0 if the input is not lattice-ordered),
 * cubes = (nx, ny, nz), spacing = (hx, hy, hz). It does not verify every point: tf_build_filter
 * does that on the device before using the model.
 * Errors: TF_ERR_INVALID (NULL argument, dim, n out of range).
 */
TF_API tf_status tf_lattice_detect_host(const double *centroids_host, int64_t n, int dim, int32_t *ntypes,
                                        int64_t cubes[3], double spacing[3]);

#define TF_BUILD_AUTO 0
#define TF_BUILD_CELL_LIST 1
#define TF_BUILD_LATTICE 2
#define TF_BUILD_CELL_LIST_BINS 3 /* the cell list with the per-bin count/fill kernels (the
                                     round-1 kernels; also the fallback for neighbourhoods beyond
                                     the group kernels' shared memory) */
#define TF_BUILD_DENSE 4          /* ablation: all-pairs build, O(n^2) (see above) */
TF_API tf_status tf_build_filter_ex(const double *centroids, int64_t n, int dim, double rmin, int flags,
                                    void *stream, tf_filter *out);

/*
 * tf_build_stencil -- matrix-free filter for a regular grid (
 * BASELINE.json north_star "matrix-free stencil variant for structured grids").
 *   Cells are indexed (k*ny + j)*nx + i with centroid ((i+1/2)h, (j+1/2)h, (k+1/2)h)
 *   (any common origin); dim = 2 ignores nz. The weight of an integer offset (a,b,c) is
 *   w = max(0, rmin - sqrt(d2)), d2 = ((a h)^2 + (b h)^2) + (c h)^2 < rmin^2 (the CSR build's
 *   expression; identical H for dyadic h such as the configs' h = 1). Row sums use the
 *   in-grid neighbours only (boundary truncation), like the CSR.
 *   The handle supports tf_sensitivity_filter / tf_density_filter (+ *_host) and
 *   tf_build_stats; tf_filter_view returns TF_ERR_INVALID (no CSR is stored). tf_filter_nnz gives the
 *   nnz of the equivalent CSR (for CSR-equivalent bandwidth figures).
 * Errors: TF_ERR_INVALID (dim, sizes, rmin/h not finite > 0, more than 4096 offsets).
 */
TF_API tf_status tf_build_stencil(int dim, int64_t nx, int64_t ny, int64_t nz, double h, double rmin,
                                  void *stream, tf_filter *out);

/* tf_filter_nnz -- stored entries of a CSR filter, or those of the equivalent CSR of a stencil. */
/* tf_build_lattice -- matrix-free filter on a periodic lattice with several cells per cube (row a10
 * generalised): cell index ntypes*((k*ny + j)*nx + i) + t with centroid h*((i, j, k) + o_t), e.g.
 * BoxMesh tetrahedra (6 per cube, PAPER.md:330-333 meshes) or triangulated squares (2 per square).
 * The weight depends only on (s, t, cube offset), so per source type a host-built table of
 * (offset, target type, w) replaces the stored rows (same fp64 pair test and weight as
 * tf_build_filter on those centroids); Hs is recomputed with boundary truncation.
 *   type_offsets_host: HOST fp64 [ntypes x dim], each component in [0, 1) (fractions of h).
 * Applies, host variants and tf_filter_both work as for any handle; tf_filter_view returns
 * TF_ERR_INVALID (no CSR is stored); tf_filter_nnz gives the equivalent CSR's nonzeros.
 * Errors: TF_ERR_INVALID (dim, sizes, ntypes not in [1, 8], offsets outside [0, 1), rmin/h not
 * finite > 0, more than 4096 offsets or a halo tile beyond shared memory). */
TF_API tf_status tf_build_lattice(int dim, int64_t nx, int64_t ny, int64_t nz, double h, int ntypes,
                                  const double *type_offsets_host, double rmin, void *stream, tf_filter *out);
TF_API int64_t tf_filter_nnz(tf_filter h);

/*
 * tf_oc_update -- NEXT-1: optimality-criteria density update with bisection on
 * the Lagrange multiplier (Eq. update; bisection PAPER.md:229-234; listing
 * PAPER.md:380-385), consuming the sensitivity filter's output:
 *     while l2 - l1 > tol:  l_mid = (l2 + l1)/2;
 *         x_new = max(0.001, max(x - move, min(1, min(x + move, x*sqrt(-dc/l_mid)))));
 *         (l1, l2) = (l_mid, l2) if sum(x_new) > volfrac*n else (l1, l_mid)
 *   The paper's call is move = 0.2, l1 = 0, l2 = 1e5, tol = 1e-4. Branch decisions use the EXACT
 *   sum (128-bit fixed point; R15), so results are bitwise reproducible.
 *   x, dc: device fp64 [n] (x in [0, 1], dc <= 0); x_new: device fp64 [n] (may alias x);
 *   lmid_out: device fp64 [1] (the last l_mid); iters_out: device int32 [2] or NULL:
 *   iters_out[0] = bisection steps, iters_out[1] = flags: bit 0 (TF_OC_BRACKET_EXHAUSTED) every step
 *   moved l1 up -- sum(x_new) still exceeded volfrac*n at l2, so the volume constraint is violated
 *   (raise l2); bit 1 (TF_OC_NO_PROGRESS) the bisection stopped before l2 - l1 <= tol because l_mid
 *   rounded to l1 or l2 (tol below the fp64 spacing) or after 4096 steps (reading R23).
 *   One cooperative kernel launch on `stream`, no host sync (read the flags after the stream).
 */
#define TF_OC_BRACKET_EXHAUSTED 1
#define TF_OC_NO_PROGRESS 2
TF_API tf_status tf_oc_update(const double *x, const double *dc, int64_t n, double volfrac, double move,
                              double l1, double l2, double tol, double *x_new, double *lmid_out,
                              int32_t *iters_out, void *stream);

/* tf_filter_view -- borrowed device pointers of the CSR and Hs (no copy). */
TF_API tf_status tf_filter_view(tf_filter h, tf_view *v);

/* tf_build_stats -- diagnostics of the build that produced h (zeros for imported CSRs). */
TF_API tf_status tf_build_stats(tf_filter h, tf_build_info *info);

/*
 * tf_sensitivity_filter -- out_i = (sum_j W_ij x_j dc_j) / (Hs_i * max(1e-3, x_i)).
 *   x, dc: device fp64 [n]; out: device fp64 [n], must not overlap x or dc
 *   (the gather reads other rows' inputs). One kernel launch on `stream`, no sync.
 *   NaNs propagate, except max(1e-3, NaN) = 1e-3 (fmax semantics).
 */
TF_API tf_status tf_sensitivity_filter(tf_filter h, const double *x, const double *dc, double *out,
                                void *stream);

/*
 * tf_sensitivity_filter_energy -- NEXT-2: the sensitivity filter with the
 *   compliance sensitivity evaluated inside the launch from the element energies U:
 *   dc_j = -penal * x_j^(penal-1) * U_j (listing PAPER.md:376), then
 *   out_i = (sum_j W_ij x_j dc_j) / (Hs_i * max(1e-3, x_i)). dc is never stored.
 *   x, U, out: device fp64 [n]; out must not overlap x or U. CSR handles only.
 */
TF_API tf_status tf_sensitivity_filter_energy(tf_filter h, const double *x, const double *U, double penal,
                                              double *out, void *stream);

/* tf_density_filter -- out_i = (sum_j W_ij x_j) / Hs_i. Same conventions. */
TF_API tf_status tf_density_filter(tf_filter h, const double *x, double *out, void *stream);

/* tf_sensitivity_filter_rows / tf_density_filter_rows -- the same filters for rows [0, nrows)
 * only (NEXT-4: a shard's local filter lists its owned rows first and its halo
 * rows after; only the owned rows are wanted). out[i] for i < nrows equals the full call's,
 * bitwise; out[i] for i >= nrows is unspecified (the last row block may write it). x (and dc)
 * are read at every column, so they must hold all n entries. out, x, dc: device fp64 [n].
 * 0 <= nrows <= n (TF_ERR_INVALID otherwise; nrows = 0: no-op). Asynchronous on `stream`.
 * Stencil handles compute all rows. */
TF_API tf_status tf_sensitivity_filter_rows(tf_filter h, const double *x, const double *dc, double *out,
                                            int64_t nrows, void *stream);
TF_API tf_status tf_density_filter_rows(tf_filter h, const double *x, double *out, int64_t nrows, void *stream);

/* tf_filter_both -- both filters of one iteration in ONE pass over H (the CSR streams from HBM
 * once; each entry gathers t_j = x_j*dc_j and x_j): sens_out as tf_sensitivity_filter,
 * dens_out as tf_density_filter, bitwise (same per-row summation order).
 *   x, dc, sens_out, dens_out: device fp64 [n]; the outputs must not overlap each other, x or dc.
 * Asynchronous on `stream`. Stencil handles run the two stencil passes. */
TF_API tf_status tf_filter_both(tf_filter h, const double *x, const double *dc, double *sens_out, double *dens_out,
                                void *stream);

/*
 * tf_sensitivity_filter_range / tf_density_filter_range -- the filters for rows [r0, r1) only
 * (NEXT-4: a shard applies its interior rows while the halo exchange is in flight, then its
 * boundary rows). out[i] for r0 <= i < r1 equals the full call's, bitwise; rows of the row block
 * holding r0 that precede it are rewritten with their full-call values; other rows unspecified.
 * The sensitivity filter reads x and dc of every local index (its fused x*dc pass covers all n).
 * 0 <= r0 <= r1 <= n (TF_ERR_INVALID otherwise). Asynchronous on `stream`.
 */
TF_API tf_status tf_sensitivity_filter_range(tf_filter h, const double *x, const double *dc, double *out,
                                             int64_t r0, int64_t r1, void *stream);
TF_API tf_status tf_density_filter_range(tf_filter h, const double *x, double *out, int64_t r0, int64_t r1,
                                         void *stream);

/*
 * NEXT-4: slab partition of one filter problem over `nranks`
 * GPUs, computed on the device from the global centroids (the same on every rank):
 *   longest bounding-box axis; slabs cut at count quantiles of a 65,536-bucket histogram of that
 *   coordinate (points with equal coordinates stay together); rank k's window = its slab widened by
 *   rmin(1 + 1e-9) plus a rounding slack on both sides (open at the domain ends); halo of rank k =
 *   the other ranks' points in its window; INTERIOR owned points lie at least that far inside
 *   both faces (no neighbour outside the slab), the other owned points are BOUNDARY.
 *   Local order: [interior | boundary | halo grouped by source rank], each ascending global id.
 *   Send list to rank j: my owned points in j's window, ascending global id, as LOCAL indices --
 *   the order in which rank j stores them in its halo.
 * tf_shard_plan: centroids device fp64 [n x dim] (finite); 1 <= nranks <= 64; 0 <= rank < nranks.
 *   Synchronises `stream` a few times (histogram, counts). Errors as tf_build_filter.
 * tf_shard_view_get: sizes and borrowed device views (valid until tf_shard_free):
 *   local_ids [n_owned + n_halo] int32 global ids; send_idx [sum of send counts] int32 local
 *   indices grouped by destination rank ascending.
 * tf_shard_counts: recv_host[k] / send_host[k] = halo points received from / sent to rank k.
 * tf_gather_rows: dst[t*dim + d] = src[idx[t]*dim + d] for t < m (device arrays; builds the local
 *   centroids of a shard). Asynchronous on `stream`.
 */
typedef struct tf_shard_s *tf_shard;
typedef struct {
    int32_t nranks, rank, axis;
    double cut_lo, cut_hi;        /* this rank's slab along `axis` (-inf / +inf at the ends) */
    int64_t n_interior, n_owned, n_halo;
    const int32_t *local_ids;
    const int32_t *send_idx;
} tf_shard_view;
TF_API tf_status tf_shard_plan(const double *centroids, int64_t n, int dim, double rmin, int32_t nranks,
                               int32_t rank, void *stream, tf_shard *out);
TF_API tf_status tf_shard_view_get(tf_shard s, tf_shard_view *v);
TF_API tf_status tf_shard_counts(tf_shard s, int64_t *recv_host, int64_t *send_host);
TF_API void tf_shard_free(tf_shard s);
TF_API tf_status tf_gather_rows(const double *src, int32_t dim, const int32_t *idx, int64_t m, double *dst,
                                void *stream);

/* tf_free -- release everything the handle owns, stream-ordered on the stream the handle was built
 * on (cudaFreeAsync; no device-wide synchronisation). Work on that stream and on the handle's own
 * host-pipeline streams is ordered before the release; work the caller issued with h on OTHER
 * streams must be complete, or ordered before that stream, when tf_free is called. NULL: no-op. */
TF_API void tf_free(tf_filter h);

/* tf_last_error -- thread-local message for the last non-OK status of this thread. */
TF_API const char *tf_last_error(void);

/* ------------------------------------------------------------------ host-buffer variants
 * The same operations on HOST arrays (end-to-end path): inputs are copied to
 * handle-owned device buffers on `stream`, the kernel runs, and the result is copied
 * back; the call synchronises `stream` before returning so `*_host` outputs are valid.
 * Pinned (page-locked) host memory gives full PCIe bandwidth; pageable also works. */
TF_API tf_status tf_build_filter_host(const double *centroids_host, int64_t n, int dim, double rmin,
                               void *stream, tf_filter *out);
TF_API tf_status tf_sensitivity_filter_host(tf_filter h, const double *x_host, const double *dc_host,
                                     double *out_host, void *stream);
TF_API tf_status tf_density_filter_host(tf_filter h, const double *x_host, double *out_host,
                                        void *stream);
/* One optimisation iteration's filtering on host buffers. Pipelined over the apply plan's (up to
 * 8) row-range chunks: x then dc upload in row pieces on a handle-owned upload stream; a chunk of
 * either filter starts once the pieces up to the one holding its largest column have landed;
 * each chunk's result downloads on a handle-owned download stream while the next chunk computes.
 * Stencil handles and one-window plans use whole-array launches. Results are bitwise those of
 * the device calls. Synchronises before returning. Not safe to call concurrently on the same
 * handle. */
TF_API tf_status tf_filter_iteration_host(tf_filter h, const double *x_host, const double *dc_host,
                                          double *sens_host, double *dens_host, void *stream);

/* ------------------------------------------------------------------ test / diagnostics */

/* tf_filter_from_csr -- TEST HOOK: wrap a host CSR (e.g. the oracle's) in a handle so the
 * apply kernels can be tested independently of the GPU build. Arrays are copied; the
 * caller keeps ownership. rowptr_host [n+1], cols_host [nnz], vals_host [nnz], hs_host [n].
 * Validates rowptr monotone and 0 <= cols < n. dim/rmin are recorded as given (0 allowed). */
TF_API tf_status tf_filter_from_csr(const int64_t *rowptr_host, const int32_t *cols_host,
                             const double *vals_host, const double *hs_host, int64_t n,
                             void *stream, tf_filter *out);

/* Number of CUDA kernels this library has launched in this process (monotone counter). */
/* tf_halo_pack -- dst[i] = src[idx[i]], i < m (device arrays; idx int32 in [0, n_src)): gathers the
 * boundary values a slab shard sends to a neighbour (NEXT-4). Asynchronous.
 * Errors: TF_ERR_INVALID (NULL / host pointers, m < 0). m = 0 is a no-op. */
TF_API tf_status tf_halo_pack(const double *src, const int32_t *idx, int64_t m, double *dst, void *stream);

TF_API uint64_t tf_kernel_launches(void);

/* TEST HOOK: make every single device allocation larger than `bytes` fail with
 * TF_ERR_NOMEM (0 = no limit). Exercises the out-of-memory paths. Process-wide. */
TF_API void tf_debug_set_alloc_limit(uint64_t bytes);

TF_API int tf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TOPOFILT_H */
