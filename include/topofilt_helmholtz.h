/*
 * topofilt_helmholtz.h -- C ABI of the Helmholtz PDE filter in
 * libtopofilt.
 *
 * The paper replaces the distance filter by "the Helmholtz filter as described in
 * [Lazarov & Sigmund 2011]" for its parallel code without stating the
 * operator; the operator here follows SPEC.md:225-233 and 243 (readings R17-R20):
 *
 *   (-R^2 Laplace + 1) s~ = s on the P1 space of a simplex mesh, natural boundary conditions.
 *   1. cell -> node projection, volume-weighted: s_n = sum_{c owns n} |c| s_c / sum |c|
 *   2. Galerkin system A = R^2 K + M (P1 stiffness K and consistent mass M), b = M s_n
 *   3. A u = b solved by Jacobi-preconditioned conjugate gradients on the GPU, starting from
 *      u = s_n, until ||b - A u||_2 <= rtol ||b||_2 or maxit iterations
 *   4. node -> cell evaluation as the nodal mean: s~_c = mean_{n in c} u_n
 *   R = rmin / (2 sqrt 3) maps the distance-filter radius to the PDE length;
 *   the caller passes R itself.
 *
 * Conventions are those of topofilt.h: device pointers, stream passed as void*, tf_status
 * returns, tf_last_error() for the message. A handle owns copies of what it needs (cell
 * connectivity, volumes, the assembled CSR and CG scratch); the caller's arrays may be freed
 * after tf_helmholtz_build returns. The CG scratch lives in the handle: calls on the SAME
 * handle must be ordered (one stream, or synchronised); different handles are independent.
 */
#ifndef TOPOFILT_HELMHOLTZ_H
#define TOPOFILT_HELMHOLTZ_H

#include "topofilt.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tf_helmholtz_s *tf_helmholtz; /* opaque */

/* Result of one solve, written by the device at the end of the call (stream-ordered). */
typedef struct {
    int32_t iterations;   /* CG iterations performed */
    int32_t converged;    /* 1 if ||r|| <= rtol ||b|| was reached within maxit */
    double rel_residual;  /* ||b - A u||_2 / ||b||_2 of the returned u (recurrence value; 0 if b = 0) */
} tf_helmholtz_info;

/* Read-only view of the assembled system (device pointers owned by the handle). */
typedef struct {
    int64_t n_nodes, n_cells, nnz;
    int dim;
    double R;
    const int64_t *rowptr;      /* [n_nodes+1] */
    const int32_t *cols;        /* [nnz], ascending within a row */
    const double *vals_A;       /* [nnz] R^2 K + M */
    const double *vals_M;       /* [nnz] M (same pattern) */
    const double *node_weight;  /* [n_nodes] sum of the volumes of the cells owning the node */
    const double *cell_volume;  /* [n_cells] */
} tf_helmholtz_system;

/* Assemble the filter for a simplex mesh.
 *   nodes  [n_nodes, dim] fp64 row-major (device), node coordinates
 *   cells  [n_cells, dim+1] int32 row-major (device), vertex indices in [0, n_nodes);
 *          triangles (dim 2) or tetrahedra (dim 3), either orientation
 *   R      PDE length >= 0 (R = 0 gives the mass-matrix projection only)
 * Row entries of A are summed over the owning cells in ascending cell order (deterministic).
 * Nodes no cell uses get an empty row and stay 0 (R20).
 * Errors: TF_ERR_INVALID (dim not 2/3, n_nodes or n_cells < 1, n_nodes >= 2^31, R not finite
 *         or < 0, a vertex index out of range, a cell of zero or non-finite volume),
 *         TF_ERR_OVERFLOW (n_cells*(dim+1)^2 >= 2^31), TF_ERR_NOMEM, TF_ERR_CUDA.
 * Synchronises `stream` (the nnz is read back). */
TF_API tf_status tf_helmholtz_build(const double *nodes, int64_t n_nodes, const int32_t *cells, int64_t n_cells,
                                    int dim, double R, void *stream, tf_helmholtz *out);

/* s~ = Helmholtz(sigma): sigma, out [n_cells] fp64 (device; may alias). rtol > 0, maxit >= 1.
 * info: optional DEVICE pointer (NULL = not reported). Asynchronous. */
TF_API tf_status tf_helmholtz_filter(tf_helmholtz h, const double *sigma, double *out, double rtol, int maxit,
                                     tf_helmholtz_info *info, void *stream);

/* Sensitivity use (floor as in the listing PAPER.md:447):
 * out = Helmholtz(x * dc) / max(1e-3, x). x, dc, out [n_cells] fp64 (device; out may alias dc). */
TF_API tf_status tf_helmholtz_sensitivity(tf_helmholtz h, const double *x, const double *dc, double *out,
                                          double rtol, int maxit, tf_helmholtz_info *info, void *stream);

TF_API tf_status tf_helmholtz_view(tf_helmholtz h, tf_helmholtz_system *v);

/* Releases the handle (synchronises the device first). NULL is ignored. */
TF_API void tf_helmholtz_free(tf_helmholtz h);

#ifdef __cplusplus
}
#endif

#endif /* TOPOFILT_HELMHOLTZ_H */
