// helmholtz.cu -- NEXT-3: the Helmholtz PDE filter on a simplex mesh.
// Operator: include/topofilt_helmholtz.h (DESIGN.md
// R17-R20). Build = P1 element geometry + deterministic assembly; apply = one cooperative
// persistent kernel that runs projection, Jacobi-PCG and the nodal-mean evaluation.
//
// Assembly (deterministic, no floating-point atomics):
//   items t = c*(d+1)^2 + a*(d+1) + b  (cell c, local rows a, cols b)
//   two stable LSD radix sorts (by column, then by row) order the items by (row, col) with t
//   ascending inside each (row, col) run; run heads -> scan -> CSR slots; each run is summed
//   in that fixed order: A = R^2 sum K_c[a,b] + sum M_c[a,b].
//   Node -> cell incidence (for the projection) by one more stable sort of (node, cell).
//
// Apply (k_hz_apply): phases separated by grid.sync(); every dot product is reduced per block
// in a fixed order and the block partials are summed in a fixed order by every block, so
// every block takes the same decisions and the result is reproducible run to run.
//   P0  s_n = sum_c |c| s_c / W_n (incident cells ascending), u = s_n
//   P1  b = M s_n, r = b - A u, z = D^-1 r, p_old = 0;   dots (b.b, r.z, r.r)
//   loop:  PA  p = z + beta p_old (row owner), q = A p computed from z and p_old directly
//              (q_a = sum_b A_ab (z_b + beta p_old_b): no separate p pass, so two grid
//              syncs per iteration instead of three; z and p_old are stored interleaved so
//              each entry costs one 16-byte gather);   dot p.q
//          PB  u += alpha p, r -= alpha q, z = D^-1 r, store (z, p);   dots (r.z, r.r)
//   P2  s~_c = mean of u over the cell's nodes (/ max(1e-3, x_c) for the sensitivity use)
// CSR rows and incidence lists use 2 lanes x 4 loads in flight; 5 blocks/SM (48 registers).
// Swept on config 5 (tools/helm_probe.py): per CG iteration 120 us at (2, 4, 5) vs 164 at
// (4, 4, -), 143 at (4, 4, 5), 151 at (1, 8, -), 198 at (8, 2, 5), 205 at (2, 2, -); more registers
// cost more than they hide.
#include <cooperative_groups.h>
#include <math.h>

#include <algorithm>

#include "../../include/topofilt_helmholtz.h"
#include "tf_internal.cuh"

struct tf_helmholtz_s {
    int device = -1;  // the CUDA device current at build time; every call must use it
    int64_t nn = 0, nc = 0, nnz = 0;
    int dim = 0;
    double R = 0;
    int32_t *cells = nullptr;     // [nc*(dim+1)]
    double *vol = nullptr;        // [nc]
    int64_t *inc_ptr = nullptr;   // [nn+1] node -> incident cells
    int32_t *inc_cell = nullptr;  // [nc*(dim+1)] ascending per node
    double *W = nullptr;          // [nn]
    int64_t *rowptr = nullptr;    // [nn+1]
    int32_t *cols = nullptr;      // [nnz]
    double *valA = nullptr, *valM = nullptr;  // [nnz]
    double *dinv = nullptr;       // [nn] 1/A_aa (0 on empty rows)
    double *vec = nullptr;        // [7*nn] CG scratch: (z,p) pairs, sn, u, r, q, p_new
    double *parts = nullptr;      // [2 * grid * 4] block partials
    int grid = 0;
};

namespace tf {
namespace {

constexpr int kHzThreads = 256;
// lanes per CSR row / incidence list, and loads each lane issues before its gathers
// (tuning macros for tools/variant_sweep.py)
#ifndef TF_HZ_LANES
#define TF_HZ_LANES 2
#endif
#ifndef TF_HZ_UNROLL
#define TF_HZ_UNROLL 4
#endif
#ifndef TF_HZ_MINB
#define TF_HZ_MINB 5
#endif
constexpr int kRowLanes = TF_HZ_LANES;
constexpr int kUnroll = TF_HZ_UNROLL;

int ceil_log2_i64(int64_t v) {
    int b = 0;
    while (b < 63 && (int64_t(1) << b) < v) ++b;
    return b;
}

// ---------------------------------------------------------------- build kernels
// Per cell: |c| and the barycentric gradients G[a] (a = 0..d) from J^-1 (adjugate / det).
// flags: bit 0 = vertex index out of range, bit 1 = zero / non-finite volume.
template <int D>
__global__ void k_hz_geom(const double *__restrict__ nodes, int64_t nn, const int32_t *__restrict__ cells, int64_t nc,
                          double *__restrict__ vol, double *__restrict__ G, int *__restrict__ flags) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
        int32_t v[D + 1];
        bool bad = false;
#pragma unroll
        for (int a = 0; a <= D; ++a) {
            v[a] = cells[c * (D + 1) + a];
            bad |= v[a] < 0 || (int64_t)v[a] >= nn;
        }
        if (bad) {
            atomicOr(flags, 1);
            vol[c] = 0.0;
            continue;
        }
        double J[D][D];  // J[i][k] = X_{k+1}[i] - X_0[i]
#pragma unroll
        for (int k = 0; k < D; ++k)
#pragma unroll
            for (int i = 0; i < D; ++i) J[i][k] = nodes[(int64_t)v[k + 1] * D + i] - nodes[(int64_t)v[0] * D + i];
        double det, inv[D][D];  // inv row k = grad lambda_{k+1}
        if (D == 2) {
            det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
            inv[0][0] = J[1][1] / det, inv[0][1] = -J[0][1] / det;
            inv[1][0] = -J[1][0] / det, inv[1][1] = J[0][0] / det;
        } else {
            const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
            const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
            const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
            det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
            const double c10 = J[0][2] * J[2][1] - J[0][1] * J[2][2];
            const double c11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
            const double c12 = J[0][1] * J[2][0] - J[0][0] * J[2][1];
            const double c20 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
            const double c21 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
            const double c22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
            // inv = adj(J)/det, adj[i][j] = cofactor[j][i]
            inv[0][0] = c00 / det, inv[0][1] = c10 / det, inv[0][2] = c20 / det;
            inv[1][0] = c01 / det, inv[1][1] = c11 / det, inv[1][2] = c21 / det;
            inv[2][0] = c02 / det, inv[2][1] = c12 / det, inv[2][2] = c22 / det;
        }
        const double vc = fabs(det) / (D == 2 ? 2.0 : 6.0);
        if (!(vc > 0.0) || !isfinite(vc)) {
            atomicOr(flags, 2);
            vol[c] = 0.0;
            continue;
        }
        vol[c] = vc;
        double *g = G + c * (D + 1) * D;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s -= inv[k][i];
            g[i] = s;  // grad lambda_0 = -sum_k grad lambda_k
#pragma unroll
            for (int k = 0; k < D; ++k) g[(k + 1) * D + i] = inv[k][i];
        }
    }
}

// (node, cell) incidence items, cell-major
template <int D>
__global__ void k_hz_inc_items(const int32_t *__restrict__ cells, int64_t nc, uint32_t *__restrict__ key,
                               uint32_t *__restrict__ val) {
    const int64_t m = nc * (D + 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        key[i] = (uint32_t)cells[i];
        val[i] = (uint32_t)(i / (D + 1));
    }
}

// start offsets of each key value in a sorted key array: ptr[k] = #items with key < k, k in
// [0, nk]; thread i assigns ptr[k] = i for key[i-1] < k <= key[i] (key[-1] = -1, key[m] = nk)
__global__ void k_hz_starts(const uint32_t *__restrict__ key, int64_t m, int64_t nk, int64_t *__restrict__ ptr) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= m; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = (i == 0) ? -1 : (int64_t)key[i - 1];
        const int64_t cur = (i == m) ? nk : (int64_t)key[i];
        for (int64_t k = prev + 1; k <= cur; ++k) ptr[k] = i;
    }
}

__global__ void k_hz_node_weight(const int64_t *__restrict__ ptr, const uint32_t *__restrict__ inc,
                                 const double *__restrict__ vol, int64_t nn, double *__restrict__ W) {
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < nn; a += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t j = ptr[a]; j < ptr[a + 1]; ++j) s += vol[inc[j]];
        W[a] = s;
    }
}

// matrix items: key = column, val = item index t
template <int D>
__global__ void k_hz_mat_items(const int32_t *__restrict__ cells, int64_t nc, uint32_t *__restrict__ key,
                               uint32_t *__restrict__ val) {
    constexpr int D1 = D + 1, D2 = D1 * D1;
    const int64_t m = nc * D2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / D2;
        const int b = (int)(t % D1);
        key[t] = (uint32_t)cells[c * D1 + b];
        val[t] = (uint32_t)t;
    }
}

template <int D>
__device__ __forceinline__ uint32_t item_row(const int32_t *cells, uint32_t t) {
    constexpr int D1 = D + 1, D2 = D1 * D1;
    return (uint32_t)cells[(int64_t)(t / D2) * D1 + (int)((t % D2) / D1)];
}
template <int D>
__device__ __forceinline__ uint32_t item_col(const int32_t *cells, uint32_t t) {
    constexpr int D1 = D + 1, D2 = D1 * D1;
    return (uint32_t)cells[(int64_t)(t / D2) * D1 + (int)(t % D1)];
}

template <int D>
__global__ void k_hz_row_keys(const int32_t *__restrict__ cells, const uint32_t *__restrict__ t_sorted, int64_t m,
                              uint32_t *__restrict__ key) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        key[i] = item_row<D>(cells, t_sorted[i]);
}

// run heads of the (row, col)-sorted items + per-row unique counts
template <int D>
__global__ void k_hz_heads(const int32_t *__restrict__ cells, const uint32_t *__restrict__ rkey,
                           const uint32_t *__restrict__ t, int64_t m, int32_t *__restrict__ head,
                           int32_t *__restrict__ rowcnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const bool h = (i == 0) || rkey[i] != rkey[i - 1] || item_col<D>(cells, t[i]) != item_col<D>(cells, t[i - 1]);
        head[i] = h ? 1 : 0;
        if (h) atomicAdd(&rowcnt[rkey[i]], 1);  // integer count: order-free
    }
}

// one thread per run: sums in ascending t (the fixed order of the sorted items)
template <int D>
__global__ void k_hz_entries(const int32_t *__restrict__ cells, const uint32_t *__restrict__ t,
                             const int32_t *__restrict__ head, const int64_t *__restrict__ slot, int64_t m,
                             const double *__restrict__ vol, const double *__restrict__ G, double R2,
                             int32_t *__restrict__ cols, double *__restrict__ valA, double *__restrict__ valM) {
    constexpr int D1 = D + 1, D2 = D1 * D1;
    const double mden = (double)((D + 1) * (D + 2));
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        if (!head[i]) continue;
        double ks = 0.0, ms = 0.0;
        int64_t j = i;
        do {
            const uint32_t tj = t[j];
            const int64_t c = tj / D2;
            const int a = (int)((tj % D2) / D1), b = (int)(tj % D1);
            const double *g = G + c * D1 * D;
            double gg = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) gg += g[a * D + k] * g[b * D + k];
            const double vc = vol[c];
            ks += vc * gg;
            ms += (vc / mden) * (a == b ? 2.0 : 1.0);  // as |c|/((d+1)(d+2)) * (1 + delta)
            ++j;
        } while (j < m && !head[j]);
        const int64_t u = slot[i];
        cols[u] = (int32_t)item_col<D>(cells, t[i]);
        valA[u] = R2 * ks + ms;
        valM[u] = ms;
    }
}

__global__ void k_hz_diag(const int64_t *__restrict__ rowptr, const int32_t *__restrict__ cols,
                          const double *__restrict__ valA, int64_t nn, double *__restrict__ dinv) {
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < nn; a += (int64_t)gridDim.x * blockDim.x) {
        double d = 0.0;
        for (int64_t k = rowptr[a]; k < rowptr[a + 1]; ++k)
            if (cols[k] == (int32_t)a) d = valA[k];
        dinv[a] = (d != 0.0) ? 1.0 / d : 0.0;
    }
}

// ---------------------------------------------------------------- apply kernel
// Fixed-order block sum of N doubles; the result is returned to every thread.
template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double (*sm)[N]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < N; ++k)
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    __syncthreads();  // sm reuse
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < N; ++k) sm[warp][k] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; ++k) {
        double s = 0.0;
        for (int w = 0; w < kHzThreads / 32; ++w) s += sm[w][k];
        v[k] = s;
    }
}

// Block partial -> parts[slot]; grid.sync; every block sums all partials in block order.
template <int N>
__device__ __forceinline__ void grid_sum(double (&v)[N], double (*sm)[N], double *parts, int slot,
                                         cooperative_groups::grid_group &grid) {
    block_sum<N>(v, sm);
    double *ps = parts + (size_t)slot * gridDim.x * 4;
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < N; ++k) ps[(size_t)blockIdx.x * 4 + k] = v[k];
    grid.sync();
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = 0.0;
    for (unsigned bb = threadIdx.x; bb < gridDim.x; bb += blockDim.x)
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] += __ldcg(ps + (size_t)bb * 4 + k);
    block_sum<N>(v, sm);
}

struct HzArgs {
    const int32_t *cells;
    const double *vol;
    const int64_t *inc_ptr;
    const int32_t *inc_cell;
    const double *W;
    const int64_t *rowptr;
    const int32_t *cols;
    const double *valA, *valM, *dinv;
    double2 *zp;  // (z, p) interleaved: one 16-byte gather per entry in the SpMV
    double *sn, *u, *r, *q, *pn;
    double *parts;
    int64_t nn, nc;
    const double *sigma;  // filter input (SENS: unused)
    const double *x, *dc; // SENS inputs
    double *out;
    double rtol2;
    int maxit;
    tf_helmholtz_info *info;
};

template <int D, bool SENS>
__global__ void __launch_bounds__(kHzThreads, TF_HZ_MINB) k_hz_apply(HzArgs A) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    __shared__ double sm3[kHzThreads / 32][3];
    __shared__ double sm2[kHzThreads / 32][2];
    __shared__ double sm1[kHzThreads / 32][1];
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t nn = A.nn;
    const int g = (int)(gid & (kRowLanes - 1));
    const int64_t rgid = gid / kRowLanes, RT = T / kRowLanes;
    const int64_t rounds = (nn + RT - 1) / RT;  // warp-uniform row loop (shuffles inside)

    // P0: projection (kRowLanes lanes per node over its incident cells, ascending per lane)
    for (int64_t it = 0; it < rounds; ++it) {
        const int64_t a = it * RT + rgid;
        double s = 0.0;
        if (a < nn) {
            const int64_t j0 = A.inc_ptr[a], j1 = A.inc_ptr[a + 1];
            for (int64_t jb = j0 + g; jb < j1; jb += kRowLanes * kUnroll) {
                int32_t c[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int64_t j = jb + (int64_t)u * kRowLanes;
                    c[u] = (j < j1) ? A.inc_cell[j] : -1;
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    if (c[u] >= 0) {
                        const double sc = SENS ? A.x[c[u]] * A.dc[c[u]] : A.sigma[c[u]];
                        s += A.vol[c[u]] * sc;
                    }
                }
            }
        }
        for (int o = 1; o < kRowLanes; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (a < nn && g == 0) {
            const double w = A.W[a];
            const double v = (w > 0.0) ? s / w : 0.0;
            A.sn[a] = v;
            A.u[a] = v;
        }
    }
    grid.sync();
    // P1: b = M sn, r = b - A u, z = D^-1 r, p_old = 0
    double d3[3] = {0.0, 0.0, 0.0};  // b.b, r.z, r.r
    for (int64_t it = 0; it < rounds; ++it) {
        const int64_t a = it * RT + rgid;
        double bm = 0.0, au = 0.0;
        if (a < nn) {
            const int64_t k0 = A.rowptr[a], k1 = A.rowptr[a + 1];
            for (int64_t kb = k0 + g; kb < k1; kb += kRowLanes * kUnroll) {
                int32_t c[kUnroll];
                double vm[kUnroll], va[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int64_t k = kb + (int64_t)u * kRowLanes;
                    const bool ok = k < k1;
                    c[u] = ok ? A.cols[k] : (int32_t)a;
                    vm[u] = ok ? A.valM[k] : 0.0;
                    va[u] = ok ? A.valA[k] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const double sv = __ldcg(A.sn + c[u]);
                    bm += vm[u] * sv;
                    au += va[u] * sv;  // u = sn here
                }
            }
        }
        for (int o = 1; o < kRowLanes; o <<= 1) {
            bm += __shfl_xor_sync(0xffffffffu, bm, o);
            au += __shfl_xor_sync(0xffffffffu, au, o);
        }
        if (a < nn && g == 0) {
            const double rr = bm - au;
            const double zz = A.dinv[a] * rr;
            A.r[a] = rr;
            A.zp[a] = make_double2(zz, 0.0);  // p_old = 0
            d3[0] += bm * bm;
            d3[1] += rr * zz;
            d3[2] += rr * rr;
        }
    }
    int slot = 0;
    grid_sum<3>(d3, sm3, A.parts, slot, grid);
    slot ^= 1;
    const double bb = d3[0];
    double rz = d3[1], rr = d3[2];
    bool conv = rr <= A.rtol2 * bb;
    double beta = 0.0;
    int iters = 0;
    while (!conv && iters < A.maxit) {
        // PA: p = z + beta p_old (owner), q = A (z + beta p_old); each lane loads up to
        // kUnroll (col, val) pairs before the gathers (memory-level parallelism)
        double d1[1] = {0.0};
        for (int64_t it = 0; it < rounds; ++it) {
            const int64_t a = it * RT + rgid;
            double qa = 0.0;
            if (a < nn) {
                const int64_t k0 = A.rowptr[a], k1 = A.rowptr[a + 1];
                for (int64_t kb = k0 + g; kb < k1; kb += kRowLanes * kUnroll) {
                    int32_t c[kUnroll];
                    double v[kUnroll];
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        const int64_t k = kb + (int64_t)u * kRowLanes;
                        const bool ok = k < k1;
                        c[u] = ok ? A.cols[k] : (int32_t)a;
                        v[u] = ok ? A.valA[k] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        const double2 t = __ldcg(A.zp + c[u]);
                        qa += v[u] * (t.x + beta * t.y);
                    }
                }
            }
            for (int o = 1; o < kRowLanes; o <<= 1) qa += __shfl_xor_sync(0xffffffffu, qa, o);
            if (a < nn && g == 0) {
                const double2 t = __ldcg(A.zp + a);
                const double pa = t.x + beta * t.y;
                A.pn[a] = pa;
                A.q[a] = qa;
                d1[0] += pa * qa;
            }
        }
        grid_sum<1>(d1, sm1, A.parts, slot, grid);
        slot ^= 1;
        const double alpha = rz / d1[0];
        // PB: u += alpha p, r -= alpha q, z = D^-1 r; (z, p) stored as the next PA's pair
        double d2[2] = {0.0, 0.0};
        for (int64_t a = gid; a < nn; a += T) {
            const double pa = __ldcg(A.pn + a);
            A.u[a] = __ldcg(A.u + a) + alpha * pa;
            const double ra = __ldcg(A.r + a) - alpha * __ldcg(A.q + a);
            const double za = A.dinv[a] * ra;
            A.r[a] = ra;
            A.zp[a] = make_double2(za, pa);
            d2[0] += ra * za;
            d2[1] += ra * ra;
        }
        grid_sum<2>(d2, sm2, A.parts, slot, grid);
        slot ^= 1;
        ++iters;
        beta = d2[0] / rz;
        rz = d2[0];
        rr = d2[1];
        conv = rr <= A.rtol2 * bb;
    }
    // P2: nodal mean per cell (u was last written before the final grid_sum's sync)
    for (int64_t c = gid; c < A.nc; c += T) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a <= D; ++a) s += __ldcg(A.u + A.cells[c * (D + 1) + a]);
        double v = s / (double)(D + 1);
        if (SENS) v = v / fmax(1e-3, A.x[c]);
        A.out[c] = v;
    }
    if (gid == 0 && A.info) {
        A.info->iterations = iters;
        A.info->converged = conv ? 1 : 0;
        A.info->rel_residual = (bb > 0.0) ? sqrt(rr / bb) : 0.0;
    }
}

template <int D, bool SENS>
tf_status hz_launch(tf_helmholtz_s *h, const double *sigma, const double *x, const double *dc, double *out,
                    double rtol, int maxit, tf_helmholtz_info *info, cudaStream_t s) {
    HzArgs A;
    A.cells = h->cells, A.vol = h->vol, A.inc_ptr = h->inc_ptr, A.inc_cell = h->inc_cell, A.W = h->W;
    A.rowptr = h->rowptr, A.cols = h->cols, A.valA = h->valA, A.valM = h->valM, A.dinv = h->dinv;
    const int64_t nn = h->nn;
    A.zp = reinterpret_cast<double2 *>(h->vec);  // first: 16-byte aligned
    A.sn = h->vec + 2 * nn, A.u = h->vec + 3 * nn, A.r = h->vec + 4 * nn, A.q = h->vec + 5 * nn;
    A.pn = h->vec + 6 * nn;
    A.parts = h->parts, A.nn = nn, A.nc = h->nc;
    A.sigma = sigma, A.x = x, A.dc = dc, A.out = out;
    A.rtol2 = rtol * rtol, A.maxit = maxit, A.info = info;
    void *args[] = {(void *)&A};
    cudaError_t e = cudaLaunchCooperativeKernel((const void *)k_hz_apply<D, SENS>, dim3(h->grid), dim3(kHzThreads),
                                                args, 0, s);
    count_launch();
    if (e != cudaSuccess) {
        set_error("tf_helmholtz: cooperative launch failed: %s", cudaGetErrorString(e));
        return TF_ERR_CUDA;
    }
    return TF_OK;
}

// Co-resident maximum, but no more blocks than the node rows need (small meshes are bound by
// the grid syncs, whose cost grows with the block count); at least one block per SM.
template <int D>
int hz_grid(const DeviceInfo &di, int64_t nn) {
    int o1 = 0, o2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_hz_apply<D, false>, kHzThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_hz_apply<D, true>, kHzThreads, 0);
    const int64_t full = (int64_t)di.sms * std::max(1, std::min(std::min(o1, o2), 8));
    const int64_t need = (nn * kRowLanes + kHzThreads - 1) / kHzThreads;
    return (int)std::max<int64_t>(std::min<int64_t>(full, need), std::min<int64_t>(full, di.sms));
}

void hz_destroy(tf_helmholtz_s *h) {
    if (!h) return;
    DeviceScope on(h->device);  // free on the handle's device, whichever is current
    cudaDeviceSynchronize();
    void *ps[] = {h->cells, h->vol, h->inc_ptr, h->inc_cell, h->W, h->rowptr, h->cols,
                  h->valA, h->valM, h->dinv, h->vec, h->parts};
    for (void *p : ps)
        if (p) cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
    delete h;
}

template <int D>
tf_status hz_build(const double *nodes, int64_t nn, const int32_t *cells, int64_t nc, double R, cudaStream_t s,
                   tf_helmholtz_s *h) {
    constexpr int D1 = D + 1, D2 = D1 * D1;
    DeviceInfo di;
    TF_TRY(device_info(&di));
    const int threads = 256;
    auto blocks = [&](int64_t work) {
        return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + threads - 1) / threads, (int64_t)di.sms * 16));
    };
    NvtxRange nv("tf_helmholtz_build");
    TF_TRY(dalloc(&h->cells, (size_t)nc * D1, s, "helmholtz cells"));
    TF_CUDA_TRY(cudaMemcpyAsync(h->cells, cells, (size_t)nc * D1 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    TF_TRY(dalloc(&h->vol, (size_t)nc, s, "helmholtz volumes"));
    DevBuf<double> G;
    TF_TRY(G.alloc((size_t)nc * D1 * D, s, "helmholtz gradients"));
    DevBuf<int> flags;
    TF_TRY(flags.alloc(1, s, "helmholtz flags"));
    TF_CUDA_TRY(cudaMemsetAsync(flags.p, 0, sizeof(int), s));
    k_hz_geom<D><<<blocks(nc), threads, 0, s>>>(nodes, nn, h->cells, nc, h->vol, G.p, flags.p);
    TF_LAUNCH_CHECK();
    int hflags = 0;
    TF_CUDA_TRY(cudaMemcpyAsync(&hflags, flags.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    if (hflags & 1) {
        set_error("tf_helmholtz_build: a cell vertex index is outside [0, n_nodes)");
        return TF_ERR_INVALID;
    }
    if (hflags & 2) {
        set_error("tf_helmholtz_build: a cell has zero or non-finite volume");
        return TF_ERR_INVALID;
    }
    const int nbits = ceil_log2_i64(nn);
    // ---- node -> cell incidence (stable: cells ascending per node)
    const int64_t mi = nc * D1;
    {
        DevBuf<uint32_t> k0, v0, k1, v1;
        TF_TRY(k0.alloc(mi, s, "incidence keys"));
        TF_TRY(v0.alloc(mi, s, "incidence vals"));
        TF_TRY(k1.alloc(mi, s, "incidence keys alt"));
        TF_TRY(v1.alloc(mi, s, "incidence vals alt"));
        k_hz_inc_items<D><<<blocks(mi), threads, 0, s>>>(h->cells, nc, k0.p, v0.p);
        TF_LAUNCH_CHECK();
        uint32_t *ks, *vs;
        int passes;
        TF_TRY(radix_sort_pairs(k0.p, v0.p, k1.p, v1.p, mi, nbits, s, &ks, &vs, &passes));
        TF_TRY(dalloc(&h->inc_ptr, (size_t)nn + 1, s, "incidence ptr"));
        TF_TRY(dalloc(&h->inc_cell, (size_t)mi, s, "incidence cells"));
        k_hz_starts<<<blocks(mi + 1), threads, 0, s>>>(ks, mi, nn, h->inc_ptr);
        TF_LAUNCH_CHECK();
        TF_CUDA_TRY(cudaMemcpyAsync(h->inc_cell, vs, (size_t)mi * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        TF_TRY(dalloc(&h->W, (size_t)nn, s, "node weights"));
        k_hz_node_weight<<<blocks(nn), threads, 0, s>>>(h->inc_ptr, (const uint32_t *)h->inc_cell, h->vol, nn, h->W);
        TF_LAUNCH_CHECK();
    }
    // ---- matrix: sort items by (row, col), t ascending inside a run
    const int64_t m = nc * D2;
    {
        DevBuf<uint32_t> k0, v0, k1, v1;
        TF_TRY(k0.alloc(m, s, "assembly keys"));
        TF_TRY(v0.alloc(m, s, "assembly vals"));
        TF_TRY(k1.alloc(m, s, "assembly keys alt"));
        TF_TRY(v1.alloc(m, s, "assembly vals alt"));
        k_hz_mat_items<D><<<blocks(m), threads, 0, s>>>(h->cells, nc, k0.p, v0.p);
        TF_LAUNCH_CHECK();
        uint32_t *ks, *vs;
        int passes;
        TF_TRY(radix_sort_pairs(k0.p, v0.p, k1.p, v1.p, m, nbits, s, &ks, &vs, &passes));
        // row keys for the column-sorted items, then the stable sort by row
        uint32_t *rk = (ks == k0.p) ? k1.p : k0.p;
        uint32_t *rv = (vs == v0.p) ? v1.p : v0.p;
        k_hz_row_keys<D><<<blocks(m), threads, 0, s>>>(h->cells, vs, m, rk);
        TF_LAUNCH_CHECK();
        TF_CUDA_TRY(cudaMemcpyAsync(rv, vs, (size_t)m * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        uint32_t *ks2, *vs2;
        TF_TRY(radix_sort_pairs(rk, rv, ks, vs, m, nbits, s, &ks2, &vs2, &passes));
        DevBuf<int32_t> head, rowcnt;
        DevBuf<int64_t> slot;
        TF_TRY(head.alloc(m, s, "assembly heads"));
        TF_TRY(rowcnt.alloc(nn, s, "assembly row counts"));
        TF_TRY(slot.alloc(m + 1, s, "assembly slots"));
        TF_CUDA_TRY(cudaMemsetAsync(rowcnt.p, 0, (size_t)nn * sizeof(int32_t), s));
        k_hz_heads<D><<<blocks(m), threads, 0, s>>>(h->cells, ks2, vs2, m, head.p, rowcnt.p);
        TF_LAUNCH_CHECK();
        TF_TRY(exclusive_scan_i32_i64(head.p, slot.p, m, s));
        TF_TRY(dalloc(&h->rowptr, (size_t)nn + 1, s, "helmholtz rowptr"));
        TF_TRY(exclusive_scan_i32_i64(rowcnt.p, h->rowptr, nn, s));
        int64_t last_slot = 0;
        int32_t last_head = 0;
        TF_CUDA_TRY(cudaMemcpyAsync(&last_slot, slot.p + (m - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        TF_CUDA_TRY(cudaMemcpyAsync(&last_head, head.p + (m - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        TF_CUDA_TRY(cudaStreamSynchronize(s));
        h->nnz = last_slot + last_head;
        TF_CUDA_TRY(cudaMemcpyAsync(h->rowptr + nn, &h->nnz, sizeof(int64_t), cudaMemcpyHostToDevice, s));
        TF_TRY(dalloc(&h->cols, (size_t)h->nnz, s, "helmholtz cols"));
        TF_TRY(dalloc(&h->valA, (size_t)h->nnz, s, "helmholtz A"));
        TF_TRY(dalloc(&h->valM, (size_t)h->nnz, s, "helmholtz M"));
        k_hz_entries<D><<<blocks(m), threads, 0, s>>>(h->cells, vs2, head.p, slot.p, m, h->vol, G.p, R * R, h->cols,
                                                       h->valA, h->valM);
        TF_LAUNCH_CHECK();
    }
    TF_TRY(dalloc(&h->dinv, (size_t)nn, s, "helmholtz diag"));
    k_hz_diag<<<blocks(nn), threads, 0, s>>>(h->rowptr, h->cols, h->valA, nn, h->dinv);
    TF_LAUNCH_CHECK();
    h->grid = hz_grid<D>(di, nn);
    TF_TRY(dalloc(&h->vec, (size_t)7 * nn, s, "helmholtz CG vectors"));
    TF_TRY(dalloc(&h->parts, (size_t)2 * h->grid * 4, s, "helmholtz partials"));
    TF_CUDA_TRY(cudaStreamSynchronize(s));  // h2d of nnz above reads a host stack value
    return TF_OK;
}

}  // namespace
}  // namespace tf

using namespace tf;

extern "C" {

TF_API tf_status tf_helmholtz_build(const double *nodes, int64_t n_nodes, const int32_t *cells, int64_t n_cells,
                                    int dim, double R, void *stream, tf_helmholtz *out) {
    if (!out) {
        set_error("tf_helmholtz_build: out is NULL");
        return TF_ERR_INVALID;
    }
    *out = nullptr;
    if (dim != 2 && dim != 3) {
        set_error("tf_helmholtz_build: dim must be 2 or 3 (got %d)", dim);
        return TF_ERR_INVALID;
    }
    if (n_nodes < 1 || n_nodes >= ((int64_t)1 << 31) || n_cells < 1) {
        set_error("tf_helmholtz_build: need 1 <= n_nodes < 2^31 and n_cells >= 1 (got %lld, %lld)",
                  (long long)n_nodes, (long long)n_cells);
        return TF_ERR_INVALID;
    }
    if (!(R >= 0.0) || !isfinite(R)) {
        set_error("tf_helmholtz_build: R must be finite and >= 0");
        return TF_ERR_INVALID;
    }
    const int64_t d1 = dim + 1;
    if (n_cells > (((int64_t)1 << 31) - 1) / (d1 * d1)) {
        set_error("tf_helmholtz_build: n_cells*(dim+1)^2 must be < 2^31");
        return TF_ERR_OVERFLOW;
    }
    TF_TRY(require_device(nodes, "tf_helmholtz_build: nodes"));
    TF_TRY(require_device(cells, "tf_helmholtz_build: cells"));
    tf_helmholtz_s *h = new tf_helmholtz_s;
    cudaGetDevice(&h->device);
    h->nn = n_nodes, h->nc = n_cells, h->dim = dim, h->R = R;
    cudaStream_t s = (cudaStream_t)stream;
    const tf_status st = (dim == 2) ? hz_build<2>(nodes, n_nodes, cells, n_cells, R, s, h)
                                    : hz_build<3>(nodes, n_nodes, cells, n_cells, R, s, h);
    if (st != TF_OK) {
        cudaStreamSynchronize(s);
        hz_destroy(h);
        return st;
    }
    *out = h;
    return TF_OK;
}

static tf_status hz_check(tf_helmholtz h, double rtol, int maxit, const char *who) {
    if (!h) {
        set_error("%s: handle is NULL", who);
        return TF_ERR_INVALID;
    }
    if (!(rtol > 0.0) || !isfinite(rtol) || maxit < 1) {
        set_error("%s: need rtol > 0 and maxit >= 1", who);
        return TF_ERR_INVALID;
    }
    return require_current_device(h->device, who);
}

TF_API tf_status tf_helmholtz_filter(tf_helmholtz h, const double *sigma, double *out, double rtol, int maxit,
                                     tf_helmholtz_info *info, void *stream) {
    TF_TRY(hz_check(h, rtol, maxit, "tf_helmholtz_filter"));
    TF_TRY(require_device(sigma, "tf_helmholtz_filter: sigma"));
    TF_TRY(require_device(out, "tf_helmholtz_filter: out"));
    if (info) TF_TRY(require_device(info, "tf_helmholtz_filter: info"));
    NvtxRange nv("tf_helmholtz_filter");
    cudaStream_t s = (cudaStream_t)stream;
    return (h->dim == 2) ? hz_launch<2, false>(h, sigma, nullptr, nullptr, out, rtol, maxit, info, s)
                         : hz_launch<3, false>(h, sigma, nullptr, nullptr, out, rtol, maxit, info, s);
}

TF_API tf_status tf_helmholtz_sensitivity(tf_helmholtz h, const double *x, const double *dc, double *out,
                                          double rtol, int maxit, tf_helmholtz_info *info, void *stream) {
    TF_TRY(hz_check(h, rtol, maxit, "tf_helmholtz_sensitivity"));
    TF_TRY(require_device(x, "tf_helmholtz_sensitivity: x"));
    TF_TRY(require_device(dc, "tf_helmholtz_sensitivity: dc"));
    TF_TRY(require_device(out, "tf_helmholtz_sensitivity: out"));
    if (out == x) {
        set_error("tf_helmholtz_sensitivity: out must not alias x");
        return TF_ERR_INVALID;
    }
    if (info) TF_TRY(require_device(info, "tf_helmholtz_sensitivity: info"));
    NvtxRange nv("tf_helmholtz_sensitivity");
    cudaStream_t s = (cudaStream_t)stream;
    return (h->dim == 2) ? hz_launch<2, true>(h, nullptr, x, dc, out, rtol, maxit, info, s)
                         : hz_launch<3, true>(h, nullptr, x, dc, out, rtol, maxit, info, s);
}

TF_API tf_status tf_helmholtz_view(tf_helmholtz h, tf_helmholtz_system *v) {
    if (!h || !v) {
        set_error("tf_helmholtz_view: NULL argument");
        return TF_ERR_INVALID;
    }
    v->n_nodes = h->nn, v->n_cells = h->nc, v->nnz = h->nnz, v->dim = h->dim, v->R = h->R;
    v->rowptr = h->rowptr, v->cols = h->cols, v->vals_A = h->valA, v->vals_M = h->valM;
    v->node_weight = h->W, v->cell_volume = h->vol;
    return TF_OK;
}

TF_API void tf_helmholtz_free(tf_helmholtz h) { hz_destroy(h); }

}  // extern "C"
