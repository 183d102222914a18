// dense_build.cu -- ABLATION, not a product path: the paper's own filter build mapped to the GPU.
//
// The paper builds the filter from the full N x N Euclidean distance matrix of the cell midpoints
// (Eq. EDM; listing PAPER.md:442-445: distance matrix, rmin - distance, clip at 0,
// row sums), i.e. every pair (i, j) is visited. This file does exactly that, tile by tile, without
// ever storing the N x N matrix (the paper's memory wall: 8 GB at ~32k cells): a count
// pass and a fill pass over all N^2 pairs, with the library's exact pair expression
// (d2 = (dx*dx + dy*dy) + dz*dz, uncontracted; w = max(0, rmin - sqrt(d2))) instead of the EDM
// expansion |x|^2 - 2x.y + |y|^2, which cancels (R2). The CSR it produces is the cell
// list's and the oracle's, bit for bit -- columns ascend because j does --, and Hs is accumulated in
// ascending j like the oracle's, so it is bitwise the oracle's too.
//
// It exists to measure what the cell list buys on the same hardware (last
// paragraph; tools/dense_probe.py): O(N^2) exact fp64 pair tests against O(N * neighbourhood).
// Reached only through tf_build_filter_ex(..., TF_BUILD_DENSE, ...).
#include <math.h>

#include <algorithm>

#include "tf_internal.cuh"

namespace tf {
namespace {

constexpr int kRows = 128;  // rows (threads) per block
constexpr int kTileJ = 512; // columns staged per step

// Thread = row i; the block walks all columns in tiles staged in shared memory (SoA fp64, every
// lane reads the same column: broadcast loads). FILL = false: row lengths (and a non-finite flag);
// FILL = true: cols, vals at rowptr[i] + rank, Hs in ascending j.
template <int DIM, bool FILL>
__global__ void __launch_bounds__(kRows) k_dense(const double *__restrict__ c, int64_t n, double rmin, double r2,
                                                 const int64_t *__restrict__ rowptr, int32_t *__restrict__ counts,
                                                 int32_t *__restrict__ cols, double *__restrict__ vals,
                                                 double *__restrict__ hs, int32_t *__restrict__ stats) {
    __shared__ double sx[kTileJ], sy[kTileJ], sz[kTileJ];
    const int64_t i = (int64_t)blockIdx.x * kRows + threadIdx.x;
    const bool have = i < n;
    double qx = 0.0, qy = 0.0, qz = 0.0;
    if (have) {
        qx = c[i * DIM];
        qy = c[i * DIM + 1];
        qz = (DIM == 3) ? c[i * DIM + 2] : 0.0;
    }
    int bad = 0;
    if (!FILL) bad = have && !(isfinite(qx) && isfinite(qy) && isfinite(qz));
    int64_t k = (FILL && have) ? rowptr[i] : 0;
    int cnt = 0;
    double hsum = 0.0;
    for (int64_t j0 = 0; j0 < n; j0 += kTileJ) {
        const int len = (int)std::min<int64_t>(kTileJ, n - j0);
        __syncthreads();
        for (int t = threadIdx.x; t < len; t += kRows) {
            sx[t] = c[(j0 + t) * DIM];
            sy[t] = c[(j0 + t) * DIM + 1];
            if (DIM == 3) sz[t] = c[(j0 + t) * DIM + 2];
        }
        __syncthreads();
        if (!have) continue;
#pragma unroll 4
        for (int t = 0; t < len; ++t) {
            const double d2 = pair_d2<DIM>(qx, qy, qz, sx[t], sy[t], (DIM == 3) ? sz[t] : 0.0);
            if (d2 < r2) {
                if (FILL) {
                    const double w = weight_of(rmin, d2);
                    cols[k] = (int32_t)(j0 + t);
                    vals[k] = w;
                    ++k;
                    hsum += w;
                } else {
                    ++cnt;
                }
            }
        }
    }
    if (FILL) {
        if (have) hs[i] = hsum;
    } else {
        if (have) counts[i] = cnt;
        int m = cnt;
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        bad = __any_sync(0xffffffffu, bad);
        if ((threadIdx.x & 31) == 0) {
            if (m > stats[3]) atomicMax(&stats[3], m);  // longest row (apply plan)
            if (bad) atomicOr(&stats[1], 1);
        }
    }
}

template <int DIM>
tf_status dense_impl(const double *c, int64_t n, double rmin, cudaStream_t s, tf_filter_s *h) {
    const double r2 = rmin * rmin;
    const unsigned blocks = (unsigned)((n + kRows - 1) / kRows);
    DevBuf<int32_t> counts, stats;
    TF_TRY(counts.alloc(n, s, "row counts"));
    TF_TRY(stats.alloc(4, s, "build stats"));
    TF_CUDA_TRY(cudaMemsetAsync(stats.p, 0, 4 * sizeof(int32_t), s));
    k_dense<DIM, false><<<blocks, kRows, 0, s>>>(c, n, rmin, r2, nullptr, counts.p, nullptr, nullptr, nullptr, stats.p);
    TF_LAUNCH_CHECK();
    build_trace().mark("dense count", s);
    TF_TRY(dalloc(&h->rowptr, n + 3, s, "rowptr (+2 padding for 16-byte bulk copies)"));
    TF_TRY(exclusive_scan_i32_i64(counts.p, h->rowptr, n, s));
    int64_t nnz = 0;
    int32_t hst[4] = {0, 0, 0, 0};
    TF_CUDA_TRY(cudaMemcpyAsync(&nnz, h->rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaMemcpyAsync(hst, stats.p, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    build_trace().mark("scan+sync", s);
    if (hst[1] != 0) {
        set_error("tf_build_filter: non-finite centroid coordinate (NaN or Inf)");
        return TF_ERR_INVALID;
    }
    if (nnz < n) {
        set_error("internal: nnz %lld < n %lld", (long long)nnz, (long long)n);
        return TF_ERR_CUDA;
    }
    h->nnz = nnz;
    h->max_row_hint = hst[3];
    TF_TRY(dalloc(&h->cols, nnz + 4, s, "cols (nnz int32, +4 padding for 16-byte bulk copies)"));
    TF_TRY(dalloc(&h->vals, nnz + 4, s, "vals (nnz fp64, +4 padding)"));
    TF_TRY(dalloc(&h->hs, n, s, "Hs"));
    k_dense<DIM, true><<<blocks, kRows, 0, s>>>(c, n, rmin, r2, h->rowptr, nullptr, h->cols, h->vals, h->hs, stats.p);
    TF_LAUNCH_CHECK();
    build_trace().mark("dense fill", s);
    return TF_OK;
}

}  // namespace

tf_status build_dense_csr(const double *c, int64_t n, int dim, double rmin, cudaStream_t s, tf_filter_s *h) {
    h->info.path = TF_PATH_DENSE;
    return dim == 3 ? dense_impl<3>(c, n, rmin, s, h) : dense_impl<2>(c, n, rmin, s, h);
}

}  // namespace tf
