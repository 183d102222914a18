// apply.cu -- the per-iteration filter applies.
//
//   sensitivity  out_i = (sum_k vals[k] * (x[cols[k]] * dc[cols[k]])) / (Hs_i * max(1e-3, x_i))
//                (Eq. filter, Eq. filter_mat, listing
//                the paper's dense GEMV becomes a CSR SpMV, with the
//                Hadamard product, the max floor and the division fused in)
//   density      out_i = (sum_k vals[k] * x[cols[k]]) / Hs_i   (BASELINE.json north_star)
//
// Work split ("CSR-stream"): the nnz stream is cut into windows of kWindow entries; block b
// owns the rows whose first entry falls in window b (row-block table rb[], built once per
// filter by make_apply_plan). A block streams its contiguous nnz range with coalesced
// loads, forms the products into shared memory, then one warp per row reduces its segment
// (lane-strided partial sums + xor-shuffle tree: deterministic, no atomics). Rows that make
// a block's range exceed the staging capacity are reduced one at a time by the whole block.
//
// Roofline: HBM. Algorithmic bytes per apply = 12*nnz + 8(N+1) + 32N (sensitivity) or
// + 24N (density); gathers of x/dc hit L2/L1 (neighbour columns are index-local).
#include <algorithm>

#include "tf_internal.cuh"

namespace tf {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kWindow = 2048;   // target nnz per block
constexpr int kStage = 4096;    // shared-memory staging capacity (doubles)

__global__ void k_plan(const int64_t *__restrict__ rowptr, int64_t n, int64_t nblocks, int32_t *__restrict__ rb) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nblocks;
         b += (int64_t)gridDim.x * blockDim.x) {
        if (b == nblocks) {
            rb[b] = (int32_t)n;
            continue;
        }
        const int64_t target = b * (int64_t)kWindow;
        int64_t lo = 0, hi = n;  // first r in [0, n] with rowptr[r] >= target
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (rowptr[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        rb[b] = (int32_t)lo;
    }
}

template <bool SENS>
__device__ __forceinline__ double finish(double acc, double hs_i, double x_i) {
    if (SENS) return acc / (hs_i * fmax(1e-3, x_i));
    return acc / hs_i;
}

template <bool SENS>
__global__ void __launch_bounds__(kThreads) k_spmv(const int64_t *__restrict__ rowptr,
                                                   const int32_t *__restrict__ cols,
                                                   const double *__restrict__ vals,
                                                   const double *__restrict__ hs,
                                                   const double *__restrict__ x,
                                                   const double *__restrict__ dc,
                                                   double *__restrict__ out,
                                                   const int32_t *__restrict__ rb) {
    __shared__ double prod[kStage];
    __shared__ double red[kWarps];
    const int r0 = rb[blockIdx.x], r1 = rb[blockIdx.x + 1];
    if (r0 >= r1) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t k0 = rowptr[r0], k1 = rowptr[r1];
    const int64_t L = k1 - k0;
    if (L <= kStage) {
        for (int i = tid; i < (int)L; i += kThreads) {
            const int64_t k = k0 + i;
            const int32_t j = __ldg(cols + k);
            const double v = __ldg(vals + k);
            const double t = SENS ? __ldg(x + j) * __ldg(dc + j) : __ldg(x + j);
            prod[i] = v * t;
        }
        __syncthreads();
        for (int r = r0 + warp; r < r1; r += kWarps) {
            const int s = (int)(rowptr[r] - k0), e = (int)(rowptr[r + 1] - k0);
            double acc = 0.0;
            for (int i = s + lane; i < e; i += 32) acc += prod[i];
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) out[r] = finish<SENS>(acc, hs[r], x[r]);
        }
    } else {
        for (int r = r0; r < r1; ++r) {
            const int64_t s = rowptr[r], e = rowptr[r + 1];
            double acc = 0.0;
            for (int64_t k = s + tid; k < e; k += kThreads) {
                const int32_t j = cols[k];
                const double t = SENS ? x[j] * dc[j] : x[j];
                acc += vals[k] * t;
            }
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) red[warp] = acc;
            __syncthreads();
            if (tid == 0) {
                double a = 0.0;
                for (int w = 0; w < kWarps; ++w) a += red[w];
                out[r] = finish<SENS>(a, hs[r], x[r]);
            }
            __syncthreads();
        }
    }
}

}  // namespace

tf_status make_apply_plan(tf_filter_s *h, cudaStream_t s) {
    const int64_t nblocks = std::max<int64_t>(1, (h->nnz + kWindow - 1) / kWindow);
    if (nblocks >= (int64_t)1 << 31) {
        set_error("apply plan: too many row blocks");
        return TF_ERR_OVERFLOW;
    }
    TF_TRY(dalloc(&h->plan.rb, nblocks + 1, s, "apply row blocks"));
    h->plan.nblocks = nblocks;
    h->plan.block_nnz = kWindow;
    h->plan.stage_cap = kStage;
    const unsigned grid = (unsigned)std::min<int64_t>((nblocks + 256) / 256, 65535);
    k_plan<<<grid, 256, 0, s>>>(h->rowptr, h->n, nblocks, h->plan.rb);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

tf_status launch_sensitivity(const tf_filter_s *h, const double *x, const double *dc, double *out,
                             cudaStream_t s) {
    k_spmv<true><<<(unsigned)h->plan.nblocks, kThreads, 0, s>>>(h->rowptr, h->cols, h->vals, h->hs, x, dc, out,
                                                                h->plan.rb);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

tf_status launch_density(const tf_filter_s *h, const double *x, double *out, cudaStream_t s) {
    k_spmv<false><<<(unsigned)h->plan.nblocks, kThreads, 0, s>>>(h->rowptr, h->cols, h->vals, h->hs, x, nullptr,
                                                                 out, h->plan.rb);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

}  // namespace tf
