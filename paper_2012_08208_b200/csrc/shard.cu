// shard.cu -- NEXT-4: the slab partition of one filter problem over several
// GPUs, computed on the device (tf_shard_plan). The paper's parallel section
// partitions the mesh across MPI ranks and notes that a partition starves the distance filter of
// neighbour midpoints; here each rank receives exactly those neighbours as a halo.
//
// Partition (identical on every rank, from the same centroids):
//   * bounding box (k_sh_bbox), longest axis a;
//   * a histogram of coordinate a over kShBuckets buckets of the box (k_sh_hist), prefix-summed on
//     the host: slab k = buckets [cb_k, cb_{k+1}), cut where the running count first reaches
//     k*n/W (balanced by count; points with equal coordinates share a bucket, so they stay
//     together). Every point's owner is a pure function of its bucket, so owner and slab agree by
//     construction.
//   * rank k's window = [lo_k - r', hi_k + r') with lo_k/hi_k the slab's coordinate bounds
//     (-inf/+inf at the ends) and r' = rmin(1 + 1e-9) + slack for the bucket rounding: every
//     neighbour of an owned point lies in owned + halo (halo = other ranks' points in the window);
//     extra halo points are harmless. Owned points at least r' inside both slab faces are
//     INTERIOR (no halo neighbour), the rest BOUNDARY.
//   * local order: [interior | boundary | halo by source rank], each ascending global id
//     (k_sh_class + one stable radix pass on the class); send list to rank j = my owned points in
//     j's window, ascending global id, as LOCAL indices (the order rank j receives them in).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <vector>

#include "tf_internal.cuh"

namespace tf {
namespace {

constexpr int kShBuckets = 1 << 16;
constexpr int kShThreads = 256;

__global__ void __launch_bounds__(kShThreads) k_sh_bbox(const double *__restrict__ c, int64_t n, int dim,
                                                        double *__restrict__ part) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        for (int d = 0; d < dim; ++d) {
            const double v = c[i * dim + d];
            bad |= !isfinite(v);
            lo[d] = fmin(lo[d], v);
            hi[d] = fmax(hi[d], v);
        }
    __shared__ double s[kShThreads / 32][7];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = 0; d < 3; ++d)
        for (int o = 16; o > 0; o >>= 1) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        for (int d = 0; d < 3; ++d) s[warp][d] = lo[d], s[warp][3 + d] = hi[d];
        s[warp][6] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kShThreads / 32; ++w) {
            for (int d = 0; d < 3; ++d) s[0][d] = fmin(s[0][d], s[w][d]), s[0][3 + d] = fmax(s[0][3 + d], s[w][3 + d]);
            s[0][6] = fmax(s[0][6], s[w][6]);
        }
        for (int k = 0; k < 7; ++k) part[blockIdx.x * 7 + k] = s[0][k];
    }
}

struct Axis {
    int a, dim;
    double lo, inv_w;  // bucket b = clamp(floor((c_a - lo) * inv_w), 0, kShBuckets - 1)
};

__device__ __forceinline__ int bucket_of(double v, const Axis &A) {
    const double f = floor((v - A.lo) * A.inv_w);
    return f < 0.0 ? 0 : (f > (double)(kShBuckets - 1) ? kShBuckets - 1 : (int)f);
}

__global__ void __launch_bounds__(kShThreads) k_sh_hist(const double *__restrict__ c, int64_t n, Axis A,
                                                        int32_t *__restrict__ hist) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&hist[bucket_of(c[i * A.dim + A.a], A)], 1);
}

// Slab table of every rank (constant memory would do; a small kernel argument struct is enough).
constexpr int kMaxRanks = 64;
struct Slabs {
    int W, me;
    int cb[kMaxRanks + 1];     // first bucket of each slab; cb[W] = kShBuckets
    double wlo[kMaxRanks];     // window lower bound of each rank (-inf for rank 0)
    double whi[kMaxRanks];     // window upper bound (+inf for the last rank)
    double ilo, ihi;           // interior band of rank me
};

__device__ __forceinline__ int owner_of(int b, const Slabs &S) {
    int k = 0;
    while (k + 1 < S.W && b >= S.cb[k + 1]) ++k;
    return k;
}

// class of each point for rank me: 0 interior, 1 boundary, 2 + src halo from src, 255 not local
__global__ void __launch_bounds__(kShThreads) k_sh_class(const double *__restrict__ c, int64_t n, Axis A, Slabs S,
                                                         uint32_t *__restrict__ key, uint32_t *__restrict__ ids) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = c[i * A.dim + A.a];
        const int o = owner_of(bucket_of(v, A), S);
        uint32_t k = 255;
        if (o == S.me) k = (v >= S.ilo && v < S.ihi) ? 0u : 1u;
        else if (v >= S.wlo[S.me] && v < S.whi[S.me]) k = 2u + (uint32_t)o;
        key[i] = k;
        ids[i] = (uint32_t)i;
    }
}

__global__ void __launch_bounds__(kShThreads) k_sh_count_classes(const uint32_t *__restrict__ key, int64_t n,
                                                                 int32_t *__restrict__ cnt) {
    __shared__ int32_t h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&h[key[i] & 255u], 1);
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd(&cnt[i], h[i]);
}

// flag[i] = 1 if point i is owned by me and lies in rank j's window
__global__ void __launch_bounds__(kShThreads) k_sh_sendflag(const double *__restrict__ c, int64_t n, Axis A, Slabs S,
                                                            int j, int32_t *__restrict__ flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = c[i * A.dim + A.a];
        flag[i] = (owner_of(bucket_of(v, A), S) == S.me && v >= S.wlo[j] && v < S.whi[j]) ? 1 : 0;
    }
}

// send[pos[i]] = local[i] for flagged i (pos = exclusive scan of flag): ascending global id
__global__ void __launch_bounds__(kShThreads) k_sh_sendlist(const int32_t *__restrict__ flag,
                                                            const int64_t *__restrict__ pos,
                                                            const int32_t *__restrict__ local, int64_t n,
                                                            int32_t *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (flag[i]) out[pos[i]] = local[i];
}

// local[id] = position of an owned point in the local order (sorted ids of classes 0 and 1)
__global__ void __launch_bounds__(kShThreads) k_sh_inverse(const uint32_t *__restrict__ sorted_ids, int64_t n_owned,
                                                           int32_t *__restrict__ local) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_owned; t += (int64_t)gridDim.x * blockDim.x)
        local[sorted_ids[t]] = (int32_t)t;
}

__global__ void __launch_bounds__(kShThreads) k_sh_gather_rows(const double *__restrict__ src, int dim,
                                                               const int32_t *__restrict__ idx, int64_t m,
                                                               double *__restrict__ dst) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m * dim; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / dim;
        dst[t] = src[(int64_t)idx[r] * dim + (t - r * dim)];
    }
}

}  // namespace

tf_status shard_plan(const double *c, int64_t n, int dim, double rmin, int W, int me, cudaStream_t s,
                     tf_shard_s *p) {
    DeviceInfo di;
    TF_TRY(device_info(&di));
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kShThreads - 1) / kShThreads, (int64_t)di.sms * 8));
    DevBuf<double> part;
    TF_TRY(part.alloc((size_t)grid * 7, s, "shard bbox partials"));
    k_sh_bbox<<<grid, kShThreads, 0, s>>>(c, n, dim, part.p);
    TF_LAUNCH_CHECK();
    std::vector<double> hp((size_t)grid * 7);
    TF_CUDA_TRY(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (unsigned b = 0; b < grid; ++b) {
        for (int d = 0; d < 3; ++d) lo[d] = fmin(lo[d], hp[b * 7 + d]), hi[d] = fmax(hi[d], hp[b * 7 + 3 + d]);
        if (hp[b * 7 + 6] != 0.0) {
            set_error("tf_shard_plan: non-finite centroid coordinate (NaN or Inf)");
            return TF_ERR_INVALID;
        }
    }
    Axis A;
    A.dim = dim;
    A.a = 0;
    for (int d = 1; d < dim; ++d)
        if (hi[d] - lo[d] > hi[A.a] - lo[A.a]) A.a = d;
    const double span = hi[A.a] - lo[A.a];
    const double width = (span > 0.0) ? span / (double)kShBuckets : 1.0;
    A.lo = lo[A.a];
    A.inv_w = 1.0 / width;
    DevBuf<int32_t> hist;
    TF_TRY(hist.alloc(kShBuckets, s, "shard histogram"));
    TF_CUDA_TRY(cudaMemsetAsync(hist.p, 0, kShBuckets * sizeof(int32_t), s));
    k_sh_hist<<<grid, kShThreads, 0, s>>>(c, n, A, hist.p);
    TF_LAUNCH_CHECK();
    std::vector<int32_t> hh(kShBuckets);
    TF_CUDA_TRY(cudaMemcpyAsync(hh.data(), hist.p, kShBuckets * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    // cuts: slab k starts at the first bucket where the running count reaches k*n/W
    Slabs S;
    S.W = W;
    S.me = me;
    {
        int64_t run = 0;
        int k = 1;
        S.cb[0] = 0;
        for (int b = 0; b < kShBuckets && k < W; ++b) {
            while (k < W && run >= (n * k) / W) S.cb[k++] = b;
            run += hh[b];
        }
        while (k < W) S.cb[k++] = kShBuckets;
        S.cb[W] = kShBuckets;
    }
    // window bounds: slab k covers coordinates [lo + cb_k w, lo + cb_{k+1} w) up to the bucket
    // rounding (a few ulps of the coordinates), widened by rmin(1 + 1e-9) + that slack
    const double slack = 1e-12 * (fabs(lo[A.a]) + fabs(hi[A.a]) + span) + 4.0 * width * 1e-12;
    const double rr = rmin * (1.0 + 1e-9) + slack;
    for (int k = 0; k < W; ++k) {
        const double slo = A.lo + (double)S.cb[k] * width, shi = A.lo + (double)S.cb[k + 1] * width;
        S.wlo[k] = (k == 0 || S.cb[k] == 0) ? -INFINITY : slo - rr;
        S.whi[k] = (k == W - 1 || S.cb[k + 1] >= kShBuckets) ? INFINITY : shi + rr;
    }
    {
        const double slo = A.lo + (double)S.cb[me] * width, shi = A.lo + (double)S.cb[me + 1] * width;
        S.ilo = (me == 0 || S.cb[me] == 0) ? -INFINITY : slo + rr;
        S.ihi = (me == W - 1 || S.cb[me + 1] >= kShBuckets) ? INFINITY : shi - rr;
    }
    p->axis = A.a;
    p->cut_lo = (me == 0) ? -INFINITY : A.lo + (double)S.cb[me] * width;
    p->cut_hi = (me == W - 1) ? INFINITY : A.lo + (double)S.cb[me + 1] * width;
    // classes -> one stable radix pass -> local order [interior | boundary | halo by source]
    DevBuf<uint32_t> k0, v0, k1, v1;
    TF_TRY(k0.alloc(n, s, "shard classes"));
    TF_TRY(v0.alloc(n, s, "shard ids"));
    TF_TRY(k1.alloc(n, s, "shard classes (alt)"));
    TF_TRY(v1.alloc(n, s, "shard ids (alt)"));
    k_sh_class<<<grid, kShThreads, 0, s>>>(c, n, A, S, k0.p, v0.p);
    TF_LAUNCH_CHECK();
    uint32_t *ks = nullptr, *vs = nullptr;
    int passes = 0;
    TF_TRY(radix_sort_pairs(k0.p, v0.p, k1.p, v1.p, n, 8, s, &ks, &vs, &passes));
    // class sizes (a 256-bin histogram of the keys)
    DevBuf<int32_t> ccount;
    TF_TRY(ccount.alloc(256, s, "shard class counts"));
    TF_CUDA_TRY(cudaMemsetAsync(ccount.p, 0, 256 * sizeof(int32_t), s));
    k_sh_count_classes<<<grid, kShThreads, 0, s>>>(ks, n, ccount.p);
    TF_LAUNCH_CHECK();
    std::vector<int32_t> cc(256);
    TF_CUDA_TRY(cudaMemcpyAsync(cc.data(), ccount.p, 256 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    p->n_interior = cc[0];
    p->n_owned = (int64_t)cc[0] + cc[1];
    p->recv.assign(W, 0);
    int64_t nh = 0;
    for (int k = 0; k < W; ++k) p->recv[k] = (k == me) ? 0 : cc[2 + k], nh += p->recv[k];
    p->n_halo = nh;
    const int64_t nloc = p->n_owned + nh;
    TF_TRY(dalloc(&p->local_ids, std::max<int64_t>(1, nloc), s, "shard local ids"));
    TF_CUDA_TRY(cudaMemcpyAsync(p->local_ids, vs, nloc * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    // send lists: my owned points in rank j's window, ascending id, as local indices
    DevBuf<int32_t> local, flag;
    DevBuf<int64_t> pos;
    TF_TRY(local.alloc(n, s, "shard inverse"));
    TF_TRY(flag.alloc(n, s, "shard send flags"));
    TF_TRY(pos.alloc(n + 1, s, "shard send positions"));
    k_sh_inverse<<<grid, kShThreads, 0, s>>>(vs, p->n_owned, local.p);
    TF_LAUNCH_CHECK();
    p->send.assign(W, 0);
    std::vector<int64_t> soff(W + 1, 0);
    std::vector<int32_t *> lists(W, nullptr);
    for (int j = 0; j < W; ++j) {
        if (j == me || p->n_owned == 0) continue;
        // only ranks whose window overlaps my slab can need my points
        if (!(S.wlo[j] < p->cut_hi && S.whi[j] > p->cut_lo)) continue;
        k_sh_sendflag<<<grid, kShThreads, 0, s>>>(c, n, A, S, j, flag.p);
        TF_LAUNCH_CHECK();
        TF_TRY(exclusive_scan_i32_i64(flag.p, pos.p, n, s));
        int64_t m = 0;
        TF_CUDA_TRY(cudaMemcpyAsync(&m, pos.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        TF_CUDA_TRY(cudaStreamSynchronize(s));
        p->send[j] = m;
        if (m == 0) continue;
        TF_TRY(dalloc(&lists[j], m, s, "shard send list"));
        k_sh_sendlist<<<grid, kShThreads, 0, s>>>(flag.p, pos.p, local.p, n, lists[j]);
        TF_LAUNCH_CHECK();
    }
    int64_t ns = 0;
    for (int j = 0; j < W; ++j) soff[j] = ns, ns += p->send[j];
    soff[W] = ns;
    TF_TRY(dalloc(&p->send_idx, std::max<int64_t>(1, ns), s, "shard send indices"));
    for (int j = 0; j < W; ++j) {
        if (!lists[j]) continue;
        TF_CUDA_TRY(cudaMemcpyAsync(p->send_idx + soff[j], lists[j], p->send[j] * sizeof(int32_t),
                                    cudaMemcpyDeviceToDevice, s));
        dev_free(lists[j], s);
    }
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    return TF_OK;
}

tf_status launch_gather_rows(const double *src, int dim, const int32_t *idx, int64_t m, double *dst, cudaStream_t s) {
    if (m <= 0) return TF_OK;
    const unsigned grid = (unsigned)std::min<int64_t>((m * dim + 255) / 256, 148 * 8);
    k_sh_gather_rows<<<grid, kShThreads, 0, s>>>(src, dim, idx, m, dst);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

}  // namespace tf
