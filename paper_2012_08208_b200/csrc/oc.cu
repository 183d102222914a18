// oc.cu -- NEXT-1: optimality-criteria update with bisection on the Lagrange
// multiplier, consuming the sensitivity filter's output (Eq. update PAPER.md:218-228;
// bisection PAPER.md:229-234; listing PAPER.md:380-385):
//
//   while l2 - l1 > tol:
//       l_mid = 0.5 * (l2 + l1)
//       d_new = max(0.001, max(d - move, min(1, min(d + move, d * sqrt(-dc / l_mid)))))
//       l1, l2 = (l_mid, l2) if sum(d_new) > volfrac * N else (l1, l_mid)
//
// One cooperative persistent launch runs the whole bisection. Each iteration is a grid-stride
// pass (alternating direction, so the most recently touched ~126 MB of x/dc is still in L2
// when the next pass starts) that accumulates the EXACT sum of d_new -- every d_new in
// [0.001, 1] is an integer multiple of 2^-62, so the per-thread, per-block and global sums
// are 128-bit integers (R15; order-independent, bitwise-reproducible decisions).
// Block partials go to a double-buffered array, one grid.sync() per iteration, and every
// block then sums the partials in the same fixed order and takes the same decision. A final
// pass writes d_new at the last l_mid. d_new uses __ddiv_rn/__dsqrt_rn (correctly rounded,
// like the oracle), so the result is bitwise identical to the oracle.
#include <cooperative_groups.h>
#include <math.h>

#include <algorithm>

#include "tf_internal.cuh"

namespace tf {
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ double np_max(double a, double b) {
    return (a != a || b != b) ? (a != a ? a : b) : (a > b ? a : b);
}
__device__ __forceinline__ double np_min(double a, double b) {
    return (a != a || b != b) ? (a != a ? a : b) : (a < b ? a : b);
}

__device__ __forceinline__ double oc_value(double d, double dc, double lmid, double move) {
    const double s = __dsqrt_rn(__ddiv_rn(-dc, lmid));
    return np_max(0.001, np_max(__dsub_rn(d, move), np_min(1.0, np_min(__dadd_rn(d, move), __dmul_rn(d, s)))));
}

// block partial: (lo, hi) of the 128-bit sum; bit 63 of hi flags a NaN (sums stay < 2^93)
constexpr unsigned long long kNanBit = 1ull << 63;

constexpr int kOcThreads = 256;
#ifndef TF_OC_UNROLL
#define TF_OC_UNROLL 8
#endif
constexpr int kOcUnroll = TF_OC_UNROLL;

constexpr int kOcMaxIter = 4096;  // safety cap (reading R23); fp64 halvings end in < 2100 steps

// v * 2^62 as an exact 128-bit integer, for finite v >= 2^-10 (every x_new >= 0.001 qualifies; the
// bound v <= 1 holds for x in [0, 1] but is not relied on)
__device__ __forceinline__ u128 units62(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const int e = (int)((b >> 52) & 0x7ff) - 1023;
    const unsigned long long m = (b & ((1ull << 52) - 1)) | (1ull << 52);
    return (u128)m << (e + 10);  // v * 2^62 = m * 2^(e - 52 + 62), e >= -10
}

// x and xnew may alias (the header allows x_new == x): no __restrict__ on them
__global__ void __launch_bounds__(kOcThreads) k_oc(const double *x, const double *__restrict__ dc,
                                                   int64_t n, double move, double l1, double l2, double tol,
                                                   unsigned long long t_lo, unsigned long long t_hi,
                                                   ulonglong2 *__restrict__ parts, double *xnew,
                                                   double *__restrict__ lmid_out, int *__restrict__ iters_out) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const u128 T = ((u128)t_hi << 64) | (u128)t_lo;
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t last = (n - 1 - gid) >= 0 ? gid + ((n - 1 - gid) / stride) * stride : -1;
    __shared__ unsigned long long s_lo[kOcThreads / 32], s_hi[kOcThreads / 32];
    __shared__ int s_nan[kOcThreads / 32];
    __shared__ int s_up;
    double lmid = 0.5 * (l2 + l1);
    int it = 0, all_up = 1, stalled = 0;
    while (l2 - l1 > tol) {  // identical fp values in every thread: uniform trip count
        lmid = 0.5 * (l2 + l1);
        if (lmid == l1 || lmid == l2 || it >= kOcMaxIter) {  // no progress possible (reading R23)
            stalled = 1;
            break;
        }
        u128 acc = 0;
        int nan = 0;
        auto add = [&](double xi, double dci) {
            const double v = oc_value(xi, dci, lmid, move);
            if (v != v) nan = 1;
            else acc += units62(v);  // exact: v >= 0.001 is a multiple of 2^-62
        };
        // kOcUnroll elements per thread in flight (loads first): with one element per thread per
        // step the pass was latency-bound (ncu: 24% DRAM, 50% issue). Config 5, 30 passes:
        // U = 1 1776 us, 4 1486 us, 8 1402 us, 16 1662 us (117 registers). Integer sums: order-free.
        if (it & 1) {
            int64_t i = last;
            for (; i - (kOcUnroll - 1) * stride >= 0; i -= kOcUnroll * stride) {
                double xv[kOcUnroll], dv[kOcUnroll];
#pragma unroll
                for (int u = 0; u < kOcUnroll; ++u) xv[u] = __ldcg(x + i - u * stride), dv[u] = __ldcg(dc + i - u * stride);
#pragma unroll
                for (int u = 0; u < kOcUnroll; ++u) add(xv[u], dv[u]);
            }
            for (; i >= 0; i -= stride) add(__ldcg(x + i), __ldcg(dc + i));
        } else {
            int64_t i = gid;
            for (; i + (kOcUnroll - 1) * stride < n; i += kOcUnroll * stride) {
                double xv[kOcUnroll], dv[kOcUnroll];
#pragma unroll
                for (int u = 0; u < kOcUnroll; ++u) xv[u] = __ldcg(x + i + u * stride), dv[u] = __ldcg(dc + i + u * stride);
#pragma unroll
                for (int u = 0; u < kOcUnroll; ++u) add(xv[u], dv[u]);
            }
            for (; i < n; i += stride) add(__ldcg(x + i), __ldcg(dc + i));
        }
        // block reduction of the 128-bit sums (integer: order does not matter)
        unsigned long long lo = (unsigned long long)acc, hi = (unsigned long long)(acc >> 64);
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long olo = __shfl_xor_sync(0xffffffffu, lo, o);
            const unsigned long long ohi = __shfl_xor_sync(0xffffffffu, hi, o);
            const u128 s = (((u128)hi << 64) | lo) + (((u128)ohi << 64) | olo);
            lo = (unsigned long long)s, hi = (unsigned long long)(s >> 64);
            nan |= __shfl_xor_sync(0xffffffffu, nan, o);
        }
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) s_lo[warp] = lo, s_hi[warp] = hi, s_nan[warp] = nan;
        __syncthreads();
        if (threadIdx.x == 0) {
            u128 b = 0;
            int bn = 0;
            for (int w = 0; w < kOcThreads / 32; ++w) b += ((u128)s_hi[w] << 64) | s_lo[w], bn |= s_nan[w];
            parts[(size_t)(it & 1) * gridDim.x + blockIdx.x] =
                make_ulonglong2((unsigned long long)b, (unsigned long long)(b >> 64) | (bn ? kNanBit : 0ull));
        }
        grid.sync();
        {
            // every block sums all partials (integer: any order gives the same total) with all its
            // threads -> the same decision everywhere; __ldcg: the buffer was last read two
            // iterations ago, so bypass possibly stale L1 lines
            u128 S = 0;
            int sn = 0;
            const ulonglong2 *pp = parts + (size_t)(it & 1) * gridDim.x;
            for (unsigned bb = threadIdx.x; bb < gridDim.x; bb += blockDim.x) {
                const ulonglong2 p = __ldcg(pp + bb);
                sn |= (p.y & kNanBit) ? 1 : 0;
                S += ((u128)(p.y & ~kNanBit) << 64) | p.x;
            }
            unsigned long long slo = (unsigned long long)S, shi = (unsigned long long)(S >> 64);
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long olo = __shfl_xor_sync(0xffffffffu, slo, o);
                const unsigned long long ohi = __shfl_xor_sync(0xffffffffu, shi, o);
                const u128 t = (((u128)shi << 64) | slo) + (((u128)ohi << 64) | olo);
                slo = (unsigned long long)t, shi = (unsigned long long)(t >> 64);
                sn |= __shfl_xor_sync(0xffffffffu, sn, o);
            }
            __syncthreads();  // s_lo/s_hi/s_nan of the block reduction above are consumed
            if (lane == 0) s_lo[warp] = slo, s_hi[warp] = shi, s_nan[warp] = sn;
            __syncthreads();
            if (threadIdx.x == 0) {
                u128 tot = 0;
                int tn = 0;
                for (int w = 0; w < kOcThreads / 32; ++w) tot += ((u128)s_hi[w] << 64) | s_lo[w], tn |= s_nan[w];
                s_up = (!tn && tot > T) ? 1 : 0;  // numpy: a NaN sum never compares > 0
            }
        }
        __syncthreads();
        if (s_up) l1 = lmid;
        else l2 = lmid, all_up = 0;
        ++it;
        __syncthreads();  // s_up / s_lo reuse
    }
    for (int64_t i = gid; i < n; i += stride) xnew[i] = oc_value(__ldcg(x + i), __ldcg(dc + i), lmid, move);
    if (gid == 0) {
        *lmid_out = lmid;
        if (iters_out) {
            iters_out[0] = it;
            iters_out[1] = ((it > 0 && all_up) ? TF_OC_BRACKET_EXHAUSTED : 0) | (stalled ? TF_OC_NO_PROGRESS : 0);
        }
    }
}

}  // namespace

tf_status oc_update(const double *x, const double *dc, int64_t n, double volfrac, double move, double l1,
                    double l2, double tol, double *xnew, double *lmid_out, int *iters_out, cudaStream_t s) {
    DeviceInfo di;
    TF_TRY(device_info(&di));
    int occ = 0;
    TF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_oc, kOcThreads, 0));
    if (occ < 1) {
        set_error("tf_oc_update: kernel does not fit on an SM");
        return TF_ERR_CUDA;
    }
    const int64_t want = (n + kOcThreads - 1) / kOcThreads;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)di.sms * std::min(occ, 4)));
    // exact target volfrac*N (one fp64 rounding, as in the listing) in units of 2^-62
    const double target = volfrac * (double)n;
    if (!(target >= 0x1p-10) || !(target < 0x1p60)) {
        set_error("tf_oc_update: volfrac*n out of range");
        return TF_ERR_INVALID;
    }
    int e = 0;
    const double m = frexp(target, &e);                  // target = m * 2^e, m in [0.5, 1)
    const unsigned long long mi = (unsigned long long)ldexp(m, 53);  // exact 53-bit integer
    const int shift = e - 53 + 62;                       // target*2^62 = mi * 2^shift, shift >= 0
    const u128 T = (u128)mi << shift;
    DevBuf<ulonglong2> parts;
    TF_TRY(parts.alloc((size_t)2 * grid, s, "oc partials"));
    unsigned long long t_lo = (unsigned long long)T, t_hi = (unsigned long long)(T >> 64);
    void *args[] = {(void *)&x,    (void *)&dc,   (void *)&n,    (void *)&move,     (void *)&l1,
                    (void *)&l2,   (void *)&tol,  (void *)&t_lo, (void *)&t_hi,     (void *)&parts.p,
                    (void *)&xnew, (void *)&lmid_out, (void *)&iters_out};
    cudaError_t err = cudaLaunchCooperativeKernel((const void *)k_oc, dim3(grid), dim3(kOcThreads), args, 0, s);
    count_launch();
    if (err != cudaSuccess) {
        set_error("tf_oc_update: cooperative launch failed: %s", cudaGetErrorString(err));
        return TF_ERR_CUDA;
    }
    return TF_OK;
}

}  // namespace tf
