// scan.cu -- device-wide exclusive prefix sum (a6 in SURVEY.md 8(a): counts -> row pointers;
// also the digit-offset table of the radix sort). Tile = 4096 elements:
//   n <= 2 tiles         one block walks the tiles with a running carry (one launch);
//   tiles <= 4096        tile sums -> per-tile scan, every block summing the tile sums before its own
//                        (two launches; the redundant reads are <= tiles^2/2 L2-resident values);
//   larger               tile sums -> single-block scan of the tile sums -> per-tile scan with carry-in.
// Deterministic (integer arithmetic). HBM-bound: reads the input twice, writes once.
#include "tf_internal.cuh"

namespace tf {
namespace {

constexpr int kThreads = 512;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Exclusive block scan of one value per thread; returns the block total in *total.
template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T *total) {
    __shared__ T warp_tot[kThreads / 32];
    __shared__ T block_tot;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = warp_incl_scan(v);
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = (lane < kThreads / 32) ? warp_tot[lane] : T(0);
        T wi = warp_incl_scan(w);
        if (lane < kThreads / 32) warp_tot[lane] = wi - w;  // exclusive warp offsets
        if (lane == kThreads / 32 - 1) block_tot = wi;
    }
    __syncthreads();
    T r = warp_tot[warp] + inc - v;
    *total = block_tot;
    __syncthreads();
    return r;
}

template <class Tin, class Tacc>
__global__ void __launch_bounds__(kThreads) k_tile_sums(const Tin *__restrict__ in, int64_t n,
                                                        Tacc *__restrict__ partials) {
    const int64_t base = (int64_t)blockIdx.x * kTile;
    Tacc s = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        int64_t k = base + i * kThreads + threadIdx.x;
        if (k < n) s += (Tacc)in[k];
    }
    // block reduce
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ Tacc ws[kThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        Tacc t = (threadIdx.x < kThreads / 32) ? ws[threadIdx.x] : Tacc(0);
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) partials[blockIdx.x] = t;
    }
}

// One block scans m partials in place (exclusive), looping over chunks with a carry.
template <class Tacc>
__global__ void __launch_bounds__(kThreads) k_scan_partials(Tacc *p, int64_t m) {
    __shared__ Tacc carry_s;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int64_t base = 0; base < m; base += kThreads) {
        int64_t k = base + threadIdx.x;
        Tacc v = (k < m) ? p[k] : Tacc(0);
        Tacc tot;
        Tacc ex = block_excl_scan<Tacc>(v, &tot);
        Tacc carry = carry_s;
        if (k < m) p[k] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry_s = carry + tot;
        __syncthreads();
    }
}

// REDUCE = false: partials[] holds exclusive tile offsets; REDUCE = true: partials[] holds the tile
// sums and the block adds up the ones before its tile itself.
template <class Tin, class Tacc, class Tout, bool REDUCE>
__global__ void __launch_bounds__(kThreads) k_tile_scan(const Tin *__restrict__ in,
                                                        Tout *__restrict__ out, int64_t n,
                                                        const Tacc *__restrict__ partials,
                                                        int write_total) {
    __shared__ Tacc tile[kTile];
    __shared__ Tacc carry_s;
    const int64_t base = (int64_t)blockIdx.x * kTile;
    if (REDUCE) {
        Tacc c = 0;
        for (int k = threadIdx.x; k < (int)blockIdx.x; k += kThreads) c += partials[k];
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        __shared__ Tacc ws[kThreads / 32];
        if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            Tacc t = 0;
            for (int w = 0; w < kThreads / 32; ++w) t += ws[w];
            carry_s = t;
        }
    }
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        int64_t k = base + i * kThreads + threadIdx.x;
        tile[i * kThreads + threadIdx.x] = (k < n) ? (Tacc)in[k] : Tacc(0);
    }
    __syncthreads();
    Tacc loc[kItems];
    Tacc run = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        loc[i] = run;
        run += tile[threadIdx.x * kItems + i];
    }
    Tacc tot;
    Tacc ex = block_excl_scan<Tacc>(run, &tot);
    const Tacc carry = REDUCE ? carry_s : partials[blockIdx.x];  // (carry_s: ordered by block_excl_scan's barriers)
#pragma unroll
    for (int i = 0; i < kItems; ++i) tile[threadIdx.x * kItems + i] = carry + ex + loc[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        int64_t k = base + i * kThreads + threadIdx.x;
        if (k < n) out[k] = (Tout)tile[i * kThreads + threadIdx.x];
    }
    if (write_total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = (Tout)(carry + tot);
}

// One block scans the whole input, tile after tile, with a running carry (small inputs: one launch).
template <class Tin, class Tacc, class Tout>
__global__ void __launch_bounds__(kThreads) k_scan_small(const Tin *__restrict__ in, Tout *__restrict__ out,
                                                         int64_t n) {
    __shared__ Tacc tile[kTile];
    Tacc carry = 0;
    for (int64_t base = 0; base < n; base += kTile) {
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const int64_t k = base + i * kThreads + threadIdx.x;
            tile[i * kThreads + threadIdx.x] = (k < n) ? (Tacc)in[k] : Tacc(0);
        }
        __syncthreads();
        Tacc loc[kItems];
        Tacc run = 0;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            loc[i] = run;
            run += tile[threadIdx.x * kItems + i];
        }
        Tacc tot;
        const Tacc ex = block_excl_scan<Tacc>(run, &tot);
#pragma unroll
        for (int i = 0; i < kItems; ++i) tile[threadIdx.x * kItems + i] = carry + ex + loc[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const int64_t k = base + i * kThreads + threadIdx.x;
            if (k < n) out[k] = (Tout)tile[i * kThreads + threadIdx.x];
        }
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[n] = (Tout)carry;
}

template <class Tin, class Tacc, class Tout>
tf_status scan_impl(const Tin *in, Tout *out, int64_t n, cudaStream_t s) {
    if (n <= 0) {
        TF_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(Tout), s));
        return TF_OK;
    }
    const int64_t tiles = (n + kTile - 1) / kTile;
    if (tiles <= 2) {
        k_scan_small<Tin, Tacc, Tout><<<1, kThreads, 0, s>>>(in, out, n);
        TF_LAUNCH_CHECK();
        return TF_OK;
    }
    DevBuf<Tacc> part;
    TF_TRY(part.alloc(tiles, s, "scan partials"));
    k_tile_sums<Tin, Tacc><<<(unsigned)tiles, kThreads, 0, s>>>(in, n, part.p);
    TF_LAUNCH_CHECK();
    if (tiles <= 4096) {
        k_tile_scan<Tin, Tacc, Tout, true><<<(unsigned)tiles, kThreads, 0, s>>>(in, out, n, part.p, 1);
        TF_LAUNCH_CHECK();
        return TF_OK;
    }
    k_scan_partials<Tacc><<<1, kThreads, 0, s>>>(part.p, tiles);
    TF_LAUNCH_CHECK();
    k_tile_scan<Tin, Tacc, Tout, false><<<(unsigned)tiles, kThreads, 0, s>>>(in, out, n, part.p, 1);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

}  // namespace

// out[0..n]: out[k] = sum_{i<k} in[i]; out[n] = total.
tf_status exclusive_scan_i32_i64(const int32_t *in, int64_t *out, int64_t n, cudaStream_t s) {
    return scan_impl<int32_t, int64_t, int64_t>(in, out, n, s);
}
tf_status exclusive_scan_i32_i32(const int32_t *in, int32_t *out, int64_t n, cudaStream_t s) {
    return scan_impl<int32_t, int64_t, int32_t>(in, out, n, s);
}

}  // namespace tf
