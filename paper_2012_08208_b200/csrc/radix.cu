// radix.cu -- hand-written stable LSD radix sort of (bin key, point id) pairs (a4 in SURVEY.md
// 8(a); BASELINE.json north_star "a hand-written radix sort of the cell keys").
//
// Per 8-bit digit pass (tile = 4096 pairs per block, 8 warps x 16 rounds x 32 lanes):
//   1. k_radix_hist    per-tile digit histogram -> hist[digit * tiles + tile]
//   2. exclusive scan of hist (digit-major) -> global base offset of (digit, tile)
//   3. k_radix_scatter stable scatter: the rank inside a tile comes from __match_any_sync
//      peer groups per 32-pair round plus per-warp digit counters, prefix-summed over
//      warps in tile order. Stability: input order inside a digit is preserved, so the
//      point ids (initially 0..n-1) ascend inside every bin after the last pass.
// HBM-bound: each pass reads 8 B/pair twice and writes 8 B/pair.
#include "tf_internal.cuh"

namespace tf {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRounds = 16;
constexpr int kTile = kThreads * kRounds;  // 4096
constexpr int kRadix = 256;

__global__ void __launch_bounds__(kThreads) k_radix_hist(const uint32_t *__restrict__ keys, int64_t n,
                                                         int shift, int32_t *__restrict__ hist,
                                                         int64_t tiles) {
    __shared__ int32_t cnt[kWarps][kRadix];
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll 4
    for (int i = 0; i < kRounds; ++i) {
        int64_t k = base + (int64_t)i * kThreads + threadIdx.x;
        if (k < n) atomicAdd(&cnt[warp][(keys[k] >> shift) & (kRadix - 1)], 1);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kThreads) {
        int32_t s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += cnt[w][d];
        hist[(int64_t)d * tiles + blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(kThreads) k_radix_scatter(
    const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint32_t *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, int shift, const int32_t *__restrict__ offs, int64_t tiles) {
    __shared__ int32_t wcnt[kWarps][kRadix];
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const int64_t strip = (int64_t)blockIdx.x * kTile + (int64_t)warp * (kRounds * 32);

    uint32_t key[kRounds], val[kRounds];
    int32_t rank[kRounds];
    int32_t dig[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        const int64_t k = strip + r * 32 + lane;
        const bool valid = k < n;
        key[r] = valid ? kin[k] : 0u;
        val[r] = valid ? vin[k] : 0u;
        const int d = valid ? (int)((key[r] >> shift) & (kRadix - 1)) : kRadix;  // sentinel
        dig[r] = d;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        const int before = (d < kRadix) ? wcnt[warp][d] : 0;
        rank[r] = before + __popc(peers & lt_mask);
        __syncwarp();
        if (lane == leader && d < kRadix) wcnt[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kThreads) {
        int32_t run = offs[(int64_t)d * tiles + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            int32_t t = wcnt[w][d];
            wcnt[w][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
        if (dig[r] < kRadix) {
            const int32_t dest = wcnt[warp][dig[r]] + rank[r];
            kout[dest] = key[r];
            vout[dest] = val[r];
        }
    }
}

}  // namespace

tf_status radix_sort_pairs(uint32_t *keys, uint32_t *vals, uint32_t *keys_alt, uint32_t *vals_alt,
                           int64_t n, int bits, cudaStream_t s, uint32_t **keys_out,
                           uint32_t **vals_out, int *passes_out) {
    const int passes = (bits + 7) / 8;
    *passes_out = passes;
    *keys_out = keys;
    *vals_out = vals;
    if (passes == 0 || n <= 1) return TF_OK;
    const int64_t tiles = (n + kTile - 1) / kTile;
    DevBuf<int32_t> hist, offs;
    TF_TRY(hist.alloc((size_t)kRadix * tiles, s, "radix histogram"));
    TF_TRY(offs.alloc((size_t)kRadix * tiles + 1, s, "radix offsets"));
    uint32_t *ki = keys, *vi = vals, *ko = keys_alt, *vo = vals_alt;
    for (int p = 0; p < passes; ++p) {
        const int shift = 8 * p;
        k_radix_hist<<<(unsigned)tiles, kThreads, 0, s>>>(ki, n, shift, hist.p, tiles);
        TF_LAUNCH_CHECK();
        TF_TRY(exclusive_scan_i32_i32(hist.p, offs.p, (int64_t)kRadix * tiles, s));
        k_radix_scatter<<<(unsigned)tiles, kThreads, 0, s>>>(ki, vi, ko, vo, n, shift, offs.p, tiles);
        TF_LAUNCH_CHECK();
        uint32_t *t;
        t = ki; ki = ko; ko = t;
        t = vi; vi = vo; vo = t;
    }
    *keys_out = ki;
    *vals_out = vi;
    return TF_OK;
}

}  // namespace tf
