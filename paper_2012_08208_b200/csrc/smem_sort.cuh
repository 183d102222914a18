// smem_sort.cuh -- block-wide stable LSD radix sort of (key, val) pairs in shared memory, used
// by the per-bin fill (build.cu) and the group count kernel (cl_build.cu). Product code only.
#pragma once

#include "tf_internal.cuh"

namespace tf {
namespace {

// Block-wide stable LSD radix sort of C (key, val) pairs in shared memory, 8-bit digits.
// Warp w owns the contiguous strip [w*Q, (w+1)*Q): per-warp digit histograms, a block scan
// over (digit, warp) in digit-major order, then a stable scatter where the rank inside a
// 32-element round comes from __match_any_sync peer groups. Returns 0 if the result is in
// (ka, va), 1 if in (kb, vb).
template <int WARPS>
__device__ int block_radix_sort_smem(uint32_t *ka, uint32_t *va, uint32_t *kb, uint32_t *vb, int C, int bits,
                                     int32_t (*wc)[256], int32_t *wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int Q = (((C + WARPS - 1) / WARPS) + 31) & ~31;
    const int s0 = min(C, warp * Q), s1 = min(C, s0 + Q);
    int which = 0;
    for (int shift = 0; shift < bits; shift += 8) {
        uint32_t *ki = which ? kb : ka, *vi = which ? vb : va, *ko = which ? ka : kb, *vo = which ? va : vb;
        for (int i = lane; i < 256; i += 32) wc[warp][i] = 0;
        __syncwarp();
        // histogram: shared-memory atomics (no return value -> no dependency chain per round)
#pragma unroll 4
        for (int base = s0; base < s1; base += 32) {
            const int i = base + lane;
            if (i < s1) atomicAdd(&wc[warp][(ki[i] >> shift) & 255u], 1);
        }
        __syncthreads();
        // exclusive scan over (digit, warp), digit-major: each thread owns DPT consecutive digits
        constexpr int DPT = 256 / (32 * WARPS);
        int tot[DPT], run = 0;
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
            const int d = tid * DPT + k;
            int t = 0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) t += wc[w][d];
            tot[k] = t;
            run += t;
        }
        int inc = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        int ex = inc - run;
        for (int w = 0; w < warp; ++w) ex += wsum[w];
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
            const int d = tid * DPT + k;
            int off = ex;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) {
                const int c = wc[w][d];
                wc[w][d] = off;
                off += c;
            }
            ex += tot[k];
        }
        __syncthreads();
        for (int base = s0; base < s1; base += 32) {
            const int i = base + lane;
            const bool valid = i < s1;
            const uint32_t key = valid ? ki[i] : 0u, val = valid ? vi[i] : 0u;
            const int d = valid ? (int)((key >> shift) & 255u) : 256;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const int before = valid ? wc[warp][d] : 0;
            __syncwarp();
            if (valid && lane == __ffs(peers) - 1) wc[warp][d] = before + __popc(peers);
            __syncwarp();
            if (valid) {
                const int dst = before + __popc(peers & lt);
                TF_DCHECK(dst >= 0 && dst < C);
                ko[dst] = key;
                vo[dst] = val;
            }
        }
        __syncthreads();
        which ^= 1;
    }
    return which;
}


// The same sort restricted to key bits [shift0, bits): after it, keys are ordered by
// key >> shift0, equal ones in input order (stable). Returns the number of passes (the result is
// in (ka, va) when even, (kb, vb) when odd). Used with shift0 > 0 by the group count kernel, which
// then repairs the few out-of-order runs of equal high bits (block_fix_low_bits).
template <int WARPS>
__device__ int block_radix_sort_bits(uint32_t *ka, uint32_t *va, uint32_t *kb, uint32_t *vb, int C, int shift0,
                                     int bits, int32_t (*wc)[256], int32_t *wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const int Q = (((C + WARPS - 1) / WARPS) + 31) & ~31;
    const int s0 = min(C, warp * Q), s1 = min(C, s0 + Q);
    int passes = 0;
    for (int shift = shift0; shift < bits; shift += 8, ++passes) {
        const bool odd = passes & 1;
        uint32_t *ki = odd ? kb : ka, *vi = odd ? vb : va, *ko = odd ? ka : kb, *vo = odd ? va : vb;
        const uint32_t dmask = (bits - shift >= 8) ? 255u : ((1u << (bits - shift)) - 1u);
        for (int i = lane; i < 256; i += 32) wc[warp][i] = 0;
        __syncwarp();
#pragma unroll 4
        for (int base = s0; base < s1; base += 32) {
            const int i = base + lane;
            if (i < s1) atomicAdd(&wc[warp][(ki[i] >> shift) & dmask], 1);
        }
        __syncthreads();
        constexpr int DPT = 256 / (32 * WARPS);
        int tot[DPT], run = 0;
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
            const int d = tid * DPT + k;
            int t = 0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) t += wc[w][d];
            tot[k] = t;
            run += t;
        }
        int inc = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        int ex = inc - run;
        for (int w = 0; w < warp; ++w) ex += wsum[w];
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
            const int d = tid * DPT + k;
            int off = ex;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) {
                const int c = wc[w][d];
                wc[w][d] = off;
                off += c;
            }
            ex += tot[k];
        }
        __syncthreads();
        for (int base = s0; base < s1; base += 32) {
            const int i = base + lane;
            const bool valid = i < s1;
            const uint32_t key = valid ? ki[i] : 0u, val = valid ? vi[i] : 0u;
            const int d = valid ? (int)((key >> shift) & dmask) : 256;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const int before = valid ? wc[warp][d] : 0;
            __syncwarp();
            if (valid && lane == __ffs(peers) - 1) wc[warp][d] = before + __popc(peers);
            __syncwarp();
            if (valid) {
                const int dst = before + __popc(peers & lt);
                TF_DCHECK(dst >= 0 && dst < C);
                ko[dst] = key;
                vo[dst] = val;
            }
        }
        __syncthreads();
    }
    return passes;
}

// After block_radix_sort_bits(shift0 = s): keys with equal key >> s form runs of at most 2^s
// distinct keys, in input order. Each run that is not ascending is sorted by the thread that owns
// its first element (insertion sort; runs are short, and inputs whose bins list ids in x order
// -- lattice and FEM numberings -- have none). Ends with __syncthreads().
__device__ __forceinline__ void block_fix_low_bits(uint32_t *k, uint32_t *v, int C, int s) {
    for (int t = threadIdx.x; t < C; t += blockDim.x) {
        const uint32_t hi = k[t] >> s;
        if (t > 0 && (k[t - 1] >> s) == hi) continue;  // not a run start
        int e = t + 1;
        bool sorted = true;
        while (e < C && (k[e] >> s) == hi) {
            sorted &= k[e - 1] < k[e];
            ++e;
        }
        if (sorted) continue;
        for (int a = t + 1; a < e; ++a) {
            const uint32_t ka = k[a], va = v[a];
            int b = a - 1;
            while (b >= t && k[b] > ka) {
                k[b + 1] = k[b];
                v[b + 1] = v[b];
                --b;
            }
            k[b + 1] = ka;
            v[b + 1] = va;
        }
    }
    __syncthreads();
}

}  // namespace
}  // namespace tf
