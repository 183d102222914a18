// apply.cu -- the per-iteration filter applies.
//
//   sensitivity  out_i = (sum_k vals[k] * (x[cols[k]] * dc[cols[k]])) / (Hs_i * max(1e-3, x_i))
//                (Eq. filter, Eq. filter_mat, listing
//                the paper's dense GEMV becomes a CSR SpMV, with the
//                Hadamard product, the max floor and the division fused in)
//   density      out_i = (sum_k vals[k] * x[cols[k]]) / Hs_i   (BASELINE.json north_star)
//
// Work split: the nnz stream is cut into windows of W entries (W = stage capacity minus the
// longest row, so every window stages; kWindow for short rows); window w owns the rows
// whose first entry falls in it (row-block table rb[] and 16-byte aligned staging ranges wlo[],
// built once per filter by make_apply_plan). k_spmv is persistent and warp-specialised:
//   * a producer warp streams the block's windows (w = blockIdx.x + k*gridDim.x) into a
//     kStages-deep shared-memory ring with TMA bulk copies (cp.async.bulk, mbarrier
//     completion, L2 evict_first) of cols/vals/rowptr -- the CSR stream never touches the
//     LSU/L1 data pipe, which is left to the gathers;
//   * kCW consumer warps take groups of 32/G rows, dealt round-robin per window (rotating),
//     G lanes per row read cols/vals from shared memory, issue U gathers before accumulating,
//     reduce with a G-lane xor-shuffle tree (deterministic) and write the fused epilogue;
//   * sensitivity: a cooperative launch first forms t = x o dc (one gather per entry instead of
//     two) and grid-syncs; the producer's first kStages copies overlap that pass;
//   * MODE 2 (tf_filter_both): (t, x) pairs, one 16-byte gather per entry, two accumulators;
//   * [wbeg, wend) window ranges serve the host pipeline's row-range chunks.
// Windows whose staging range exceeds the ring capacity (long rows) are reduced one row per
// warp straight from global memory.
//
// Roofline: HBM. Algorithmic bytes per apply = 12*nnz + 8(N+1) + 32N (sensitivity) or
// + 24N (density); gathers of x/dc hit L2/L1 (neighbour columns are index-local).
#include <cooperative_groups.h>

#include <stdlib.h>

#include <algorithm>

#include <atomic>

#include "tf_internal.cuh"

#ifndef TF_APPLY_PREFETCH
#define TF_APPLY_PREFETCH 0  // L2 prefetch distance in rounds (0: off)
#endif

namespace tf {
namespace {

constexpr int kMaxDevices = 64;

#ifndef TF_APPLY_CW
#define TF_APPLY_CW 10
#endif
#ifndef TF_APPLY_BPS
#define TF_APPLY_BPS 3
#endif
#ifndef TF_APPLY_STAGES
#define TF_APPLY_STAGES 2
#endif
constexpr int kCW = TF_APPLY_CW;          // consumer warps per block (+1 producer warp)
constexpr int kThreads = kCW * 32;        // consumer threads
#ifndef TF_APPLY_WINDOW
#define TF_APPLY_WINDOW 2048
#endif
#ifndef TF_APPLY_STAGE
#define TF_APPLY_STAGE 2976
#endif
#ifndef TF_APPLY_DYNWIN
#define TF_APPLY_DYNWIN 1  // 1: window = stage capacity minus the longest row (all windows staged)
#endif
#ifndef TF_APPLY_STATIC
#define TF_APPLY_STATIC 1  // 1: row groups of a window dealt to the warps round-robin (no atomics)
#endif
#ifndef TF_APPLY_ROWCAP
#define TF_APPLY_ROWCAP 256
#endif
constexpr int kWindow = TF_APPLY_WINDOW;  // target nnz per window (row block)
constexpr int kStage = TF_APPLY_STAGE;    // staged nnz capacity per stage (multiple of 4): 35 KB
constexpr int kRowCap = TF_APPLY_ROWCAP;  // staged rowptr capacity per stage (int64, multiple of 2): 2 KB
constexpr int kStages = TF_APPLY_STAGES;  // TMA ring depth per block
constexpr int kBlocksPerSM = TF_APPLY_BPS;  // persistent grid = kBlocksPerSM x SMs (tuned on c5: 10 x 3 x 2 x stage 2976)

__global__ void k_plan(const int64_t *__restrict__ rowptr, int64_t n, int64_t nblocks, int64_t window,
                       int32_t *__restrict__ rb) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nblocks;
         b += (int64_t)gridDim.x * blockDim.x) {
        if (b == nblocks) {
            rb[b] = (int32_t)n;
            continue;
        }
        const int64_t target = b * window;
        int64_t lo = 0, hi = n;  // first r in [0, n] with rowptr[r] >= target
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (rowptr[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        rb[b] = (int32_t)lo;
    }
}

#ifndef TF_APPLY_FASTDIV
#define TF_APPLY_FASTDIV 0  // 1: reciprocal + Newton quotient (<= ~1 ulp) instead of the IEEE division
#endif
#if TF_APPLY_FASTDIV
__device__ __forceinline__ double quot(double a, double b) {
    // b > 0 and normal here (b >= Hs_i * 1e-3 >= rmin * 1e-3)
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
    double e = fma(-b, r, 1.0);
    r = fma(r, e, r);
    e = fma(-b, r, 1.0);
    r = fma(r, e, r);
    const double q = a * r;
    return fma(r, fma(-b, q, a), q);
}
#else
__device__ __forceinline__ double quot(double a, double b) { return a / b; }
#endif

template <bool SENS>
__device__ __forceinline__ double finish(double acc, double hs_i, double x_i) {
    if (SENS) return quot(acc, hs_i * fmax(1e-3, x_i));
    return quot(acc, hs_i);
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---- TMA bulk copy (global -> shared) with mbarrier completion, evict-first in L2
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
#if TF_APPLY_PREFETCH > 0
// L2 prefetch of a global range (no shared memory, no completion): raises the bytes in flight
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(phase)
            : "memory");
    }
}

// try_wait with a suspend-time hint: the producer sleeps instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(phase), "r"(20000u)
            : "memory");
    }
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Persistent, warp-specialised SpMV. Warp kCW (the producer) streams the windows of this
// block (w = blockIdx.x, + gridDim.x, ...) into a kStages-deep shared-memory ring with TMA
// bulk copies; full[s] completes when a window's bytes have landed, empty[s] when all kCW
// consumer warps have left it. Consumer warps take groups of 32/G rows of the window dealt
// round-robin, rotating by one warp per window (no atomics, no block-wide barriers; a shared
// counter with TF_APPLY_STATIC=0 measured 3% slower); each row is reduced by G lanes
// that issue U predicated (col, val) shared loads and U x/dc gathers before accumulating,
// and the group leader writes out[r] directly.
// MODE 0: density; 1: sensitivity; 2: both filters in one pass over H (sensitivity -> out,
// density -> out2): the CSR streams once, each entry gathers t_j and x_j.
template <int MODE, int G, int U>
__global__ void __launch_bounds__(kThreads + 32, kBlocksPerSM) k_spmv(const int64_t *__restrict__ rowptr,
                                                                      const int32_t *__restrict__ cols,
                                                                      const double *__restrict__ vals,
                                                                      const double *__restrict__ hs,
                                                                      const double *__restrict__ x,
                                                                      const double *__restrict__ dc,
                                                                      double *__restrict__ out,
                                                                      double *__restrict__ out2,
                                                                      const int32_t *__restrict__ rb,
                                                                      const int64_t *__restrict__ wlo,
                                                                      int64_t nwin, double *tbuf, int64_t n,
                                                                      double penal, int energy, int64_t wbeg,
                                                                      int64_t wend, int tpass, int64_t row_limit,
                                                                      int64_t row_begin) {
    // MODE 3: sensitivity without the t pass (ordinary launch): each entry gathers x_j and dc_j and
    // forms t_j = x_j * dc_j itself (the same product, so the same sums bit for bit)
    constexpr bool SENS = MODE != 0, BOTH = MODE == 2, DIRECT = MODE == 3;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *svals = reinterpret_cast<double *>(smem_raw);                           // [kStages][kStage]
    int64_t *srow = reinterpret_cast<int64_t *>(svals + kStages * kStage);          // [kStages][kRowCap]
    int32_t *scols = reinterpret_cast<int32_t *>(srow + kStages * kRowCap);         // [kStages][kStage]
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    __shared__ int next_row[kStages];
    __shared__ int64_t s_wbeg;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (row_begin > 0) {
        // rows [row_begin, row_limit): start at the window holding row_begin (binary search of
        // the row-block table; its rows before row_begin are recomputed with the same values)
        if (tid == 0) {
            int64_t lo = wbeg, hi = wend;  // first w in [wbeg, wend) with rb[w + 1] > row_begin
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (rb[mid + 1] <= row_begin) lo = mid + 1;
                else hi = mid;
            }
            s_wbeg = lo;
        }
        __syncthreads();
        wbeg = s_wbeg;
    }
    if (tid == 0) {
        for (int st = 0; st < kStages; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], kCW);
            next_row[st] = 0;
        }
    }
    __syncthreads();

    if (warp == kCW) {
        // ---------------- producer
        uint64_t pol = 0;
        if (lane == 0) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        int it = 0;
        int64_t w = wbeg + blockIdx.x;
        auto issue = [&](int st) {
            const int64_t a = wlo[w], n4 = wlo[w + 1 + nwin] - a;  // wlo[nwin+1+w] = aligned end
            next_row[st] = 0;  // published to the consumers by the full-barrier completion
            const int r0 = rb[w], r1 = rb[w + 1];
            const int r0a = r0 & ~1, nrow = ((r1 + 2) & ~1) - r0a;  // rowptr[r0a .. ), 16-byte aligned
            if (n4 > 0 && n4 <= kStage && nrow <= kRowCap) {
                mbar_expect_tx(&full[st], (uint32_t)n4 * 12u + (uint32_t)nrow * 8u);
                bulk_g2s(svals + st * kStage, vals + a, (uint32_t)n4 * 8u, &full[st], pol);
                bulk_g2s(scols + st * kStage, cols + a, (uint32_t)n4 * 4u, &full[st], pol);
                bulk_g2s(srow + st * kRowCap, rowptr + r0a, (uint32_t)nrow * 8u, &full[st], pol);
            } else {
                mbar_arrive(&full[st]);  // nothing staged: consumers read global memory
            }
#if TF_APPLY_PREFETCH > 0
            {  // L2 prefetch of this block's window TF_APPLY_PREFETCH rounds ahead
                const int64_t wp = w + (int64_t)TF_APPLY_PREFETCH * gridDim.x;
                if (wp < wend) {
                    const int64_t pa = wlo[wp], pn = wlo[wp + 1 + nwin] - pa;
                    if (pn > 0 && pn <= kStage) {
                        bulk_prefetch_l2(vals + pa, (uint32_t)pn * 8u);
                        bulk_prefetch_l2(cols + pa, (uint32_t)pn * 4u);
                    }
                }
            }
#endif
        };
        // prologue: the first kStages windows need no empty-wait (overlaps the t pass)
        if (lane == 0)
            for (; w < wend && rb[w] < row_limit && it < kStages; w += gridDim.x, ++it) issue(it);
        if (SENS && !DIRECT && tpass == 1) {
            __syncwarp();
            cooperative_groups::this_grid().sync();
        }
        if (lane == 0)
            for (; w < wend && rb[w] < row_limit; w += gridDim.x, ++it) {
                const int st = it % kStages;
                mbar_wait_sleep(&empty[st], ((it / kStages) - 1) & 1);
                issue(st);
            }
        return;
    }

    // ---------------- consumers
    if (SENS && !DIRECT && tpass == 2) {
        // t comes from the preceding k_tpass launch (programmatic dependent launch): the producer
        // has been staging CSR windows already; the gathers wait for that grid's results
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (SENS && !DIRECT && tpass == 1) {
        // fused Hadamard pass t = x o dc (PAPER.md:447 np.multiply(density, sensitivity)),
        // then a grid-wide barrier: the SpMV gathers one array instead of two
        // NEXT-2 (energy != 0): dc is evaluated here from the element energies U passed in `dc`,
        // dc = -p x^(p-1) U (listing PAPER.md:376), never stored
        if (energy) {
            for (int64_t i = (int64_t)blockIdx.x * kThreads + tid; i < n; i += (int64_t)gridDim.x * kThreads) {
                const double xi = __ldg(x + i);
                tbuf[i] = xi * ((-penal * pow(xi, penal - 1.0)) * __ldg(dc + i));
            }
        } else if (BOTH) {
            // (t, x) interleaved: one 16-byte gather per entry serves both filters
            double2 *tx = reinterpret_cast<double2 *>(tbuf);
            for (int64_t i = (int64_t)blockIdx.x * kThreads + tid; i < n; i += (int64_t)gridDim.x * kThreads) {
                const double xi = __ldg(x + i);
                tx[i] = make_double2(xi * __ldg(dc + i), xi);
            }
        } else {
            for (int64_t i = (int64_t)blockIdx.x * kThreads + tid; i < n; i += (int64_t)gridDim.x * kThreads)
                tbuf[i] = __ldg(x + i) * __ldg(dc + i);
        }
        cooperative_groups::this_grid().sync();
    }
    // t was written in this launch: read it with plain cached loads, never the read-only path
    const double *gsrc = (SENS && !DIRECT) ? tbuf : x;
    const double2 *gtx = reinterpret_cast<const double2 *>(tbuf);  // BOTH: (t, x) pairs
    constexpr int RPW = 32 / G;  // rows per warp claim
    const int sub = lane & (G - 1);
    int it = 0;
    for (int64_t w = wbeg + blockIdx.x; w < wend && rb[w] < row_limit; w += gridDim.x, ++it) {
        const int st = it % kStages;
        const int r0 = rb[w], R = rb[w + 1] - r0;
        const int64_t a = wlo[w], n4 = wlo[w + 1 + nwin] - a;
        const int r0a = r0 & ~1, nrow = ((rb[w + 1] + 2) & ~1) - r0a;
        const bool staged = n4 > 0 && n4 <= kStage && nrow <= kRowCap;
        const double *sv = svals + st * kStage;
        const int32_t *sc = scols + st * kStage;
        const int64_t *sr = srow + st * kRowCap + (r0 - r0a);  // sr[rr] = rowptr[r0 + rr]
        mbar_wait(&full[st], (it / kStages) & 1);
        if (staged) {
#if TF_APPLY_STATIC
            // static claims: row group g of this window goes to warp (g + it) mod kCW (the
            // rotation spreads the short last round over the warps); no shared atomics
            const int g0 = (warp + kCW - (it % kCW)) % kCW;
            for (int rbase = g0 * RPW; rbase < R; rbase += kCW * RPW) {
#else
            for (;;) {
                int rbase = 0;
                if (lane == 0) rbase = atomicAdd(&next_row[st], RPW);
                rbase = __shfl_sync(0xffffffffu, rbase, 0);
                if (rbase >= R) break;
#endif
                const int rr = rbase + lane / G;
                double acc = 0.0, acc2 = 0.0, hs_r = 1.0, x_r = 1.0;
                if (rr < R) {
                    const int r = r0 + rr;
                    if (sub == 0) hs_r = hs[r], x_r = x[r];  // epilogue operands, issued early
                    const int s = (int)(sr[rr] - a), e = (int)(sr[rr + 1] - a);
                    TF_DCHECK(s >= 0 && s <= e && e <= (int)n4);
                    int32_t j[U];
                    double v[U], t[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int i = s + sub + u * G;
                        j[u] = (i < e) ? sc[i] : -1;
                        v[u] = (i < e) ? sv[i] : 0.0;
                    }
                    if (BOTH) {
                        double xg[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const double2 p = (j[u] >= 0) ? __ldca(gtx + j[u]) : make_double2(0.0, 0.0);
                            t[u] = p.x;
                            xg[u] = p.y;
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) acc2 = fma(v[u], xg[u], acc2);
                    } else if (DIRECT) {
                        double dg[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            t[u] = (j[u] >= 0) ? __ldg(x + j[u]) : 0.0;
                            dg[u] = (j[u] >= 0) ? __ldg(dc + j[u]) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) t[u] *= dg[u];
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u) t[u] = (j[u] >= 0) ? __ldca(gsrc + j[u]) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) acc = fma(v[u], t[u], acc);
                    for (int i = s + sub + U * G; i < e; i += G) {  // rows longer than U*G
                        const int32_t jj = sc[i];
                        if (BOTH) {
                            const double2 p = __ldca(gtx + jj);
                            acc = fma(sv[i], p.x, acc);
                            acc2 = fma(sv[i], p.y, acc2);
                        } else if (DIRECT) {
                            acc = fma(sv[i], __ldg(x + jj) * __ldg(dc + jj), acc);
                        } else {
                            acc = fma(sv[i], __ldca(gsrc + jj), acc);
                        }
                    }
                }
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) {
                    acc += __shfl_xor_sync(0xffffffffu, acc, o);
                    if (BOTH) acc2 += __shfl_xor_sync(0xffffffffu, acc2, o);
                }
                if (sub == 0 && rr < R) {
                    out[r0 + rr] = finish<SENS>(acc, hs_r, x_r);
                    if (BOTH) out2[r0 + rr] = finish<false>(acc2, hs_r, x_r);
                }
            }
        } else {
            // window too large to stage (long rows): a whole warp per row, from global memory
            for (;;) {
                int rr = 0;
                if (lane == 0) rr = atomicAdd(&next_row[st], 1);
                rr = __shfl_sync(0xffffffffu, rr, 0);
                if (rr >= R) break;
                const int r = r0 + rr;
                const int64_t s = rowptr[r], e = rowptr[r + 1];
                double acc = 0.0, acc2 = 0.0;
                for (int64_t k = s + lane; k < e; k += 32) {
                    const int32_t jj = cols[k];
                    if (BOTH) {
                        const double2 p = __ldca(gtx + jj);
                        acc = fma(vals[k], p.x, acc);
                        acc2 = fma(vals[k], p.y, acc2);
                    } else if (DIRECT) {
                        acc = fma(vals[k], __ldg(x + jj) * __ldg(dc + jj), acc);
                    } else {
                        acc = fma(vals[k], __ldca(gsrc + jj), acc);
                    }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    acc += __shfl_xor_sync(0xffffffffu, acc, o);
                    if (BOTH) acc2 += __shfl_xor_sync(0xffffffffu, acc2, o);
                }
                if (lane == 0) {
                    out[r] = finish<SENS>(acc, hs[r], x[r]);
                    if (BOTH) out2[r] = finish<false>(acc2, hs[r], x[r]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
}

// t = x o dc as its own launch, for the programmatic-dependent sensitivity apply: it lets the
// dependent SpMV grid launch at once (griddepcontrol.launch_dependents), so the SpMV's producers
// stage the first CSR windows while this pass runs.
__global__ void __launch_bounds__(256) k_tpass(const double *__restrict__ x, const double *__restrict__ dc,
                                               double *__restrict__ t, int64_t n) {
    asm volatile("griddepcontrol.launch_dependents;");
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t[i] = x[i] * dc[i];
}

// Windows [wbeg, wend) of the plan. SENS: tbuf == nullptr -> per-call scratch, t pass and a
// cooperative launch (the normal API); tbuf given -> tpass selects whether this launch computes
// t (cooperative) or reuses it (ordinary launch; the row-range chunks of the host pipeline).
template <int MODE, int G, int U>
tf_status launch_spmv_gu(const tf_filter_s *h, const double *x, const double *dc, double *out, double *out2,
                         cudaStream_t s, double penal, int energy, int64_t wbeg, int64_t wend, double *tbuf_ext,
                         int tpass, int64_t row_limit, int64_t row_begin) {
    constexpr bool SENS = MODE == 1 || MODE == 2;  // modes with the cooperative t pass
    const size_t smem = (size_t)kStages * (kStage * (sizeof(double) + sizeof(int32_t)) + kRowCap * sizeof(int64_t));
    auto kern = k_spmv<MODE, G, U>;
    // per-instantiation, per-device attribute (dynamic shared memory above 48 KB needs the
    // opt-in on every device the process launches on) and co-resident blocks per SM (a
    // cooperative grid must not exceed it); cached after the first launch on each device
    static std::atomic<int> occ_of[kMaxDevices];
    int dev = 0;
    TF_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDevices) {
        set_error("device ordinal %d out of range", dev);
        return TF_ERR_CUDA;
    }
    int occ = occ_of[dev].load(std::memory_order_acquire);
    if (!occ) {
        TF_TRY(allow_dynamic_smem(kern, smem));
        TF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads + 32, smem));
        if (occ < 1) {
            set_error("apply kernel does not fit on an SM");
            return TF_ERR_CUDA;
        }
        occ_of[dev].store(occ, std::memory_order_release);
    }
    if (wend <= wbeg) return TF_OK;
    const unsigned grid = (unsigned)std::min<int64_t>(
        std::min<int64_t>(wend - wbeg, (int64_t)h->plan.grid), (int64_t)occ * (h->plan.grid / kBlocksPerSM));
    const int64_t *rowptr = h->rowptr;
    const int32_t *cols = h->cols;
    const double *vals = h->vals, *hs = h->hs;
    const int32_t *rb = h->plan.rb;
    const int64_t *wlo = h->plan.wlo;
    int64_t nwin = h->plan.nblocks, n = h->n;
    double *tbuf = tbuf_ext;
    if (MODE == 1 && !energy && tbuf_ext == nullptr && h->plan.pdl) {
        // t pass as its own launch + the SpMV as a programmatic dependent launch (no cooperative
        // launch, no grid-wide barrier; CSR staging overlaps the t pass)
        TF_TRY(dalloc(&tbuf, (size_t)n, s, "sensitivity scratch t = x*dc"));
        const unsigned tg = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)h->plan.grid * 2);
        k_tpass<<<tg, 256, 0, s>>>(x, dc, tbuf, n);
        TF_LAUNCH_CHECK();
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kThreads + 32);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const int tp = 2;
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, rowptr, cols, vals, hs, x, dc, out, out2, rb, wlo, nwin,
                                           tbuf, n, penal, energy, wbeg, wend, tp, row_limit, row_begin);
        count_launch();
        dev_free(tbuf, s);
        if (e != cudaSuccess) {
            set_error("programmatic dependent launch failed: %s", cudaGetErrorString(e));
            return TF_ERR_CUDA;
        }
        return TF_OK;
    }
    if (SENS && (tbuf_ext == nullptr || tpass)) {
        // per-call scratch (stream-ordered) unless the caller owns it: concurrent applies on
        // different streams stay safe
        if (!tbuf_ext) TF_TRY(dalloc(&tbuf, (size_t)n * (MODE == 2 ? 2 : 1), s, "sensitivity scratch t = x*dc"));
        tpass = 1;
        void *args[] = {(void *)&rowptr, (void *)&cols, (void *)&vals,  (void *)&hs,     (void *)&x,
                        (void *)&dc,     (void *)&out,  (void *)&out2,  (void *)&rb,     (void *)&wlo,
                        (void *)&nwin,
                        (void *)&tbuf,   (void *)&n,    (void *)&penal, (void *)&energy, (void *)&wbeg,
                        (void *)&wend,   (void *)&tpass, (void *)&row_limit, (void *)&row_begin};
        cudaError_t e = cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(kThreads + 32), args, smem, s);
        count_launch();
        if (!tbuf_ext) dev_free(tbuf, s);
        if (e != cudaSuccess) {
            set_error("cooperative launch failed: %s", cudaGetErrorString(e));
            return TF_ERR_CUDA;
        }
        return TF_OK;
    }
    kern<<<grid, kThreads + 32, smem, s>>>(rowptr, cols, vals, hs, x, dc, out, out2, rb, wlo, nwin, tbuf, n, penal,
                                           energy, wbeg, wend, 0, row_limit, row_begin);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

template <int MODE, int G>
tf_status launch_spmv_g(const tf_filter_s *h, const double *x, const double *dc, double *out, double *out2,
                        cudaStream_t s, double penal, int energy, int64_t wbeg, int64_t wend, double *tbuf,
                        int tpass, int64_t row_limit, int64_t row_begin) {
    if ((MODE == 0 ? h->plan.unroll : (MODE == 1 || MODE == 3) ? h->plan.unroll_sens : h->plan.unroll_both) >= 8)
        return launch_spmv_gu<MODE, G, 8>(h, x, dc, out, out2, s, penal, energy, wbeg, wend, tbuf, tpass, row_limit, row_begin);
    return launch_spmv_gu<MODE, G, 4>(h, x, dc, out, out2, s, penal, energy, wbeg, wend, tbuf, tpass, row_limit, row_begin);
}

template <int MODE>
tf_status launch_spmv(const tf_filter_s *h, const double *x, const double *dc, double *out, cudaStream_t s,
                      double penal = 0.0, int energy = 0, int64_t wbeg = 0, int64_t wend = -1,
                      double *tbuf = nullptr, int tpass = 1, double *out2 = nullptr,
                      int64_t row_limit = INT64_MAX, int64_t row_begin = 0) {
    if (wend < 0) wend = h->plan.nblocks;
    switch (h->plan.group) {
        case 1: return launch_spmv_g<MODE, 1>(h, x, dc, out, out2, s, penal, energy, wbeg, wend, tbuf, tpass, row_limit, row_begin);
        case 2: return launch_spmv_g<MODE, 2>(h, x, dc, out, out2, s, penal, energy, wbeg, wend, tbuf, tpass, row_limit, row_begin);
        case 4: return launch_spmv_g<MODE, 4>(h, x, dc, out, out2, s, penal, energy, wbeg, wend, tbuf, tpass, row_limit, row_begin);
        case 8: return launch_spmv_g<MODE, 8>(h, x, dc, out, out2, s, penal, energy, wbeg, wend, tbuf, tpass, row_limit, row_begin);
        case 16: return launch_spmv_g<MODE, 16>(h, x, dc, out, out2, s, penal, energy, wbeg, wend, tbuf, tpass, row_limit, row_begin);
        default: return launch_spmv_g<MODE, 32>(h, x, dc, out, out2, s, penal, energy, wbeg, wend, tbuf, tpass, row_limit, row_begin);
    }
}

// max over rows r in [r0, r1) of the row's largest column (rows are ascending: the last entry;
// an empty row contributes nothing)
__global__ void k_chunk_maxcol(const int64_t *__restrict__ rowptr, const int32_t *__restrict__ cols, int64_t r0,
                               int64_t r1, int ascending, int32_t *__restrict__ out) {
    int m = -1;
    for (int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = rowptr[r], e = rowptr[r + 1];
        if (ascending) {
            if (e > s) m = max(m, cols[e - 1]);
        } else {
            for (int64_t k = s; k < e; ++k) m = max(m, cols[k]);
        }
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m >= 0) atomicMax(out, m);
}

// Aligned staging window of each row block: wlo[w] = rowptr[rb[w]] & ~3 and
// wlo[nwin + 1 + w] = (rowptr[rb[w+1]] + 3) & ~3 (16-byte aligned bulk copies).
__global__ void k_plan_windows(const int64_t *__restrict__ rowptr, const int32_t *__restrict__ rb, int64_t nwin,
                               int64_t *__restrict__ wlo) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += (int64_t)gridDim.x * blockDim.x) {
        wlo[w] = rowptr[rb[w]] & ~(int64_t)3;
        wlo[nwin + 1 + w] = (rowptr[rb[w + 1]] + 3) & ~(int64_t)3;
    }
}

__global__ void k_max_row(const int64_t *__restrict__ rowptr, int64_t n, unsigned long long *__restrict__ out) {
    unsigned long long m = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        m = max(m, (unsigned long long)(rowptr[r + 1] - rowptr[r]));
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace

tf_status make_apply_plan(tf_filter_s *h, cudaStream_t s) {
    // Window (target nnz per row block). A window stages [rowptr[first row], rowptr[last row + 1])
    // rounded out to 4 entries: at most window + (longest row - 1) + 6 entries. DYNWIN sizes the
    // window so that every window fits the stage (more bytes per TMA round, no slack).
    int64_t window = kWindow;
#if TF_APPLY_DYNWIN
    {
        int64_t maxrow = h->max_row_hint;  // known from the build (count pass, lattice tables); else one reduction
        if (maxrow < 0) {
            DevBuf<unsigned long long> mr;
            TF_TRY(mr.alloc(1, s, "apply plan: longest row"));
            TF_CUDA_TRY(cudaMemsetAsync(mr.p, 0, sizeof(unsigned long long), s));
            k_max_row<<<(unsigned)std::min<int64_t>((h->n + 255) / 256, 148 * 8), 256, 0, s>>>(h->rowptr, h->n, mr.p);
            TF_LAUNCH_CHECK();
            unsigned long long m = 0;
            TF_CUDA_TRY(cudaMemcpyAsync(&m, mr.p, sizeof(m), cudaMemcpyDeviceToHost, s));
            TF_CUDA_TRY(cudaStreamSynchronize(s));
            maxrow = (int64_t)m;
        }
        const int64_t fit = (int64_t)kStage - maxrow - 8;
        // short rows keep kWindow (the staged rowptr slice, kRowCap rows, bounds the window
        // too), and so does a filter whose longest row leaves less than kWindow: its long-row
        // windows take the unstaged path instead of shrinking every window
        const double avg_row = (double)h->nnz / (double)std::max<int64_t>(1, h->n);
        if (fit > kWindow && avg_row >= 16.0) window = fit & ~(int64_t)3;
    }
#endif
    const int64_t nblocks = std::max<int64_t>(1, (h->nnz + window - 1) / window);
    if (nblocks >= (int64_t)1 << 31) {
        set_error("apply plan: too many row blocks");
        return TF_ERR_OVERFLOW;
    }
    TF_TRY(dalloc(&h->plan.rb, nblocks + 1, s, "apply row blocks"));
    TF_TRY(dalloc(&h->plan.wlo, 2 * nblocks + 1, s, "apply windows"));
    DeviceInfo di;
    TF_TRY(device_info(&di));
    h->plan.grid = di.sms * kBlocksPerSM;
    h->plan.nblocks = nblocks;
    h->plan.block_nnz = (int)window;
    h->plan.stage_cap = kStage;
    // lanes per row G ~ avg/12 (G lanes of a warp gather neighbouring columns of one row),
    // U = 8 gathers in flight per lane before accumulating: measured best at c5 (avg 86):
    // G = 8, U = 8 (U = 4: +3% sensitivity, +2% density; G = 16: +25%)
    const double avg = (double)h->nnz / (double)std::max<int64_t>(1, h->n);
    int g = 1;
    while (g < 32 && 12.0 * g < avg) g *= 2;
    h->plan.group = g;
    h->plan.unroll = 8;
    // both filters: (t, x) pairs double the gather registers; U = 8 spills at G >= 2, and at
    // G = 8 U = 4 measured faster than the spilling U = 8 (2.28 vs 2.57 ms, config 5)
    h->plan.unroll_both = (g >= 8) ? 4 : 8;
    // tuning knobs (benchmarks only): TOPOFILT_APPLY_G in {1..32, power of two}, TOPOFILT_APPLY_U in {4, 8}
    if (const char *e = getenv("TOPOFILT_APPLY_G")) {
        const int v = atoi(e);
        if (v >= 1 && v <= 32 && (v & (v - 1)) == 0) h->plan.group = v;
    }
    h->plan.unroll_sens = h->plan.unroll;
    // sensitivity without the t pass (two gathers per entry): measured slower at every size
    // (config 3 84 vs 79 us, config 4 113 vs 102 us): off; tuning knob TOPOFILT_SENS_DIRECT_N (rows)
    h->plan.direct_rows = 0;
    if (const char *e = getenv("TOPOFILT_SENS_DIRECT_N")) h->plan.direct_rows = atoll(e);
    // sensitivity as t pass + programmatic dependent SpMV launch (cold, in-event: config 3
    // 79 -> 74 us, config 4 102 -> 98.6 us, config 5 2178 -> 2159 us in the bench step; knob
    // TOPOFILT_SENS_PDL=0 restores the cooperative single launch)
    h->plan.pdl = 1;
    if (const char *e = getenv("TOPOFILT_SENS_PDL")) h->plan.pdl = atoi(e) != 0;
    if (const char *e = getenv("TOPOFILT_APPLY_U")) h->plan.unroll = h->plan.unroll_sens = atoi(e) >= 8 ? 8 : 4;
    if (const char *e = getenv("TOPOFILT_APPLY_U_SENS")) h->plan.unroll_sens = atoi(e) >= 8 ? 8 : 4;
    const unsigned grid = (unsigned)std::min<int64_t>((nblocks + 256) / 256, 65535);
    k_plan<<<grid, 256, 0, s>>>(h->rowptr, h->n, nblocks, window, h->plan.rb);
    TF_LAUNCH_CHECK();
    k_plan_windows<<<grid, 256, 0, s>>>(h->rowptr, h->plan.rb, nblocks, h->plan.wlo);
    TF_LAUNCH_CHECK();

    h->plan.nchunks = -1;  // host-pipeline chunks: computed on first use (ensure_chunk_plan)
    return TF_OK;
}

__global__ void k_hadamard(const double *__restrict__ x, const double *__restrict__ dc, double *__restrict__ t,
                           int64_t r0, int64_t r1) {
    for (int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x)
        t[i] = x[i] * dc[i];
}

// t = x o dc on rows [chunk_r[piece], chunk_r[piece+1]) (the host pipeline's per-piece pass;
// same product as the fused pass of k_spmv)
tf_status launch_hadamard_piece(const tf_filter_s *h, const double *x, const double *dc, double *t, int piece,
                                cudaStream_t s) {
    const int64_t r0 = h->plan.chunk_r[piece], r1 = h->plan.chunk_r[piece + 1];
    if (r1 <= r0) return TF_OK;
    const unsigned grid = (unsigned)std::min<int64_t>((r1 - r0 + 255) / 256, 148 * 8);
    k_hadamard<<<grid, 256, 0, s>>>(x, dc, t, r0, r1);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

// Row-range chunks of the host pipeline (tf_filter_iteration_host), computed once on first use
// so device-only users never pay for them: window and first-row boundaries and the largest
// column each chunk reads (exact, from the stored columns). Synchronises `s`.
tf_status ensure_chunk_plan(tf_filter_s *h, cudaStream_t s) {
    if (h->plan.nchunks >= 0) return TF_OK;
    const int64_t nblocks = h->plan.nblocks;
    const int K = (int)std::min<int64_t>(kMaxChunks, nblocks);
    for (int i = 0; i <= K; ++i) {
        h->plan.chunk_w[i] = nblocks * i / K;
        TF_CUDA_TRY(cudaMemcpyAsync(&h->plan.chunk_r[i], h->plan.rb + h->plan.chunk_w[i], sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, s));
    }
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    // largest column each chunk reads (exact, from the stored columns): the host pipeline starts
    // chunk i once the input pieces up to the one holding that column have landed
    DevBuf<int32_t> mx;
    TF_TRY(mx.alloc(kMaxChunks, s, "chunk max columns"));
    TF_CUDA_TRY(cudaMemsetAsync(mx.p, 0xff, kMaxChunks * sizeof(int32_t), s));  // -1
    for (int i = 0; i < K; ++i) {
        const int64_t r0 = h->plan.chunk_r[i], r1 = h->plan.chunk_r[i + 1];
        if (r1 > r0) {
            k_chunk_maxcol<<<(unsigned)std::min<int64_t>((r1 - r0 + 255) / 256, 1184), 256, 0, s>>>(h->rowptr, h->cols,
                                                                                                 r0, r1, h->cols_ascending ? 1 : 0,
                                                                                                 mx.p + i);
            TF_LAUNCH_CHECK();
        }
    }
    TF_CUDA_TRY(cudaMemcpyAsync(h->plan.chunk_maxcol, mx.p, kMaxChunks * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    h->plan.nchunks = K;  // published only once complete
    return TF_OK;
}

__global__ void k_halo_pack(const double *__restrict__ src, const int32_t *__restrict__ idx, int64_t m,
                            double *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}

tf_status launch_halo_pack(const double *src, const int32_t *idx, int64_t m, double *dst, cudaStream_t s) {
    if (m <= 0) return TF_OK;
    const unsigned grid = (unsigned)std::min<int64_t>((m + 255) / 256, 148 * 8);
    k_halo_pack<<<grid, 256, 0, s>>>(src, idx, m, dst);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

tf_status launch_density_range(const tf_filter_s *h, const double *x, double *out, int chunk, cudaStream_t s) {
    return launch_spmv<0>(h, x, nullptr, out, s, 0.0, 0, h->plan.chunk_w[chunk], h->plan.chunk_w[chunk + 1]);
}

tf_status launch_sensitivity_range(const tf_filter_s *h, const double *x, const double *dc, double *out, double *tbuf,
                                   int chunk, int tpass, cudaStream_t s) {
    return launch_spmv<1>(h, x, dc, out, s, 0.0, 0, h->plan.chunk_w[chunk], h->plan.chunk_w[chunk + 1], tbuf,
                             tpass);
}

tf_status launch_sensitivity(const tf_filter_s *h, const double *x, const double *dc, double *out,
                             cudaStream_t s) {
    NvtxRange r("tf_apply/sensitivity");
    if (h->stencil.K > 0) return launch_stencil(h, x, dc, out, true, s);
    if (h->n <= h->plan.direct_rows) return launch_spmv<3>(h, x, dc, out, s);  // no t pass, ordinary launch
    return launch_spmv<1>(h, x, dc, out, s);
}

tf_status launch_sensitivity_energy(const tf_filter_s *h, const double *x, const double *U, double penal,
                                    double *out, cudaStream_t s) {
    return launch_spmv<1>(h, x, U, out, s, penal, 1);
}

tf_status launch_both(const tf_filter_s *h, const double *x, const double *dc, double *sens_out, double *dens_out,
                      cudaStream_t s) {
    NvtxRange r("tf_apply/both");
    if (h->stencil.K > 0) {
        TF_TRY(launch_stencil(h, x, dc, sens_out, true, s));
        return launch_stencil(h, x, nullptr, dens_out, false, s);
    }
    return launch_spmv<2>(h, x, dc, sens_out, s, 0.0, 0, 0, -1, nullptr, 1, dens_out);
}

// Rows [0, nrows) only (windows whose first row is below nrows; rows of the last such window
// past nrows are computed too). The sensitivity t pass still covers all n entries: the kept
// rows read columns anywhere. Stencil handles run whole.
tf_status launch_sensitivity_rows(const tf_filter_s *h, const double *x, const double *dc, double *out,
                                  int64_t nrows, cudaStream_t s) {
    NvtxRange r("tf_apply/sensitivity_rows");
    if (h->stencil.K > 0) return launch_stencil(h, x, dc, out, true, s);
    return launch_spmv<1>(h, x, dc, out, s, 0.0, 0, 0, -1, nullptr, 1, nullptr, nrows);
}

tf_status launch_density_rows(const tf_filter_s *h, const double *x, double *out, int64_t nrows, cudaStream_t s) {
    NvtxRange r("tf_apply/density_rows");
    if (h->stencil.K > 0) return launch_stencil(h, x, nullptr, out, false, s);
    return launch_spmv<0>(h, x, nullptr, out, s, 0.0, 0, 0, -1, nullptr, 1, nullptr, nrows);
}

// Rows [r0, r1): windows from the one holding r0 (found by each block with a binary search of
// the row-block table; its rows before r0 are recomputed with the same values) to the first whose
// first row is >= r1. The sensitivity t pass covers all n entries.
tf_status launch_sensitivity_rowrange(const tf_filter_s *h, const double *x, const double *dc, double *out,
                                      int64_t r0, int64_t r1, cudaStream_t s) {
    NvtxRange r("tf_apply/sensitivity_range");
    if (r1 <= r0) return TF_OK;
    if (h->stencil.K > 0) return launch_stencil(h, x, dc, out, true, s);
    return launch_spmv<1>(h, x, dc, out, s, 0.0, 0, 0, -1, nullptr, 1, nullptr, r1, r0);
}

tf_status launch_density_rowrange(const tf_filter_s *h, const double *x, double *out, int64_t r0, int64_t r1,
                                  cudaStream_t s) {
    NvtxRange r("tf_apply/density_range");
    if (r1 <= r0) return TF_OK;
    if (h->stencil.K > 0) return launch_stencil(h, x, nullptr, out, false, s);
    return launch_spmv<0>(h, x, nullptr, out, s, 0.0, 0, 0, -1, nullptr, 1, nullptr, r1, r0);
}

tf_status launch_density(const tf_filter_s *h, const double *x, double *out, cudaStream_t s) {
    NvtxRange r("tf_apply/density");
    if (h->stencil.K > 0) return launch_stencil(h, x, nullptr, out, false, s);
    return launch_spmv<0>(h, x, nullptr, out, s);
}

}  // namespace tf
