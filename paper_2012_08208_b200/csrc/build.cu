// build.cu -- GPU build of the filter weight matrix H (CSR) and its row sums Hs.
//
// Method (sec. 3.2.2 / 4.5): W_ij = rmin - dist(c_i, c_j) for midpoints within
// rmin (Eq. filter_cond), Hs = row sums, built once
// (PAPER.md:449). The paper forms the dense N x N Euclidean distance matrix
// (PAPER.md:390-396, 442-444); this build never does: a uniform cell list restricts the
// pair tests to the 3^dim neighbour bins (bin side >= rmin) and only the pairs inside
// rmin are written (the paper's own chunking remark, taken to O(N + nnz)).
//
// Steps:
//   a2 k_bbox_*     bounding box + finiteness check (host reads 7 doubles back)
//   a3 k_keys       bin key per centroid, key = (kz*ny + ky)*nx + kx
//   a4 radix sort (radix.cu), k_cellstart, k_gather_sorted (SoA copy of sorted centroids)
//   a5 k_count      block per query bin: the 3^(dim-1) candidate x-triples staged once as
//                   bin-local fp32 SoA; each warp sweeps two queries at a time with packed
//                   f32x2 math (per-lane counts); pairs inside the proven fp32 error band are
//                   decided by the exact fp64 test (R4b) -> row lengths
//   a6 scan (scan.cu) -> rowptr; nnz read back (the one data-dependent host sync)
//   a7 k_fill       block per query bin: the candidates are staged and sorted by id with a
//                   block-wide shared-memory radix sort, so ballot compaction emits every
//                   row's columns already ascending; phase A (packed fp32 sweep) lists the
//                   candidates that may lie inside rmin, phase B decides them exactly in fp64
//                   and writes cols, weights and Hs. Neighbourhoods larger than the shared
//                   memory capacity take a global-memory path plus k_rowsort. An always-on
//                   invariant flags any row whose fill length differs from its count.
// Phase boundaries are traceable with TOPOFILT_TRACE=1 (ms per phase on stderr).
//
// Exactness (R2-R4): the pair test and weight use the caller's centroid bytes,
// d2 = (dx*dx + dy*dy) + dz*dz with __dmul_rn/__dadd_rn (never contracted to FMA),
// w = max(0, rmin - __dsqrt_rn(d2)). This is the oracle's expression, so the CSR
// structure and weights are bit-identical to it.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "tf_internal.cuh"
#include "smem_sort.cuh"

namespace tf {
namespace {

// ------------------------------------------------------------------ a2: bounding box
// part[b*7 + 0..2] = min, [3..5] = max, [6] = non-finite flag (as double)
__global__ void __launch_bounds__(256) k_bbox_partial(const double *__restrict__ c, int64_t n, int dim,
                                                      double *__restrict__ part) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        for (int d = 0; d < dim; ++d) {
            double v = c[i * dim + d];
            bad |= !isfinite(v);
            lo[d] = fmin(lo[d], v);
            hi[d] = fmax(hi[d], v);
        }
    }
    __shared__ double slo[3][8], shi[3][8];
    __shared__ int sbad[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = 0; d < 3; ++d)
        for (int o = 16; o > 0; o >>= 1) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        for (int d = 0; d < 3; ++d) slo[d][warp] = lo[d], shi[d][warp] = hi[d];
        sbad[warp] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            for (int d = 0; d < 3; ++d) slo[d][0] = fmin(slo[d][0], slo[d][w]), shi[d][0] = fmax(shi[d][0], shi[d][w]);
            sbad[0] |= sbad[w];
        }
        for (int d = 0; d < 3; ++d) part[blockIdx.x * 7 + d] = slo[d][0], part[blockIdx.x * 7 + 3 + d] = shi[d][0];
        part[blockIdx.x * 7 + 6] = sbad[0] ? 1.0 : 0.0;
    }
}

__global__ void __launch_bounds__(256) k_bbox_final(const double *__restrict__ part, int nparts,
                                                    double *__restrict__ out) {
    double r[7] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY, 0.0};
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) {
        for (int d = 0; d < 3; ++d) r[d] = fmin(r[d], part[b * 7 + d]), r[3 + d] = fmax(r[3 + d], part[b * 7 + 3 + d]);
        r[6] = fmax(r[6], part[b * 7 + 6]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        for (int d = 0; d < 3; ++d) {
            r[d] = fmin(r[d], __shfl_xor_sync(0xffffffffu, r[d], o));
            r[3 + d] = fmax(r[3 + d], __shfl_xor_sync(0xffffffffu, r[3 + d], o));
        }
        r[6] = fmax(r[6], __shfl_xor_sync(0xffffffffu, r[6], o));
    }
    __shared__ double sr[8][7];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
        for (int k = 0; k < 7; ++k) sr[warp][k] = r[k];
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            for (int d = 0; d < 3; ++d) sr[0][d] = fmin(sr[0][d], sr[w][d]), sr[0][3 + d] = fmax(sr[0][3 + d], sr[w][3 + d]);
            sr[0][6] = fmax(sr[0][6], sr[w][6]);
        }
        for (int k = 0; k < 7; ++k) out[k] = sr[0][k];
    }
}

// ------------------------------------------------------------------ a3: bin keys
__device__ __forceinline__ int bin_coord(double v, double lo, double inv_s, int nb) {
    double f = floor(__dmul_rn(__dsub_rn(v, lo), inv_s));
    int k = (f < 0.0) ? 0 : (f > (double)(nb - 1) ? nb - 1 : (int)f);
    return k;
}

__global__ void __launch_bounds__(256) k_keys(const double *__restrict__ c, int64_t n, Grid g,
                                              uint32_t *__restrict__ keys, uint32_t *__restrict__ ids) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int kx = bin_coord(c[i * g.dim + 0], g.lo[0], g.inv_s, g.nb[0]);
        const int ky = bin_coord(c[i * g.dim + 1], g.lo[1], g.inv_s, g.nb[1]);
        const int kz = (g.dim == 3) ? bin_coord(c[i * g.dim + 2], g.lo[2], g.inv_s, g.nb[2]) : 0;
        keys[i] = (uint32_t)(((int64_t)kz * g.nb[1] + ky) * g.nb[0] + kx);
        ids[i] = (uint32_t)i;
    }
}

// ------------------------------------------------------------------ a4: cell start + gather
// cs[b] = first sorted position with key >= b, for b in [0, nbins]; cs[nbins] = n.
__global__ void __launch_bounds__(256) k_cellstart(const uint32_t *__restrict__ keys, int64_t n,
                                                   int64_t nbins, int32_t *__restrict__ cs) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = (i == 0) ? -1 : (int64_t)keys[i - 1];
        const int64_t cur = (i == n) ? nbins : (int64_t)keys[i];
        for (int64_t b = prev + 1; b <= cur; ++b) cs[b] = (int32_t)i;
    }
}

// SoA copy of the centroids in sorted order (exact bytes; no shift, no rounding).
__global__ void __launch_bounds__(256) k_gather_sorted(const double *__restrict__ c, int64_t n, int dim,
                                                       const uint32_t *__restrict__ ids,
                                                       double *__restrict__ sxyz, double4 *__restrict__ aos) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = ids[p];
        double v[3] = {0.0, 0.0, 0.0};
        for (int d = 0; d < dim; ++d) {
            v[d] = c[i * dim + d];
            if (sxyz) sxyz[d * n + p] = v[d];
        }
        // the group kernels gather whole points: (x, y, z, id) in one 32-byte sector
        if (aos) aos[p] = make_double4(v[0], v[1], v[2], __longlong_as_double((long long)i));
    }
}

// ------------------------------------------------------------------ neighbourhood helpers
using SortedPts = SortedPtsView;

__device__ __forceinline__ void decode_bin(int64_t b, const Grid &g, int &bx, int &by, int &bz) {
    bx = (int)(b % g.nb[0]);
    const int64_t t = b / g.nb[0];
    by = (int)(t % g.nb[1]);
    bz = (int)(t / g.nb[1]);
}

// Contiguous sorted-position range of the x-triple (bx-1..bx+1) at row (by+dy, bz+dz).
template <int DIM>
__device__ __forceinline__ void xtriple_range(int r, int bx, int by, int bz, const Grid &g,
                                              const int32_t *cs, int &s, int &e) {
    const int dz = (DIM == 3) ? (r / 3 - 1) : 0;
    const int dy = r % 3 - 1;
    const int yy = by + dy, zz = bz + dz;
    s = e = 0;
    if (yy < 0 || yy >= g.nb[1] || zz < 0 || zz >= g.nb[2]) return;
    const int xl = max(bx - 1, 0), xh = min(bx + 1, g.nb[0] - 1);
    const int64_t row = ((int64_t)zz * g.nb[1] + yy) * g.nb[0];
    s = cs[row + xl];
    e = cs[row + xh + 1];
}

// ------------------------------------------------------------------ a5/a7 shared machinery
// fp32 bin-local prefilter (R4b). Candidates of a query bin are staged as
// float offsets from the bin centre o: u = fl32(fl64(c - o)). With every staged point within
// M = 1.5*s*(1+1e-4) of o per component, |d2_f32 - d2| <= E = 1e-5*M^2 (+1e-12*r2 for the
// fp64 rounding of the reference test); derivation in DESIGN.md. Hence
//   d2f <  t_in  => the exact fp64 test accepts,   d2f >= t_out => it rejects,
// and only pairs in [t_in, t_out) -- plus every pair the fill pass keeps -- are decided or
// weighted by the exact fp64 expression on the original centroid bytes.
struct BinView {
    int bx, by, bz;
    double ox, oy, oz;  // bin centre (fp64)
};

__device__ __forceinline__ BinView bin_view(int64_t b, const Grid &g) {
    BinView v;
    decode_bin(b, g, v.bx, v.by, v.bz);
    v.ox = g.lo[0] + ((double)v.bx + 0.5) * g.s;
    v.oy = g.lo[1] + ((double)v.by + 0.5) * g.s;
    v.oz = (g.dim == 3) ? g.lo[2] + ((double)v.bz + 0.5) * g.s : 0.0;
    return v;
}

__device__ __forceinline__ float4 local_f32(double x, double y, double z, const BinView &v) {
    return make_float4(__double2float_rn(x - v.ox), __double2float_rn(y - v.oy), __double2float_rn(z - v.oz), 0.f);
}

template <int DIM>
__device__ __forceinline__ float d2_f32(const float4 &a, const float4 &b) {
    const float dx = a.x - b.x, dy = a.y - b.y;
    float d2 = fmaf(dy, dy, dx * dx);
    if (DIM == 3) {
        const float dz = a.z - b.z;
        d2 = fmaf(dz, dz, d2);
    }
    return d2;
}

// ---- packed fp32x2 arithmetic (sm_100a FADD2 / FMUL2 / FFMA2): two candidates per lane
typedef unsigned long long f2u;
__device__ __forceinline__ f2u f2_pack(float a, float b) {
    return ((f2u)__float_as_uint(b) << 32) | (f2u)__float_as_uint(a);
}
__device__ __forceinline__ float f2_lo(f2u v) { return __uint_as_float((unsigned)(v & 0xffffffffull)); }
__device__ __forceinline__ float f2_hi(f2u v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ f2u f2_sub(f2u a, f2u b) {
    f2u r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2u f2_mul(f2u a, f2u b) {
    f2u r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2u f2_fma(f2u a, f2u b, f2u c) {
    f2u r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
// d2 of two staged candidates (SoA float pairs) against the query (q?2 = (q, q)).
// Three roundings per result, like d2_f32: the R4b error bound applies unchanged.
template <int DIM>
__device__ __forceinline__ f2u d2_f32x2(f2u X, f2u Y, f2u Z, f2u qx2, f2u qy2, f2u qz2) {
    const f2u dx = f2_sub(X, qx2), dy = f2_sub(Y, qy2);
    f2u d2;
    if (DIM == 3) {
        const f2u dz = f2_sub(Z, qz2);
        d2 = f2_fma(dy, dy, f2_mul(dz, dz));
    } else {
        d2 = f2_mul(dy, dy);
    }
    return f2_fma(dx, dx, d2);
}
constexpr float kFar = 1e30f;  // padding coordinate: d2 overflows to +inf, never "maybe"

// 3^(dim-1) contiguous x-triple ranges of a bin, computed by lanes 0..NR-1 into shared memory.
template <int DIM>
__device__ __forceinline__ void load_ranges(const BinView &v, const Grid &g, const int32_t *cs, int *rs, int *rp) {
    constexpr int NR = (DIM == 3) ? 9 : 3;
    if (threadIdx.x < NR) {
        int s, e;
        xtriple_range<DIM>(threadIdx.x, v.bx, v.by, v.bz, g, cs, s, e);
        rs[threadIdx.x] = s;
        rp[threadIdx.x + 1] = e - s;  // lengths, prefix-summed below
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        rp[0] = 0;
        for (int r = 0; r < NR; ++r) rp[r + 1] += rp[r];
    }
    __syncthreads();
}

// Largest candidate set of any bin (sizes the shared-memory staging).
template <int DIM>
__global__ void __launch_bounds__(256) k_binstats(const int32_t *__restrict__ cs, Grid g, int32_t *__restrict__ stats) {
    constexpr int NR = (DIM == 3) ? 9 : 3;
    int best = 0;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < g.nbins; b += (int64_t)gridDim.x * blockDim.x) {
        if (cs[b] == cs[b + 1]) continue;
        int bx, by, bz;
        decode_bin(b, g, bx, by, bz);
        int C = 0;
        for (int r = 0; r < NR; ++r) {
            int s, e;
            xtriple_range<DIM>(r, bx, by, bz, g, cs, s, e);
            C += e - s;
        }
        best = max(best, C);
    }
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&stats[0], best);
}

// ------------------------------------------------------------------ a5: count pass
// Longest row for the apply plan: an atomic only when a row beats the value already seen (the
// plain read is a cached broadcast; the maximum settles after a few rows, so atomics stay rare).
// Each warp keeps its own maximum and reports it once per block; a stale cached read only costs
// an extra atomic.
__device__ __forceinline__ void note_max(int32_t *m, int v) {
    if (v > 0 && v > *m) atomicMax(m, v);
}

// Block per query bin, WARPS warps, one warp per query. The bin's candidates (the 3^(dim-1)
// contiguous x-triples) are staged once as bin-local fp32 SoA (padded with far sentinels to
// a multiple of 64) plus their sorted position for the rare exact re-test; each query sweeps
// them 64 at a time, two per lane with packed f32x2 math: surely-in pairs are counted by
// ballot/popc, band pairs are decided by the exact fp64 test. Neighbourhoods over `cap`
// (or inputs where the fp32 band is unusable) fall back to exact fp64 tests from the SoA.
template <int DIM, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_count(SortedPts P, Grid g, int cap, int32_t *__restrict__ counts,
                                                       int32_t *__restrict__ maxrow) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int NR = (DIM == 3) ? 9 : 3;
    __shared__ int rs[NR], rp[NR + 1];
    const int64_t b = blockIdx.x;
    const int q0 = P.cs[b], q1 = P.cs[b + 1];
    if (q0 == q1) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int wmax = 0;  // lane 0: longest row this warp counted
    const BinView v = bin_view(b, g);
    load_ranges<DIM>(v, g, P.cs, rs, rp);
    const int C = rp[NR];
    const double r2 = g.r2;
    if (C <= cap && g.use_f32) {
        const int CP = (C + 63) & ~63;  // padded length
        float *FX = reinterpret_cast<float *>(smem_raw);
        float *FY = FX + cap;
        float *FZ = FY + cap;
        int32_t *POS = reinterpret_cast<int32_t *>(FZ + cap);
        for (int r = warp; r < NR; r += WARPS) {
            const int s = rs[r], off = rp[r], len = rp[r + 1] - rp[r];
            for (int i = lane; i < len; i += 32) {
                const int p = s + i;
                const float4 f = local_f32(P.x[p], P.y[p], (DIM == 3) ? P.z[p] : 0.0, v);
                FX[off + i] = f.x;
                FY[off + i] = f.y;
                FZ[off + i] = f.z;
                POS[off + i] = p;
            }
        }
        for (int t = C + tid; t < CP; t += WARPS * 32) FX[t] = kFar, FY[t] = kFar, FZ[t] = kFar, POS[t] = 0;
        __syncthreads();
        const float t_in = g.t_in, t_out = g.t_out;
        const f2u *X2 = reinterpret_cast<const f2u *>(FX), *Y2 = reinterpret_cast<const f2u *>(FY),
                  *Z2 = reinterpret_cast<const f2u *>(FZ);
        // two queries per warp pass (the second may be absent: far sentinel, never in or band):
        // the staged candidate pairs are loaded once for both; per-lane counts packed as
        // lo16 + hi16 (<= 2*32*... < 65536 per lane) into one warp reduction.
        for (int q = q0 + warp; q < q1; q += 2 * WARPS) {
            const int qb = q + WARPS;
            const bool hasb = qb < q1;
            const double ax = P.x[q], ay = P.y[q], az = (DIM == 3) ? P.z[q] : 0.0;
            const double bx = hasb ? P.x[qb] : 0.0, by = hasb ? P.y[qb] : 0.0,
                         bz = (DIM == 3 && hasb) ? P.z[qb] : 0.0;
            const float4 fa = local_f32(ax, ay, az, v);
            const float4 fb = hasb ? local_f32(bx, by, bz, v) : make_float4(kFar, kFar, kFar, 0.f);
            const f2u ax2 = f2_pack(fa.x, fa.x), ay2 = f2_pack(fa.y, fa.y), az2 = f2_pack(fa.z, fa.z);
            const f2u bx2 = f2_pack(fb.x, fb.x), by2 = f2_pack(fb.y, fb.y), bz2 = f2_pack(fb.z, fb.z);
            int cnt = 0;  // query a in the low 16 bits, query b in the high 16 bits
            auto exact = [&](int t, double x, double y, double z) -> bool {
                const int p = POS[t];
                return pair_d2<DIM>(x, y, z, P.x[p], P.y[p], (DIM == 3) ? P.z[p] : 0.0) < r2;
            };
            for (int k0 = 0; k0 < CP / 2; k0 += 32) {
                const int k = k0 + lane;
                const f2u X = X2[k], Y = Y2[k], Z = (DIM == 3) ? Z2[k] : 0ull;
                const f2u da = d2_f32x2<DIM>(X, Y, Z, ax2, ay2, az2);
                const f2u db = d2_f32x2<DIM>(X, Y, Z, bx2, by2, bz2);
                const float a0 = f2_lo(da), a1 = f2_hi(da), b0 = f2_lo(db), b1 = f2_hi(db);
                if (a0 < t_in) cnt += 1;
                if (a1 < t_in) cnt += 1;
                if (b0 < t_in) cnt += 0x10000;
                if (b1 < t_in) cnt += 0x10000;
                const bool ba0 = !(a0 < t_in) && a0 < t_out, ba1 = !(a1 < t_in) && a1 < t_out;
                const bool bb0 = !(b0 < t_in) && b0 < t_out, bb1 = !(b1 < t_in) && b1 < t_out;
                if (ba0 || ba1 || bb0 || bb1) {
                    if (ba0 && exact(2 * k, ax, ay, az)) cnt += 1;
                    if (ba1 && exact(2 * k + 1, ax, ay, az)) cnt += 1;
                    if (bb0 && exact(2 * k, bx, by, bz)) cnt += 0x10000;
                    if (bb1 && exact(2 * k + 1, bx, by, bz)) cnt += 0x10000;
                }
            }
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            if (lane == 0) {
                counts[P.id[q]] = cnt & 0xffff;
                if (hasb) counts[P.id[qb]] = cnt >> 16;
                wmax = max(wmax, max(cnt & 0xffff, cnt >> 16));
            }
        }
    } else {
        for (int q = q0 + warp; q < q1; q += WARPS) {
            const double qx = P.x[q], qy = P.y[q], qz = (DIM == 3) ? P.z[q] : 0.0;
            int cnt = 0;
            for (int r = 0; r < NR; ++r) {
                const int s = rs[r], e = rs[r] + rp[r + 1] - rp[r];
                for (int base = s; base < e; base += 32) {
                    const int p = base + lane;
                    bool ok = false;
                    if (p < e) ok = pair_d2<DIM>(qx, qy, qz, P.x[p], P.y[p], (DIM == 3) ? P.z[p] : 0.0) < r2;
                    cnt += __popc(__ballot_sync(0xffffffffu, ok));
                }
            }
            if (lane == 0) counts[P.id[q]] = cnt, wmax = max(wmax, cnt);
        }
    }
    if (lane == 0) note_max(maxrow, wmax);
}

// ------------------------------------------------------------------ a7: fill pass
// (block_radix_sort_smem: smem_sort.cuh)

// Shared-memory layout of the fill staging: five 4-byte arrays of `cap` entries (20 B per
// candidate), reused across the phases of k_fill:
//   staging:  b[0] = sorted-SoA position (run order), (b[1], b[2]) = (key = id - lo, staging index)
//   sort:     ping-pong between (b[1], b[2]) and (b[3], b[4])
//   sweeps:   skey (ids - lo, sorted), sp (sorted-SoA position of sorted candidate t, written in
//             place over perm), fx/fy/fz (bin-local fp32, sorted) in the free sort pair and b[0].
struct FillSmem {
    uint32_t *b[5];
    __device__ FillSmem(unsigned char *raw, int cap) {
        for (int k = 0; k < 5; ++k) b[k] = reinterpret_cast<uint32_t *>(raw) + (size_t)k * cap;
    }
    static constexpr size_t bytes_per() { return 5 * sizeof(uint32_t); }
};

constexpr int kListCap = 128;  // per-warp compacted candidate list (phase A -> phase B)

// Phase B over list[0, nl): exact fp64 test on the original centroid bytes, weight, CSR write
// at rowptr[row] + rank (ballot compaction keeps the sorted order), Hs partial per lane.
// FULL: nl is a multiple of 32 (every lane has an entry: no bounds checks, no divergence).
template <int DIM, bool FULL>
__device__ __forceinline__ void fill_flush(const SortedPts &P, const uint32_t *skey, const uint32_t *sp,
                                           const int32_t *list, int nl, int lo, double qx, double qy, double qz,
                                           double r2, double rmin, int &wpos, double &hsum,
                                           int32_t *__restrict__ colsq, double *__restrict__ valsq) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    for (int e0 = 0; e0 < nl; e0 += 32) {
        const int e = e0 + lane;
        const bool have = FULL || e < nl;
        const int t = have ? list[e] : list[e0];  // idle lanes redo a valid entry, then drop it
        const int p = (int)sp[t];
        const double d2 = pair_d2<DIM>(qx, qy, qz, P.x[p], P.y[p], (DIM == 3) ? P.z[p] : 0.0);
        const bool ok = have && d2 < r2;
        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
        const double w = weight_of(rmin, d2);
        if (ok) {
            const int k = wpos + __popc(bal & lt);  // row-relative: the row's base is hoisted
            TF_DCHECK(t >= 0 && p >= 0);
            colsq[k] = (int32_t)skey[t] + lo;
            valsq[k] = w;
            hsum += w;
        }
        wpos += __popc(bal);
    }
}

// Block per query bin. Stage the candidates, sort them by id with the whole block (so
// ballot compaction emits every row's columns ascending); phase A: fp32 prefilter -> per-
// warp list of candidates that may lie inside rmin; phase B: exact fp64 test on the original
// centroid bytes, weight, CSR write, Hs.
template <int DIM, int WARPS>
#ifdef TF_FILL_MINB
#define TF_FILL_BOUNDS __launch_bounds__(WARPS * 32, TF_FILL_MINB)
#else
#define TF_FILL_BOUNDS __launch_bounds__(WARPS * 32)
#endif
__global__ void TF_FILL_BOUNDS k_fill(SortedPts P, Grid g, const int64_t *__restrict__ rowptr,
                                                     int32_t *__restrict__ cols, double *__restrict__ vals,
                                                     double *__restrict__ hs, int cap,
                                                     int32_t *__restrict__ large_rows,
                                                     int32_t *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int NR = (DIM == 3) ? 9 : 3;
    __shared__ int rs[NR], rp[NR + 1];
    static_assert(kListCap <= 256, "lists alias the sort's digit-counter table");
    __shared__ int32_t wc[WARPS][256];  // radix digit counters during the sort, per-warp lists after
    __shared__ int32_t wsum[WARPS];
    __shared__ int s_lo, s_hi;
    const int64_t b = blockIdx.x;
    const int q0 = P.cs[b], q1 = P.cs[b + 1];
    if (q0 == q1) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const BinView v = bin_view(b, g);
    load_ranges<DIM>(v, g, P.cs, rs, rp);
    const int C = rp[NR];
    const double r2 = g.r2, rmin = g.rmin;

    if (C <= cap) {
        FillSmem S(smem_raw, cap);
        // ---- stage (run order) + id range
        int lo = 0x7fffffff, hi = 0;
        for (int r = warp; r < NR; r += WARPS) {
            const int s = rs[r], off = rp[r], len = rp[r + 1] - rp[r];
            for (int i = lane; i < len; i += 32) {
                const int p = s + i;
                const int32_t id = P.id[p];
                S.b[0][off + i] = (uint32_t)p;
                S.b[1][off + i] = (uint32_t)id;
                S.b[2][off + i] = (uint32_t)(off + i);
                lo = min(lo, id);
                hi = max(hi, id);
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (tid == 0) s_lo = 0x7fffffff, s_hi = 0;
        __syncthreads();
        if (lane == 0) atomicMin(&s_lo, lo), atomicMax(&s_hi, hi);
        __syncthreads();
        lo = s_lo;
        hi = s_hi;
        for (int t = tid; t < C; t += WARPS * 32) S.b[1][t] -= (uint32_t)lo;
        __syncthreads();
        // ---- sort by id (whole block)
        const int bits = (hi > lo) ? 32 - __clz((unsigned)(hi - lo)) : 0;
        const int which = block_radix_sort_smem<WARPS>(S.b[1], S.b[2], S.b[3], S.b[4], C, bits, wc, wsum);
        const uint32_t *skey = which ? S.b[3] : S.b[1];
        uint32_t *sp = which ? S.b[4] : S.b[2];  // perm, then overwritten in place by positions
        float *fx = reinterpret_cast<float *>(which ? S.b[1] : S.b[3]);
        float *fy = reinterpret_cast<float *>(which ? S.b[2] : S.b[4]);
        float *fz = reinterpret_cast<float *>(S.b[0]);
        for (int t = tid; t < C; t += WARPS * 32) sp[t] = S.b[0][sp[t]];  // perm -> sorted-SoA position
        __syncthreads();
        const int CP = (C + 63) & ~63;
        for (int t = tid; t < CP; t += WARPS * 32) {
            if (t < C) {
                const int p = (int)sp[t];
                const float4 f = local_f32(P.x[p], P.y[p], (DIM == 3) ? P.z[p] : 0.0, v);
                fx[t] = f.x, fy[t] = f.y, fz[t] = f.z;
            } else {
                fx[t] = kFar, fy[t] = kFar, fz[t] = kFar;
            }
        }
        __syncthreads();
        // ---- queries: one warp each
        int32_t *list = wc[warp];
        const float t_out = g.use_f32 ? g.t_out : INFINITY;
        const f2u *X2 = reinterpret_cast<const f2u *>(fx), *Y2 = reinterpret_cast<const f2u *>(fy),
                  *Z2 = reinterpret_cast<const f2u *>(fz);
        for (int q = q0 + warp; q < q1; q += WARPS) {
            const double qx = P.x[q], qy = P.y[q], qz = (DIM == 3) ? P.z[q] : 0.0;
            const float4 fq = local_f32(qx, qy, qz, v);
            const f2u qx2 = f2_pack(fq.x, fq.x), qy2 = f2_pack(fq.y, fq.y), qz2 = f2_pack(fq.z, fq.z);
            const int32_t qid = P.id[q];
            const int64_t base = rowptr[qid];
            int32_t *colsq = cols + base;
            double *valsq = vals + base;
            int wpos = 0, nl = 0;
            double hsum = 0.0;
            for (int k0 = 0; k0 < CP / 2; k0 += 32) {  // warp-uniform trip count
                const int k = k0 + lane;
                // candidates 2k and 2k+1 (sorted order): phase A keeps every "maybe" in order
                const f2u d2 = d2_f32x2<DIM>(X2[k], Y2[k], (DIM == 3) ? Z2[k] : 0ull, qx2, qy2, qz2);
                const bool m0 = f2_lo(d2) < t_out, m1 = f2_hi(d2) < t_out;
                const uint32_t b0 = __ballot_sync(0xffffffffu, m0), b1 = __ballot_sync(0xffffffffu, m1);
                const int pre = nl + __popc(b0 & lt_mask) + __popc(b1 & lt_mask);
                TF_DCHECK(pre + 1 < kListCap || !(m0 || m1));  // nl < 64 before a 64-wide chunk
                if (m0) list[pre] = 2 * k;
                if (m1) list[pre + (m0 ? 1 : 0)] = 2 * k + 1;
                nl += __popc(b0) + __popc(b1);
                if (nl >= kListCap - 64) {
                    // flush whole 32-entry chunks only; the < 32 tail moves to the front
                    const int full = nl & ~31;
                    __syncwarp();
                    fill_flush<DIM, true>(P, skey, sp, list, full, lo, qx, qy, qz, r2, rmin, wpos, hsum, colsq,
                                          valsq);
                    const int tail = nl - full;
                    const int moved = (lane < tail) ? list[full + lane] : 0;
                    __syncwarp();
                    if (lane < tail) list[lane] = moved;
                    __syncwarp();
                    nl = tail;
                }
            }
            __syncwarp();
            fill_flush<DIM, false>(P, skey, sp, list, nl, lo, qx, qy, qz, r2, rmin, wpos, hsum, colsq, valsq);
            __syncwarp();
            for (int o = 16; o > 0; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
            if (lane == 0) {
                hs[qid] = hsum;
                // the fill must write exactly the row length the count pass produced
                if (base + wpos != rowptr[qid + 1]) atomicOr(&stats[2], 1);
            }
        }
    } else {
        // ---- large neighbourhood: exact tests straight from the sorted SoA, written in
        // candidate order; the rows are listed and sorted afterwards by k_rowsort.
        for (int q = q0 + warp; q < q1; q += WARPS) {
            const double qx = P.x[q], qy = P.y[q], qz = (DIM == 3) ? P.z[q] : 0.0;
            const int32_t qid = P.id[q];
            const int64_t base = rowptr[qid];
            int wpos = 0;
            double hsum = 0.0;
            for (int r = 0; r < NR; ++r) {
                const int s = rs[r], e = rs[r] + rp[r + 1] - rp[r];
                for (int b0 = s; b0 < e; b0 += 32) {
                    const int p = b0 + lane;
                    bool ok = false;
                    double d2 = 0.0;
                    if (p < e) {
                        d2 = pair_d2<DIM>(qx, qy, qz, P.x[p], P.y[p], (DIM == 3) ? P.z[p] : 0.0);
                        ok = d2 < r2;
                    }
                    const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                    if (ok) {
                        const double w = weight_of(rmin, d2);
                        const int64_t k = base + wpos + __popc(bal & lt_mask);
                        cols[k] = P.id[p];
                        vals[k] = w;
                        hsum += w;
                    }
                    wpos += __popc(bal);
                }
            }
            for (int o = 16; o > 0; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
            if (lane == 0) {
                hs[qid] = hsum;
                if (base + wpos != rowptr[qid + 1]) atomicOr(&stats[2], 1);
                const int slot = atomicAdd(&stats[1], 1);
                large_rows[slot] = qid;
            }
        }
    }
}

// ------------------------------------------------------------------ a7 fill for short rows
// Warp per query (sorted order, so the warps of a block share their bins through L1), used
// when the longest row (count pass) is <= 32*KS. No staging and no block sort: every candidate
// of the 3^(dim-1) x-triples takes the exact fp64 test (pair_d2, the count pass's exact
// expression on the same bytes, so the accepted set equals the counted one), the accepted
// (id, d2) pairs are compacted into a per-warp list, and each entry's place in the ascending
// row is its rank among the row's (distinct) ids: rank = #{ids < id}, counted against the list
// four ids per shared load. Rows are a few dozen entries, so the O(K^2/32) rank costs less
// than staging + sorting the bin's candidates -- estimated; measured 1.4x slower than k_fill at
// configs 3 and 4 (issue-bound: the rank loop is 31% of the instructions, the query's bin
// decode 7%), so it is opt-in (TOPOFILT_FILL=warp) and kept parity-tested.
constexpr int kFillWarpWarps = 8;

template <int DIM, int KS>
__global__ void __launch_bounds__(kFillWarpWarps * 32)
    k_fill_warp(SortedPts P, const uint32_t *__restrict__ keys, Grid g, int64_t n,
                const int64_t *__restrict__ rowptr, int32_t *__restrict__ cols, double *__restrict__ vals,
                double *__restrict__ hs, int32_t *__restrict__ stats) {
    constexpr int NR = (DIM == 3) ? 9 : 3;
    constexpr int CAPK = 32 * KS;
    __shared__ __align__(16) int32_t s_id[kFillWarpWarps][CAPK + 4];
    __shared__ double s_d2[kFillWarpWarps][CAPK];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const double r2 = g.r2, rmin = g.rmin;
    int32_t *sid = s_id[warp];
    double *sd2 = s_d2[warp];
    for (int64_t q = (int64_t)blockIdx.x * kFillWarpWarps + warp; q < n; q += (int64_t)gridDim.x * kFillWarpWarps) {
        int bx, by, bz;
        decode_bin((int64_t)keys[q], g, bx, by, bz);
        int rs_ = 0, re_ = 0;
        if (lane < NR) xtriple_range<DIM>(lane, bx, by, bz, g, P.cs, rs_, re_);
        const double qx = P.x[q], qy = P.y[q], qz = (DIM == 3) ? P.z[q] : 0.0;
        const int32_t qid = P.id[q];
        const int64_t base = rowptr[qid];
        const int64_t len = rowptr[qid + 1] - base;
        // the runs flattened: candidate t of the query lies in run r with ex[r] <= t < ex[r+1] at
        // sorted position st[r] + (t - ex[r]); every lane holds the NR run bounds in registers
        int incl = re_ - rs_;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int ex[NR + 1], st[NR];
        ex[0] = 0;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            ex[r + 1] = __shfl_sync(0xffffffffu, incl, r);
            st[r] = __shfl_sync(0xffffffffu, rs_, r);
        }
        const int C = ex[NR];
        int nacc = 0;
        for (int t0 = 0; t0 < C; t0 += 64) {
            bool ok[2];
            double d2[2];
            int pp[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int t = t0 + 32 * u + lane;
                int p = st[0] + t;
#pragma unroll
                for (int r = 1; r < NR; ++r)
                    if (t >= ex[r]) p = st[r] + (t - ex[r]);
                pp[u] = p;
                ok[u] = false;
                d2[u] = 0.0;
                if (t < C) {
                    d2[u] = pair_d2<DIM>(qx, qy, qz, P.x[p], P.y[p], (DIM == 3) ? P.z[p] : 0.0);
                    ok[u] = d2[u] < r2;
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t bal = __ballot_sync(0xffffffffu, ok[u]);
                if (ok[u]) {
                    const int k = nacc + __popc(bal & lt);
                    if (k < CAPK) sid[k] = P.id[pp[u]], sd2[k] = d2[u];
                }
                nacc += __popc(bal);
            }
        }
        const int K = min(nacc, CAPK);
        if (lane < 4) sid[K + lane] = 0x7fffffff;  // pads of the 4-wide rank loads
        __syncwarp();
        int32_t myid[KS];
        int rank[KS];
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            const int e = lane + 32 * t;
            myid[t] = (e < K) ? sid[e] : 0x7fffffff;
            rank[t] = 0;
        }
        for (int j = 0; j < K; j += 4) {
            const int4 v = *reinterpret_cast<const int4 *>(sid + j);
#pragma unroll
            for (int t = 0; t < KS; ++t)
                rank[t] += (v.x < myid[t]) + (v.y < myid[t]) + (v.z < myid[t]) + (v.w < myid[t]);
        }
        double hsum = 0.0;
#pragma unroll
        for (int t = 0; t < KS; ++t) {
            const int e = lane + 32 * t;
            if (e < K && rank[t] < len) {
                const double w = weight_of(rmin, sd2[e]);
                cols[base + rank[t]] = myid[t];
                vals[base + rank[t]] = w;
                hsum += w;
            }
        }
        for (int o = 16; o > 0; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
        if (lane == 0) {
            hs[qid] = hsum;
            // the fill must write exactly the row length the count pass produced
            if ((int64_t)nacc != len) atomicOr(&stats[2], 1);
        }
        __syncwarp();  // the list is reused by the warp's next query
    }
}

// ------------------------------------------------------------------ row sort (large path only)
// Sorts (col, val) of each listed row ascending by col. Uses the all-ascending bitonic
// network (mirror step i ^ (k-1), then half-cleaners i ^ j), so indices >= L act as +inf
// and need no padding. Shared memory when the row fits, else in place in global memory.
constexpr int kSortThreads = 512;

__device__ __forceinline__ void ce_pair(int32_t *kc, double *kv, int i, int l) {
    const int32_t a = kc[i], bb = kc[l];
    if (a > bb) {
        kc[i] = bb;
        kc[l] = a;
        const double t = kv[i];
        kv[i] = kv[l];
        kv[l] = t;
    }
}

__device__ void bitonic_block(int32_t *kc, double *kv, int L) {
    int P2 = 1;
    while (P2 < L) P2 <<= 1;
    for (int k = 2; k <= P2; k <<= 1) {
        for (int i = threadIdx.x; i < P2; i += blockDim.x) {
            const int l = i ^ (k - 1);
            if (l > i && l < L) ce_pair(kc, kv, i, l);
        }
        __syncthreads();
        for (int j = k >> 2; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P2; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i && l < L) ce_pair(kc, kv, i, l);
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(kSortThreads) k_rowsort(const int32_t *__restrict__ rows,
                                                          const int32_t *__restrict__ stats,
                                                          const int64_t *__restrict__ rowptr,
                                                          int32_t *__restrict__ cols,
                                                          double *__restrict__ vals, int smem_cap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *sv = reinterpret_cast<double *>(smem_raw);
    int32_t *sc = reinterpret_cast<int32_t *>(sv + smem_cap);
    const int nrows = stats[1];
    for (int li = blockIdx.x; li < nrows; li += gridDim.x) {
        const int32_t row = rows[li];
        const int64_t s = rowptr[row];
        const int L = (int)(rowptr[row + 1] - s);
        if (L <= smem_cap) {
            for (int i = threadIdx.x; i < L; i += blockDim.x) sc[i] = cols[s + i], sv[i] = vals[s + i];
            __syncthreads();
            bitonic_block(sc, sv, L);
            for (int i = threadIdx.x; i < L; i += blockDim.x) cols[s + i] = sc[i], vals[s + i] = sv[i];
            __syncthreads();
        } else {
            bitonic_block(cols + s, vals + s, L);
        }
    }
}

// ------------------------------------------------------------------ host helpers
int ceil_log2(int64_t v) {
    int b = 0;
    while (((int64_t)1 << b) < v) ++b;
    return b;
}

// Round a double to float toward -inf / +inf (conservative prefilter thresholds).
float f32_down(double v) {
    float f = (float)v;
    if ((double)f > v) f = nextafterf(f, -INFINITY);
    return f;
}
float f32_up(double v) {
    float f = (float)v;
    if ((double)f < v) f = nextafterf(f, INFINITY);
    return f;
}

tf_status make_grid(const double *bb, int64_t n, int dim, double rmin, Grid *g) {
    g->dim = dim;
    g->rmin = rmin;
    g->r2 = rmin * rmin;  // the oracle's r2 = rmin*rmin (one rounding, same on both sides)
    double lo[3] = {0, 0, 0}, span[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) lo[d] = bb[d], span[d] = bb[3 + d] - bb[d];
    // Bin side s >= rmin*(1+1e-6): a pair within rmin lies in adjacent bins (R5).
    double s = rmin * (1.0 + 1e-6);
    if (const char *e = getenv("TOPOFILT_BIN_SCALE")) {  // tuning knob (benchmarks only): f in [1, 4]
        const double f = atof(e);
        if (f >= 1.0 && f <= 4.0) s *= f;
    }
    const double cap_total = std::max(4.0 * (double)n, 64.0);
    for (int it = 0; it < 4096; ++it) {
        double total = 1.0;
        bool ok = true;
        for (int d = 0; d < dim; ++d) {
            const double nb = floor(span[d] / s) + 1.0;
            if (!(nb <= (double)(1 << 26))) ok = false;  // keeps the binning error << 1e-6
            total *= nb;
        }
        if (ok && total <= cap_total) break;
        s *= 1.25;
    }
    if (!isfinite(s) || !(s > 0)) {
        set_error("bin side overflow (span too large for rmin)");
        return TF_ERR_INVALID;
    }
    g->s = s;
    g->inv_s = 1.0 / s;
    int64_t nbins = 1;
    for (int d = 0; d < 3; ++d) {
        g->lo[d] = lo[d];
        g->nb[d] = (d < dim) ? (int)(floor(span[d] / s) + 1.0) : 1;
        nbins *= g->nb[d];
    }
    g->nbins = nbins;
    // fp32 prefilter band (R4b): staged offsets from the bin centre are within
    // M per component; |d2_f32 - d2| <= 1e-5 M^2; 1e-12 r2 covers the fp64 reference rounding.
    const double M = 1.5 * s * (1.0 + 1e-4);
    const double E = 1e-5 * M * M + 1e-12 * g->r2;
    g->use_f32 = (s > 1e-15 && s < 1e15) ? 1 : 0;
    g->t_in = (g->r2 - E > 0) ? f32_down(g->r2 - E) : -1.0f;
    g->t_out = f32_up(g->r2 + E);
    return TF_OK;
}

template <int DIM, int WARPS>
tf_status launch_count(const SortedPts &P, const Grid &g, int cap, int32_t *counts, int32_t *maxrow, cudaStream_t s) {
    const size_t smem = (size_t)cap * (3 * sizeof(float) + sizeof(int32_t));
    auto kern = k_count<DIM, WARPS>;
    // always set: dynamic + static shared memory above 48 KB needs the opt-in attribute
    TF_TRY(allow_dynamic_smem(kern, smem));
    kern<<<(unsigned)g.nbins, WARPS * 32, smem, s>>>(P, g, cap, counts, maxrow);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

template <int DIM, int WARPS>
tf_status launch_fill(const SortedPts &P, const Grid &g, tf_filter_s *h, int cap, int32_t *large_rows,
                      int32_t *stats, cudaStream_t s) {
    const size_t smem = (size_t)cap * FillSmem::bytes_per();
    TF_TRY(allow_dynamic_smem(k_fill<DIM, WARPS>, smem));
#ifdef TF_FILL_CARVEOUT
    TF_CUDA_TRY(cudaFuncSetAttribute(k_fill<DIM, WARPS>, cudaFuncAttributePreferredSharedMemoryCarveout, TF_FILL_CARVEOUT));
#endif
    k_fill<DIM, WARPS><<<(unsigned)g.nbins, WARPS * 32, smem, s>>>(P, g, h->rowptr, h->cols, h->vals, h->hs,
                                                                   cap, large_rows, stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

template <int DIM, int KS>
tf_status launch_fill_warp(const SortedPts &P, const uint32_t *keys, const Grid &g, int64_t n, tf_filter_s *h,
                           int sms, int32_t *stats, cudaStream_t s) {
    const int64_t need = (n + kFillWarpWarps - 1) / kFillWarpWarps;
    const unsigned grid = (unsigned)std::min<int64_t>(need, (int64_t)sms * 32);
    k_fill_warp<DIM, KS><<<grid, kFillWarpWarps * 32, 0, s>>>(P, keys, g, n, h->rowptr, h->cols, h->vals, h->hs,
                                                                stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

}  // namespace

tf_status build_filter_device(const double *c, int64_t n, int dim, double rmin, int flags, cudaStream_t s,
                              tf_filter_s *h) {
    const bool speculate = (flags & kBuildNoSpeculation) == 0;
    flags &= ~kBuildNoSpeculation;
    if (flags == TF_BUILD_DENSE) return build_dense_csr(c, n, dim, rmin, s, h);  // ablation (dense_build.cu)
    if (flags != TF_BUILD_CELL_LIST && flags != TF_BUILD_CELL_LIST_BINS) {
        bool used = false;
        TF_TRY(build_lattice_csr(c, n, dim, rmin, s, h, &used, speculate));
        if (used) return TF_OK;
        if (flags == TF_BUILD_LATTICE) {
            set_error("tf_build_filter_ex: TF_BUILD_LATTICE but the centroids are not a verified cube lattice");
            return TF_ERR_INVALID;
        }
    }
    h->info.path = TF_PATH_CELL_LIST;
    DeviceInfo di;
    TF_TRY(device_info(&di));
    const int threads = 256;
    const unsigned grid_n = (unsigned)std::min<int64_t>((n + threads - 1) / threads, (int64_t)di.sms * 16);

    NvtxRange r_all("tf_build");
    // a2 bounding box
    NvtxRange r_bbox("tf_build/a2 bbox");
    DevBuf<double> part, bbd;
    TF_TRY(part.alloc((size_t)grid_n * 7, s, "bbox partials"));
    TF_TRY(bbd.alloc(8, s, "bbox"));
    k_bbox_partial<<<grid_n, threads, 0, s>>>(c, n, dim, part.p);
    TF_LAUNCH_CHECK();
    k_bbox_final<<<1, 256, 0, s>>>(part.p, (int)grid_n, bbd.p);
    TF_LAUNCH_CHECK();
    double bb[7];
    TF_CUDA_TRY(cudaMemcpyAsync(bb, bbd.p, 7 * sizeof(double), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    build_trace().mark("bbox+sync", s);
    if (bb[6] != 0.0) {
        set_error("tf_build_filter: non-finite centroid coordinate (NaN or Inf)");
        return TF_ERR_INVALID;
    }
    Grid g;
    TF_TRY(make_grid(bb, n, dim, rmin, &g));
    h->info.bin_side = g.s;
    for (int d = 0; d < 3; ++d) h->info.bins[d] = g.nb[d];
    h->info.nbins = g.nbins;

    // a3 keys
    NvtxRange r_keys("tf_build/a3-a4 keys, radix sort, cell start");
    DevBuf<uint32_t> k0, v0, k1, v1;
    TF_TRY(k0.alloc(n, s, "keys"));
    TF_TRY(v0.alloc(n, s, "ids"));
    TF_TRY(k1.alloc(n, s, "keys (alt)"));
    TF_TRY(v1.alloc(n, s, "ids (alt)"));
    k_keys<<<grid_n, threads, 0, s>>>(c, n, g, k0.p, v0.p);
    TF_LAUNCH_CHECK();

    // a4 radix sort + cell start + sorted SoA
    uint32_t *ks = nullptr, *vs = nullptr;
    int passes = 0;
    build_trace().mark("keys", s);
    TF_TRY(radix_sort_pairs(k0.p, v0.p, k1.p, v1.p, n, ceil_log2(g.nbins), s, &ks, &vs, &passes));
    build_trace().mark("radix", s);
    h->info.radix_passes = passes;
    DevBuf<int32_t> cs;
    TF_TRY(cs.alloc(g.nbins + 1, s, "cell start"));
    k_cellstart<<<(unsigned)std::min<int64_t>((n + threads) / threads, (int64_t)di.sms * 16), threads, 0, s>>>(
        ks, n, g.nbins, cs.p);
    TF_LAUNCH_CHECK();
    // sorted copies of the centroids: the group kernels read whole points (AoS); the per-bin kernels
    // read SoA, which is only written when they run (asked for, or as the fallback below)
    DevBuf<double> sxyz;
    bool legacy = (flags == TF_BUILD_CELL_LIST_BINS);
    if (const char *e = getenv("TOPOFILT_CL")) legacy = legacy || !strcmp(e, "bins");  // benchmarks
    DevBuf<double4> aos;
    if (legacy) TF_TRY(sxyz.alloc((size_t)dim * n, s, "sorted centroids"));
    else TF_TRY(aos.alloc(n, s, "sorted centroids (AoS)"));
    k_gather_sorted<<<grid_n, threads, 0, s>>>(c, n, dim, vs, legacy ? sxyz.p : nullptr, legacy ? nullptr : aos.p);
    TF_LAUNCH_CHECK();
    SortedPts P;
    P.a = aos.p;
    P.x = P.y = P.z = nullptr;
    P.id = reinterpret_cast<const int32_t *>(vs);
    P.cs = cs.p;
    const uint32_t *ks_keys = ks;  // sorted bin keys (the warp fill decodes each query's bin)

    // a5-a7 by query groups (cl_build.cu) unless the per-bin kernels are asked for or a group's
    // neighbourhood union exceeds the group kernels' shared-memory capacity
    if (!legacy) {
        bool done = false;
        TF_TRY(build_cell_list_groups(P, ks_keys, g, n, s, h, &done));
        if (done) return TF_OK;
        // fallback (a union beyond the group kernels' capacity): the per-bin kernels need the SoA copy
        TF_TRY(sxyz.alloc((size_t)dim * n, s, "sorted centroids"));
        k_gather_sorted<<<grid_n, threads, 0, s>>>(c, n, dim, vs, sxyz.p, nullptr);
        TF_LAUNCH_CHECK();
    }
    P.x = sxyz.p;
    P.y = sxyz.p + n;
    P.z = (dim == 3) ? sxyz.p + 2 * n : sxyz.p + n;

    // largest neighbourhood -> shared-memory capacity of the count / fill passes
    DevBuf<int32_t> counts, stats;
    build_trace().mark("cellstart+gather", s);
    TF_TRY(counts.alloc(n, s, "row counts"));
    TF_TRY(stats.alloc(4, s, "build stats"));
    TF_CUDA_TRY(cudaMemsetAsync(stats.p, 0, 4 * sizeof(int32_t), s));
    {
        const unsigned blocks = (unsigned)std::min<int64_t>((g.nbins + 255) / 256, (int64_t)di.sms * 8);
        if (dim == 3) k_binstats<3><<<blocks, 256, 0, s>>>(cs.p, g, stats.p);
        else k_binstats<2><<<blocks, 256, 0, s>>>(cs.p, g, stats.p);
        TF_LAUNCH_CHECK();
    }
    int32_t hstats[4];
    TF_CUDA_TRY(cudaMemcpyAsync(hstats, stats.p, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    const int maxC = hstats[0];
    h->info.max_candidates = maxC;
    const int hard_cap = 3072;  // fill staging <= ~110 KB of shared memory
    const int cap = (std::max(1, std::min(maxC, hard_cap)) + 63) & ~63;  // multiple of 64 (packed sweeps)
    // warps per count / fill block follow the mean queries per bin (n / bins): a block serves one bin,
    // so sparse bins want small blocks (config 4, 6.2 per bin: 1 warp, count -12% / fill -8%
    // vs 2; config 3, 8 per bin: 2 warps; config 5, 20 per bin: 4 warps)
    const double qpb = (double)n / (double)g.nbins;
    const bool wide = qpb >= 12.0;
    const int bw = wide ? 4 : (qpb >= 7.0 ? 2 : 1);

    // a5 count
    build_trace().mark("binstats+sync", s);
    NvtxRange r_count("tf_build/a5 count + a6 scan");
    int cw = bw;  // warps per count block
    if (const char *e = getenv("TOPOFILT_COUNT_WARPS")) cw = atoi(e);  // tuning knob (benchmarks only)
    if (dim == 3) TF_TRY(cw >= 4 ? (launch_count<3, 4>(P, g, cap, counts.p, stats.p + 3, s))
                         : cw >= 2 ? (launch_count<3, 2>(P, g, cap, counts.p, stats.p + 3, s)) : (launch_count<3, 1>(P, g, cap, counts.p, stats.p + 3, s)));
    else TF_TRY(cw >= 4 ? (launch_count<2, 4>(P, g, cap, counts.p, stats.p + 3, s))
                : cw >= 2 ? (launch_count<2, 2>(P, g, cap, counts.p, stats.p + 3, s)) : (launch_count<2, 1>(P, g, cap, counts.p, stats.p + 3, s)));

    // a6 row pointers + nnz readback
    build_trace().mark("count", s);
    TF_TRY(dalloc(&h->rowptr, n + 3, s, "rowptr (+2 padding for 16-byte bulk copies)"));
    TF_TRY(exclusive_scan_i32_i64(counts.p, h->rowptr, n, s));
    int64_t nnz = 0;
    int32_t maxrow = 0;  // longest row (count pass), for the apply plan's window size
    TF_CUDA_TRY(cudaMemcpyAsync(&nnz, h->rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaMemcpyAsync(&maxrow, stats.p + 3, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    if (nnz < n || nnz < 0) {
        set_error("internal: nnz %lld < n %lld", (long long)nnz, (long long)n);
        return TF_ERR_CUDA;
    }
    h->nnz = nnz;
    h->max_row_hint = maxrow;

    // a7 fill
    build_trace().mark("scan+sync", s);
    NvtxRange r_fill("tf_build/a7 fill");
    TF_TRY(dalloc(&h->cols, nnz + 4, s, "cols (nnz int32, +4 padding for 16-byte bulk copies)"));
    TF_TRY(dalloc(&h->vals, nnz + 4, s, "vals (nnz fp64, +4 padding)"));
    TF_TRY(dalloc(&h->hs, n, s, "Hs"));
    DevBuf<int32_t> large_rows;
    build_trace().mark("alloc_csr", s);
    // a7 kernel: the block-per-bin fill. TOPOFILT_FILL=warp selects the warp-per-query fill for
    // rows up to 128 entries (measured slower: config 4 fill 1.08 vs 0.77 ms, config 3 1.24 vs
    // 1.05 ms); both are parity-tested (tests/test_gpu_fuzz.py)
    int fill_kind = 0;
    if (const char *e = getenv("TOPOFILT_FILL")) {
        if (!strcmp(e, "block")) fill_kind = 0;
        else if (!strcmp(e, "warp") && maxrow <= 128) fill_kind = 1;
    }
    if (fill_kind == 1) {
        const int ks = std::max(1, (maxrow + 31) / 32);
        if (dim == 3) {
            if (ks == 1) TF_TRY((launch_fill_warp<3, 1>(P, ks_keys, g, n, h, di.sms, stats.p, s)));
            else if (ks == 2) TF_TRY((launch_fill_warp<3, 2>(P, ks_keys, g, n, h, di.sms, stats.p, s)));
            else if (ks == 3) TF_TRY((launch_fill_warp<3, 3>(P, ks_keys, g, n, h, di.sms, stats.p, s)));
            else TF_TRY((launch_fill_warp<3, 4>(P, ks_keys, g, n, h, di.sms, stats.p, s)));
        } else {
            if (ks == 1) TF_TRY((launch_fill_warp<2, 1>(P, ks_keys, g, n, h, di.sms, stats.p, s)));
            else if (ks == 2) TF_TRY((launch_fill_warp<2, 2>(P, ks_keys, g, n, h, di.sms, stats.p, s)));
            else if (ks == 3) TF_TRY((launch_fill_warp<2, 3>(P, ks_keys, g, n, h, di.sms, stats.p, s)));
            else TF_TRY((launch_fill_warp<2, 4>(P, ks_keys, g, n, h, di.sms, stats.p, s)));
        }
    }
    if (fill_kind == 0 && maxC > cap) TF_TRY(large_rows.alloc(n, s, "large-neighbourhood rows"));
    int fw = bw;  // warps per fill block (queries of one bin in parallel)
    if (const char *e = getenv("TOPOFILT_FILL_WARPS")) fw = atoi(e);  // tuning knob (benchmarks only)
    if (fill_kind == 1) {
        // done above
    } else if (dim == 3) {
        if (fw >= 8) TF_TRY((launch_fill<3, 8>(P, g, h, cap, large_rows.p, stats.p, s)));
        else if (fw >= 4) TF_TRY((launch_fill<3, 4>(P, g, h, cap, large_rows.p, stats.p, s)));
        else if (fw >= 2) TF_TRY((launch_fill<3, 2>(P, g, h, cap, large_rows.p, stats.p, s)));
        else TF_TRY((launch_fill<3, 1>(P, g, h, cap, large_rows.p, stats.p, s)));
    } else {
        if (fw >= 8) TF_TRY((launch_fill<2, 8>(P, g, h, cap, large_rows.p, stats.p, s)));
        else if (fw >= 4) TF_TRY((launch_fill<2, 4>(P, g, h, cap, large_rows.p, stats.p, s)));
        else if (fw >= 2) TF_TRY((launch_fill<2, 2>(P, g, h, cap, large_rows.p, stats.p, s)));
        else TF_TRY((launch_fill<2, 1>(P, g, h, cap, large_rows.p, stats.p, s)));
    }
    build_trace().mark("fill", s);
    if (fill_kind == 0 && maxC > cap) {
        const int scap = 8192;
        const size_t smem = (size_t)scap * (sizeof(double) + sizeof(int32_t));
        TF_TRY(allow_dynamic_smem(k_rowsort, smem));
        k_rowsort<<<(unsigned)di.sms * 2, kSortThreads, smem, s>>>(large_rows.p, stats.p, h->rowptr, h->cols,
                                                                    h->vals, scap);
        TF_LAUNCH_CHECK();
    }
    // stats[1] = rows that took the large-neighbourhood path; stats[2] = count/fill disagreement
    // flag (always-on invariant: every row's fill writes exactly its counted length)
    int32_t tail[2] = {0, 0};
    TF_CUDA_TRY(cudaMemcpyAsync(tail, stats.p + 1, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    build_trace().mark("rowsort+stats+sync", s);
    h->info.large_rows = tail[0];
    if (tail[1] != 0) {
        set_error("internal: fill pass disagreed with the count pass (row lengths)");
        return TF_ERR_CUDA;
    }
    return TF_OK;
}

}  // namespace tf
