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
//   a5 k_count      warp per query bin: exact fp64 pair test, ballot/popc -> row lengths
//   a6 scan (scan.cu) -> rowptr; nnz read back (the one data-dependent host sync)
//   a7 k_fill       block per query bin: the 3^dim candidate bins are staged in shared
//                   memory IN ASCENDING ID ORDER (merge-rank of the per-bin sorted runs),
//                   so ballot compaction emits every row's columns already ascending;
//                   weights fp64 with Hs fused. Neighbourhoods larger than the shared
//                   memory capacity take a global-memory path plus k_rowsort.
//
// Exactness (R2-R4): the pair test and weight use the caller's centroid bytes,
// d2 = (dx*dx + dy*dy) + dz*dz with __dmul_rn/__dadd_rn (never contracted to FMA),
// w = max(0, rmin - __dsqrt_rn(d2)). This is the oracle's expression, so the CSR
// structure and weights are bit-identical to it.
#include <math.h>
#include <stdio.h>

#include <algorithm>

#include "tf_internal.cuh"

namespace tf {
namespace {

template <int DIM>
__device__ __forceinline__ double pair_d2(double ax, double ay, double az, double bx, double by,
                                          double bz) {
    const double dx = __dsub_rn(ax, bx);
    const double dy = __dsub_rn(ay, by);
    double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    if (DIM == 3) {
        const double dz = __dsub_rn(az, bz);
        d2 = __dadd_rn(d2, __dmul_rn(dz, dz));
    }
    return d2;
}

__device__ __forceinline__ double weight_of(double rmin, double d2) {
    double w = __dsub_rn(rmin, __dsqrt_rn(d2));
    return w < 0.0 ? 0.0 : w;
}

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

__global__ void k_bbox_final(const double *__restrict__ part, int nparts, double *__restrict__ out) {
    if (threadIdx.x != 0) return;
    double r[7] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY, 0.0};
    for (int b = 0; b < nparts; ++b) {
        for (int d = 0; d < 3; ++d) r[d] = fmin(r[d], part[b * 7 + d]), r[3 + d] = fmax(r[3 + d], part[b * 7 + 3 + d]);
        r[6] = fmax(r[6], part[b * 7 + 6]);
    }
    for (int k = 0; k < 7; ++k) out[k] = r[k];
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
                                                       double *__restrict__ sxyz) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = ids[p];
        for (int d = 0; d < dim; ++d) sxyz[d * n + p] = c[i * dim + d];
    }
}

// ------------------------------------------------------------------ neighbourhood helpers
struct SortedPts {
    const double *x, *y, *z;  // SoA, sorted by (bin key, id)
    const int32_t *id;
    const int32_t *cs;        // cell start [nbins+1]
};

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

// ------------------------------------------------------------------ a5: count pass
// One warp per query bin. For each query in the bin, lanes sweep the 3^(dim-1)
// contiguous x-triple ranges 32 candidates at a time; the exact fp64 test feeds a
// warp ballot and popc accumulates the row length. Also records the largest
// neighbourhood (for sizing the fill pass's shared memory).
template <int DIM>
__global__ void __launch_bounds__(256) k_count(SortedPts P, Grid g, int32_t *__restrict__ counts,
                                               int32_t *__restrict__ stats) {
    const int lane = threadIdx.x & 31;
    const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= g.nbins) return;
    const int q0 = P.cs[b], q1 = P.cs[b + 1];
    if (q0 == q1) return;
    int bx, by, bz;
    decode_bin(b, g, bx, by, bz);
    constexpr int NR = (DIM == 3) ? 9 : 3;
    int rs = 0, re = 0;
    if (lane < NR) xtriple_range<DIM>(lane, bx, by, bz, g, P.cs, rs, re);
    int total = re - rs;
    for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    if (lane == 0) atomicMax(&stats[0], total);
    const double r2 = g.r2;
    for (int q = q0; q < q1; ++q) {
        const double qx = P.x[q], qy = P.y[q], qz = (DIM == 3) ? P.z[q] : 0.0;
        int cnt = 0;
#pragma unroll 1
        for (int r = 0; r < NR; ++r) {
            const int s = __shfl_sync(0xffffffffu, rs, r), e = __shfl_sync(0xffffffffu, re, r);
            for (int base = s; base < e; base += 32) {
                const int p = base + lane;
                bool ok = false;
                if (p < e) {
                    const double d2 = pair_d2<DIM>(qx, qy, qz, P.x[p], P.y[p], (DIM == 3) ? P.z[p] : 0.0);
                    ok = d2 < r2;
                }
                cnt += __popc(__ballot_sync(0xffffffffu, ok));
            }
        }
        if (lane == 0) counts[P.id[q]] = cnt;
    }
}

// ------------------------------------------------------------------ a7: fill pass
template <int DIM>
struct FillSmem {
    double *x, *y, *z;
    int32_t *id;
    __device__ FillSmem(unsigned char *raw, int cap) {
        x = reinterpret_cast<double *>(raw);
        y = x + cap;
        z = (DIM == 3) ? y + cap : y;
        id = reinterpret_cast<int32_t *>((DIM == 3 ? z : y) + cap);
    }
};

__device__ __forceinline__ int lower_bound_i32(const int32_t *a, int len, int32_t v) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Block per query bin, WARPS warps. See file header.
template <int DIM, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_fill(SortedPts P, Grid g, const int64_t *__restrict__ rowptr,
                                                     int32_t *__restrict__ cols, double *__restrict__ vals,
                                                     double *__restrict__ hs, int cap,
                                                     int32_t *__restrict__ large_rows,
                                                     int32_t *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int NRUN = (DIM == 3) ? 27 : 9;
    __shared__ int run_s[NRUN], run_l[NRUN], run_p[NRUN + 1], run_min[NRUN], run_max[NRUN];
    const int64_t b = blockIdx.x;
    const int q0 = P.cs[b], q1 = P.cs[b + 1];
    if (q0 == q1) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int bx, by, bz;
    decode_bin(b, g, bx, by, bz);
    if (tid < NRUN) {
        const int dz = (DIM == 3) ? (tid / 9 - 1) : 0;
        const int dy = (tid / 3) % 3 - 1;
        const int dx = tid % 3 - 1;
        const int xx = bx + dx, yy = by + dy, zz = bz + dz;
        int s = 0, l = 0;
        if (xx >= 0 && xx < g.nb[0] && yy >= 0 && yy < g.nb[1] && zz >= 0 && zz < g.nb[2]) {
            const int64_t key = ((int64_t)zz * g.nb[1] + yy) * g.nb[0] + xx;
            s = P.cs[key];
            l = P.cs[key + 1] - s;
        }
        run_s[tid] = s;
        run_l[tid] = l;
        run_min[tid] = l ? P.id[s] : 0;
        run_max[tid] = l ? P.id[s + l - 1] : -1;
    }
    __syncthreads();
    if (tid == 0) {
        int acc = 0;
        for (int r = 0; r < NRUN; ++r) run_p[r] = acc, acc += run_l[r];
        run_p[NRUN] = acc;
    }
    __syncthreads();
    const int C = run_p[NRUN];
    const double r2 = g.r2, rmin = g.rmin;
    const uint32_t lt_mask = (1u << lane) - 1u;

    if (C <= cap) {
        // ---- stage the candidates in ascending id order (merge-rank of the sorted runs)
        FillSmem<DIM> S(smem_raw, cap);
        for (int t = tid; t < C; t += WARPS * 32) {
            int r = 0;
            while (t >= run_p[r + 1]) ++r;
            const int off = t - run_p[r];
            const int p = run_s[r] + off;
            const int32_t id = P.id[p];
            int rank = off;
#pragma unroll 1
            for (int r2i = 0; r2i < NRUN; ++r2i) {
                if (r2i == r) continue;
                const int l = run_l[r2i];
                if (l == 0 || id < run_min[r2i]) continue;
                if (id > run_max[r2i]) {
                    rank += l;
                    continue;
                }
                rank += lower_bound_i32(P.id + run_s[r2i], l, id);
            }
            S.id[rank] = id;
            S.x[rank] = P.x[p];
            S.y[rank] = P.y[p];
            if (DIM == 3) S.z[rank] = P.z[p];
        }
        __syncthreads();
        // ---- one warp per query; candidates in ascending id -> columns ascending
        for (int q = q0 + warp; q < q1; q += WARPS) {
            const double qx = P.x[q], qy = P.y[q], qz = (DIM == 3) ? P.z[q] : 0.0;
            const int32_t qid = P.id[q];
            const int64_t base = rowptr[qid];
            int pos = 0;
            double hsum = 0.0;
            for (int t0 = 0; t0 < C; t0 += 32) {
                const int t = t0 + lane;
                bool ok = false;
                double d2 = 0.0;
                if (t < C) {
                    d2 = pair_d2<DIM>(qx, qy, qz, S.x[t], S.y[t], (DIM == 3) ? S.z[t] : 0.0);
                    ok = d2 < r2;
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                if (ok) {
                    const double w = weight_of(rmin, d2);
                    const int64_t k = base + pos + __popc(bal & lt_mask);
                    cols[k] = S.id[t];
                    vals[k] = w;
                    hsum += w;
                }
                pos += __popc(bal);
            }
            for (int o = 16; o > 0; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
            if (lane == 0) hs[qid] = hsum;
        }
    } else {
        // ---- large neighbourhood: candidates from global memory in run order; the rows
        // are recorded and sorted afterwards by k_rowsort.
        for (int q = q0 + warp; q < q1; q += WARPS) {
            const double qx = P.x[q], qy = P.y[q], qz = (DIM == 3) ? P.z[q] : 0.0;
            const int32_t qid = P.id[q];
            const int64_t base = rowptr[qid];
            int pos = 0;
            double hsum = 0.0;
            for (int r = 0; r < NRUN; ++r) {
                const int s = run_s[r], e = run_s[r] + run_l[r];
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
                        const int64_t k = base + pos + __popc(bal & lt_mask);
                        cols[k] = P.id[p];
                        vals[k] = w;
                        hsum += w;
                    }
                    pos += __popc(bal);
                }
            }
            for (int o = 16; o > 0; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
            if (lane == 0) {
                hs[qid] = hsum;
                const int slot = atomicAdd(&stats[1], 1);
                large_rows[slot] = qid;
            }
        }
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

tf_status make_grid(const double *bb, int64_t n, int dim, double rmin, Grid *g) {
    g->dim = dim;
    g->rmin = rmin;
    g->r2 = rmin * rmin;  // the oracle's r2 = rmin*rmin (one rounding, same on both sides)
    double lo[3] = {0, 0, 0}, span[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) lo[d] = bb[d], span[d] = bb[3 + d] - bb[d];
    // Bin side s >= rmin*(1+1e-6): a pair within rmin lies in adjacent bins (R5).
    double s = rmin * (1.0 + 1e-6);
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
    return TF_OK;
}

template <int DIM, int WARPS>
tf_status launch_fill(const SortedPts &P, const Grid &g, tf_filter_s *h, int cap, int32_t *large_rows,
                      int32_t *stats, cudaStream_t s) {
    const size_t smem = (size_t)cap * (DIM * sizeof(double) + sizeof(int32_t));
    if (smem > 48 * 1024)
        TF_CUDA_TRY(cudaFuncSetAttribute(k_fill<DIM, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
    k_fill<DIM, WARPS><<<(unsigned)g.nbins, WARPS * 32, smem, s>>>(P, g, h->rowptr, h->cols, h->vals, h->hs,
                                                                   cap, large_rows, stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

}  // namespace

tf_status build_filter_device(const double *c, int64_t n, int dim, double rmin, cudaStream_t s,
                              tf_filter_s *h) {
    DeviceInfo di;
    TF_TRY(device_info(&di));
    const int threads = 256;
    const unsigned grid_n = (unsigned)std::min<int64_t>((n + threads - 1) / threads, (int64_t)di.sms * 16);

    // a2 bounding box
    DevBuf<double> part, bbd;
    TF_TRY(part.alloc((size_t)grid_n * 7, s, "bbox partials"));
    TF_TRY(bbd.alloc(8, s, "bbox"));
    k_bbox_partial<<<grid_n, threads, 0, s>>>(c, n, dim, part.p);
    TF_LAUNCH_CHECK();
    k_bbox_final<<<1, 32, 0, s>>>(part.p, (int)grid_n, bbd.p);
    TF_LAUNCH_CHECK();
    double bb[7];
    TF_CUDA_TRY(cudaMemcpyAsync(bb, bbd.p, 7 * sizeof(double), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
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
    TF_TRY(radix_sort_pairs(k0.p, v0.p, k1.p, v1.p, n, ceil_log2(g.nbins), s, &ks, &vs, &passes));
    h->info.radix_passes = passes;
    DevBuf<int32_t> cs;
    TF_TRY(cs.alloc(g.nbins + 1, s, "cell start"));
    k_cellstart<<<(unsigned)std::min<int64_t>((n + threads) / threads, (int64_t)di.sms * 16), threads, 0, s>>>(
        ks, n, g.nbins, cs.p);
    TF_LAUNCH_CHECK();
    DevBuf<double> sxyz;
    TF_TRY(sxyz.alloc((size_t)dim * n, s, "sorted centroids"));
    k_gather_sorted<<<grid_n, threads, 0, s>>>(c, n, dim, vs, sxyz.p);
    TF_LAUNCH_CHECK();
    SortedPts P;
    P.x = sxyz.p;
    P.y = sxyz.p + n;
    P.z = (dim == 3) ? sxyz.p + 2 * n : sxyz.p + n;
    P.id = reinterpret_cast<const int32_t *>(vs);
    P.cs = cs.p;

    // a5 count
    DevBuf<int32_t> counts, stats;
    TF_TRY(counts.alloc(n, s, "row counts"));
    TF_TRY(stats.alloc(4, s, "build stats"));
    TF_CUDA_TRY(cudaMemsetAsync(stats.p, 0, 4 * sizeof(int32_t), s));
    {
        const int64_t warps = g.nbins;
        const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
        if (dim == 3) k_count<3><<<blocks, 256, 0, s>>>(P, g, counts.p, stats.p);
        else k_count<2><<<blocks, 256, 0, s>>>(P, g, counts.p, stats.p);
        TF_LAUNCH_CHECK();
    }

    // a6 row pointers + nnz readback
    TF_TRY(dalloc(&h->rowptr, n + 1, s, "rowptr"));
    TF_TRY(exclusive_scan_i32_i64(counts.p, h->rowptr, n, s));
    int64_t nnz = 0;
    int32_t hstats[4];
    TF_CUDA_TRY(cudaMemcpyAsync(&nnz, h->rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaMemcpyAsync(hstats, stats.p, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    if (nnz < n || nnz < 0) {
        set_error("internal: nnz %lld < n %lld", (long long)nnz, (long long)n);
        return TF_ERR_CUDA;
    }
    h->nnz = nnz;
    const int maxC = hstats[0];
    h->info.max_candidates = maxC;

    // a7 fill
    TF_TRY(dalloc(&h->cols, nnz, s, "cols (nnz int32)"));
    TF_TRY(dalloc(&h->vals, nnz, s, "vals (nnz fp64)"));
    TF_TRY(dalloc(&h->hs, n, s, "Hs"));
    const int hard_cap = (dim == 3) ? 4096 : 5632;  // <= ~112 KB of shared memory
    const int cap = std::max(1, std::min(maxC, hard_cap));
    DevBuf<int32_t> large_rows;
    if (maxC > cap) TF_TRY(large_rows.alloc(n, s, "large-neighbourhood rows"));
    const double avg = (double)n / (double)g.nbins;
    if (dim == 3) {
        if (avg >= 12) TF_TRY((launch_fill<3, 4>(P, g, h, cap, large_rows.p, stats.p, s)));
        else TF_TRY((launch_fill<3, 2>(P, g, h, cap, large_rows.p, stats.p, s)));
    } else {
        if (avg >= 12) TF_TRY((launch_fill<2, 4>(P, g, h, cap, large_rows.p, stats.p, s)));
        else TF_TRY((launch_fill<2, 2>(P, g, h, cap, large_rows.p, stats.p, s)));
    }
    if (maxC > cap) {
        const int scap = 8192;
        const size_t smem = (size_t)scap * (sizeof(double) + sizeof(int32_t));
        TF_CUDA_TRY(cudaFuncSetAttribute(k_rowsort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_rowsort<<<(unsigned)di.sms * 2, kSortThreads, smem, s>>>(large_rows.p, stats.p, h->rowptr, h->cols,
                                                                    h->vals, scap);
        TF_LAUNCH_CHECK();
        int32_t nl = 0;
        TF_CUDA_TRY(cudaMemcpyAsync(&nl, stats.p + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        TF_CUDA_TRY(cudaStreamSynchronize(s));
        h->info.large_rows = nl;
    }
    return TF_OK;
}

}  // namespace tf
