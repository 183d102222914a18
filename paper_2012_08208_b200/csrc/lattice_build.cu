// lattice_build.cu -- structured-mesh path of tf_build_filter (SURVEY.md 8(a) rows a5-a7 on
// lattice-ordered centroids).
//
// The paper's meshes are FEniCS BoxMesh / RectangleMesh lattices: cell
// T*((k*ny + j)*nx + i) + t of a cube grid with T cells per cube (1 quad/hex, 2 triangles,
// 6 Kuhn tetrahedra), so cell centroids repeat with the cube. For such inputs the cell list is
// not needed to find the neighbours of a row: they lie in the cubes within a reach R of the
// row's cube, and, ordered by (dz, dy, dx, target type), their indices ASCEND -- the CSR column
// order W is stored in (PAPER.md:442-445 builds the same W densely).
//
// Detection (host, from a prefix of the centroids + a few probes) proposes a model
//   L(cell) = c[t] + (i*hx, j*hy, k*hz)        (c[t] = the actual centroid of cell t of cube 0)
// and k_lat_verify measures, over EVERY centroid, dev = max |c - L| per component, finiteness,
// and whether the input is "exact" (every coordinate on a dyadic grid 2^-e, |coordinate| <=
// 2^50 quanta, and exactly equal to L). The rows are then built from a per-type table of (column delta,
// cube offset[, weight]) entries, sorted by column delta:
//   * tested mode (any dev): the table lists every (offset, type) whose nominal distance is below
//     rmin + 2*sqrt(dim)*dev + slack -- a superset of every true neighbour (R21) -- and
//     each candidate is decided by the exact fp64 pair test on the caller's bytes (pair_d2, the
//     oracle's expression), with the weight w = max(0, rmin - sqrt(d2)) as in the cell-list path;
//   * exact mode (dev = 0 on a dyadic grid): every pair difference c_j - c_i is exact in fp64 and
//     equals the entry's nominal vector, so d2 (the same uncontracted expression on the same
//     operands) -- hence the test and the weight -- depends only on the table entry (DESIGN.md
//     R22); the host evaluates the oracle's expression once per entry and rows are written from
//     the table with no per-pair arithmetic (interior rows: a copy of the table; Hs = the table's
//     sum in ascending column order).
// Rows whose cube lies within R of the grid boundary drop the out-of-grid entries (ballot
// compaction keeps the order). Count -> scan -> nnz readback -> fill, like the cell-list path.
// Anything that does not verify falls back to the cell list (tf_build_filter), or is rejected
// with TF_ERR_INVALID when the caller requires this path (TF_BUILD_LATTICE).
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <vector>

#include "tf_internal.cuh"

namespace tf {
namespace {

constexpr int kLatMaxTable = 4096;  // table entries over all types (shared memory: 16 B tested, 48 B exact)
constexpr int kLatMaxReach = 100;   // cube offsets are stored as int8 (+128 bias)
#ifndef TF_LAT_RPL
#define TF_LAT_RPL 2
#endif
constexpr int kLatRPL = TF_LAT_RPL;  // exact fill: rows per warp task = 32 * kLatRPL (1: 2.46, 2: 2.41 ms at config 5)

struct LatEntry {
    int32_t delta;  // column - row (the same for every row of this type)
    int32_t off;    // (dx + 128) | (dy + 128) << 8 | (dz + 128) << 16
    double w;       // exact mode: the weight; tested mode: unused
};

struct LatDev {
    int64_t n;
    int T, nx, ny, nz;
    int R[3];
    int C[3];  // boundary classes per axis (exact mode)
    int kstart[kMaxTypes + 1];
    double hs_full[kMaxTypes];  // exact mode: interior row sums (ascending-column order)
    double rmin, r2;
};

// Exact mode boundary classes: class cid = ((cz*C1 + cy)*C0 + cx)*T + t owns the list
// [off[cid], off[cid+1]) of (delta, w) -- its type table restricted to in-grid offsets -- and hs[cid].
// Class cid = ((cz*C1 + cy)*C0 + cx)*T + t keeps the entries of its type table whose offsets stay
// in the grid: bit e of mask[cid*W + e/32] (W = words per class); pre[cid*W + w] = set bits in
// words < w; len[cid] = set bits; hs[cid] = their weights summed in ascending column order.
struct LatClasses {
    const uint32_t *mask;
    const int32_t *pre;
    const int32_t *len;
    const double *hs;
    int ncls, W;
    static size_t smem_bytes(int ncls, int W) {
        return (size_t)ncls * (sizeof(double) + sizeof(int32_t)) + (size_t)ncls * W * 2 * sizeof(uint32_t);
    }
};

struct LatVerifyArgs {
    int dim, T;
    uint32_t nx, ny;
    double c0[kMaxTypes][3];
    double h[3];
    double q;  // 2^e of the dyadic grid candidate (0: none)
};

// ------------------------------------------------------------------ device kernels
__global__ void k_lat_probe(const double *__restrict__ c, int dim, const int64_t *__restrict__ idx, int m,
                            double *__restrict__ out) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x)
        for (int d = 0; d < dim; ++d) out[p * 3 + d] = c[idx[p] * dim + d];
}

// out[0] = max deviation (bits of a non-negative double), out[1] = flags (1: non-finite, 2: not
// exact: some coordinate is off the 2^-e grid, beyond 2^50 quanta, or not exactly the model value).
// Block-stride over the rows of cubes (j, k known per row); threads over the row's T*nx points.
template <int DIM>
__global__ void __launch_bounds__(256) k_lat_verify(const double *__restrict__ c, int64_t n, LatVerifyArgs a,
                                                    unsigned long long *__restrict__ out) {
    __shared__ double sc0[kMaxTypes][3];
    __shared__ double shh[3];
    if (threadIdx.x < kMaxTypes * 3) sc0[threadIdx.x / 3][threadIdx.x % 3] = a.c0[threadIdx.x / 3][threadIdx.x % 3];
    if (threadIdx.x < 3) shh[threadIdx.x] = a.h[threadIdx.x];
    __syncthreads();
    double dev = 0.0;
    unsigned flags = 0;
    const int64_t rowlen = (int64_t)a.T * a.nx;  // points per row of cubes
    const int64_t nrows = n / rowlen;
    const int64_t elems = rowlen * DIM;
    for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
        const uint32_t jj = (uint32_t)(row % a.ny), kk = (uint32_t)(row / a.ny);
        const double *cr = c + row * elems;
        // thread per point (one 32-bit division per point, the DIM coordinates from one 8*DIM-byte
        // span: a warp's loads cover the row's bytes contiguously)
        // kVU points per thread per step, all loads issued first (one point per step was
        // latency-bound: 137 us for 288 MB at config 5)
        constexpr int kVU = 4;
        for (uint32_t p0 = threadIdx.x; p0 < (uint32_t)rowlen; p0 += kVU * blockDim.x) {
            double cv[kVU][DIM];
#pragma unroll
            for (int u = 0; u < kVU; ++u) {
                const uint32_t p = p0 + u * blockDim.x;
#pragma unroll
                for (int d = 0; d < DIM; ++d) cv[u][d] = (p < (uint32_t)rowlen) ? cr[(int64_t)p * DIM + d] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kVU; ++u) {
                const uint32_t p = p0 + u * blockDim.x;
                if (p >= (uint32_t)rowlen) break;
                const uint32_t i = p / (uint32_t)a.T, t = p - i * (uint32_t)a.T;
#pragma unroll
                for (int d = 0; d < DIM; ++d) {
                    const uint32_t idx = (d == 0) ? i : (d == 1 ? jj : kk);
                    const double v = cv[u][d];
                    const double L = fma((double)idx, shh[d], sc0[t][d]);
                    if (!isfinite(v)) flags |= 1u;
                    dev = fmax(dev, fabs(v - L));
                    const double s = v * a.q;
                    if (!(a.q > 0.0 && s == rint(s) && fabs(s) <= 1125899906842624.0 && v == L)) flags |= 2u;
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
        flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out[0], (unsigned long long)__double_as_longlong(dev));
        if (flags) atomicOr(&out[1], (unsigned long long)flags);
    }
}

template <int DIM>
__device__ __forceinline__ bool lat_interior(const LatDev &m, int i, int j, int k) {
    return i >= m.R[0] && i < m.nx - m.R[0] && j >= m.R[1] && j < m.ny - m.R[1] &&
           (DIM == 2 || (k >= m.R[2] && k < m.nz - m.R[2]));
}

template <int DIM>
__device__ __forceinline__ bool lat_in_grid(const LatDev &m, int off, int i, int j, int k) {
    const int dx = (off & 255) - 128, dy = ((off >> 8) & 255) - 128, dz = ((off >> 16) & 255) - 128;
    return (unsigned)(i + dx) < (unsigned)m.nx && (unsigned)(j + dy) < (unsigned)m.ny &&
           (DIM == 2 || (unsigned)(k + dz) < (unsigned)m.nz);
}

// Boundary classes (exact mode): per axis, c = p for p < R, 2R - (n-1-p) for p > n-1-R, else R
// (c = p when n < 2R+1): rows of one class and type keep the same table entries in the grid.
__device__ __forceinline__ int lat_axis_class(int p, int n, int R) {
    return (n < 2 * R + 1) ? p : (p < R ? p : (p > n - 1 - R ? 2 * R - (n - 1 - p) : R));
}
template <int DIM>
__device__ __forceinline__ int lat_class_id(const LatDev &m, int t, int i, int j, int k) {
    const int cx = lat_axis_class(i, m.nx, m.R[0]), cy = lat_axis_class(j, m.ny, m.R[1]);
    const int cz = (DIM == 3) ? lat_axis_class(k, m.nz, m.R[2]) : 0;
    return ((cz * m.C[1] + cy) * m.C[0] + cx) * m.T + t;
}

// Exact mode row lengths: thread per row, the length of its class list.
template <int DIM>
__global__ void __launch_bounds__(256) k_lat_count_exact(LatDev m, LatClasses cls, int32_t *__restrict__ counts) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m.n; r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t u = (uint32_t)r;
        const int t = (int)(u % (uint32_t)m.T);
        const uint32_t cube = u / (uint32_t)m.T;
        const int i = (int)(cube % (uint32_t)m.nx);
        const uint32_t rr = cube / (uint32_t)m.nx;
        const int j = (int)(rr % (uint32_t)m.ny), k = (int)(rr / (uint32_t)m.ny);
        const int cid = lat_class_id<DIM>(m, t, i, j, k);
        TF_DCHECK(cid >= 0 && cid < cls.ncls);
        counts[r] = cls.len[cid];
    }
}

// Exact mode row pointers in closed form (speculative build): the row length depends on the row's
// boundary class only, so the prefix sum over rows in lattice order splits per axis into a prefix
// over the classes before the row's position plus (interior positions before it) x (the interior
// class's total): rowptr = Z(k) + Y(j | cz) + X(i | cy, cz) + T(t | cx, cy, cz), all from a few
// host-built int64 tables -- no count pass, no scan.
struct LatRowptrTabs {
    const int64_t *tp;   // [ncls] entries of the cube's types before t
    const int64_t *px;   // [C2*C1][C0+1] prefix over x classes of the cube totals
    const int64_t *sxr;  // [C2*C1] cube total of the interior x class
    const int64_t *py;   // [C2][C1+1] prefix over y classes of the x-line totals
    const int64_t *syr;  // [C2] x-line total of the interior y class
    const int64_t *pz;   // [C2+1] prefix over z classes of the plane totals
    int64_t szr;         // plane total of the interior z class
    int64_t total;       // nnz
};
__device__ __forceinline__ int64_t lat_axis_prefix(int p, int n, int R, const int64_t *P, int64_t SR) {
    if (n < 2 * R + 1) return P[p];
    const int c = lat_axis_class(p, n, R);
    return (c <= R) ? P[c] + (int64_t)max(0, p - R) * SR : P[c] + (int64_t)(n - 2 * R - 1) * SR;
}
template <int DIM>
__global__ void __launch_bounds__(256) k_lat_rowptr_exact(LatDev m, LatRowptrTabs tb, int64_t *__restrict__ rowptr) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= m.n; r += (int64_t)gridDim.x * blockDim.x) {
        if (r == m.n) {
            rowptr[r] = tb.total;
            continue;
        }
        const uint32_t u = (uint32_t)r;
        const int t = (int)(u % (uint32_t)m.T);
        const uint32_t cube = u / (uint32_t)m.T;
        const int i = (int)(cube % (uint32_t)m.nx);
        const uint32_t rr = cube / (uint32_t)m.nx;
        const int j = (int)(rr % (uint32_t)m.ny), k = (int)(rr / (uint32_t)m.ny);
        const int cy = lat_axis_class(j, m.ny, m.R[1]);
        const int cz = (DIM == 3) ? lat_axis_class(k, m.nz, m.R[2]) : 0;
        const int yz = cz * m.C[1] + cy;
        int64_t v = tb.tp[lat_class_id<DIM>(m, t, i, j, k)];
        v += lat_axis_prefix(i, m.nx, m.R[0], tb.px + (size_t)yz * (m.C[0] + 1), tb.sxr[yz]);
        v += lat_axis_prefix(j, m.ny, m.R[1], tb.py + (size_t)cz * (m.C[1] + 1), tb.syr[cz]);
        if (DIM == 3) v += lat_axis_prefix(k, m.nz, m.R[2], tb.pz, tb.szr);
        rowptr[r] = v;
    }
}

// Cycle table of the exact fill, four shifted copies so that any four consecutive entries are one
// 16-byte-aligned vector read: copy s holds entries s, s+1, ... of the extended cycle sequence
// (types 0..T-1 concatenated, S entries; entries S.. repeat the start one cycle later, coloff + T).
struct LatCycle {
    const int32_t *col;  // [4][SP] coloff = type + delta
    const double *w;     // [4][SP]
    int S, SP;
    int LW;  // > 0: the weight cycle is replicated to LW entries (two copies, shifted by 0 and 1) in
             // shared memory and interior chunks store their weights with TMA bulk copies
    int LP;  // entries per bulk copy (even); LW >= S + LP, so a copy may start at any cycle position
};

__device__ __forceinline__ void lat_decode(int64_t r, const LatDev &m, int &t, int &i, int &j, int &k) {
    const uint32_t u = (uint32_t)r;
    t = (int)(u % (uint32_t)m.T);
    const uint32_t cube = u / (uint32_t)m.T;
    i = (int)(cube % (uint32_t)m.nx);
    const uint32_t rr = cube / (uint32_t)m.nx;
    j = (int)(rr % (uint32_t)m.ny);
    k = (int)(rr / (uint32_t)m.ny);
}

// Exact-mode fill: warp per 32 consecutive rows.
//  * all rows interior (one row of cubes, no wrap): the chunk's output is a window of the periodic
//    cycle sequence (position P = entry P mod S of cycle P div S; column = first row of that cycle
//    + coloff), written flat over [rowptr[r0], rowptr[r0+nr]): four 16-byte-aligned entries per
//    lane and step (one int4 of columns, two double2 of weights, read as three LDS.128 from the
//    shifted copies); the < 4-entry head and tail are scalar;
//  * otherwise per row: a copy of its boundary class list (interior rows: the type table).
// Hs = the class's (type's) sum in ascending column order -- the oracle's order.
#ifndef TF_LAT_MINB
#define TF_LAT_MINB 1
#endif
template <int DIM>
__global__ void __launch_bounds__(256, TF_LAT_MINB) k_lat_fill_exact(LatDev m, LatCycle cy, LatClasses cls,
                                                        const int64_t *__restrict__ rowptr,
                                                        int32_t *__restrict__ cols, double *__restrict__ vals,
                                                        double *__restrict__ hs, int32_t *__restrict__ flag) {
    extern __shared__ __align__(16) unsigned char lat_smem[];
    double *wrep = reinterpret_cast<double *>(lat_smem);                  // [2][LW] (LW even)
    int32_t *scol = reinterpret_cast<int32_t *>(wrep + 2 * cy.LW);        // [4][SP]
    double *sw = reinterpret_cast<double *>(scol + 4 * cy.SP);            // [4][SP]
    double *chs = sw + 4 * cy.SP;                                         // [ncls]
    int32_t *clen = reinterpret_cast<int32_t *>(chs + cls.ncls);          // [ncls]
    uint32_t *cmask = reinterpret_cast<uint32_t *>(clen + cls.ncls);      // [ncls*W]
    int32_t *cpre = reinterpret_cast<int32_t *>(cmask + cls.ncls * cls.W);  // [ncls*W]
    __shared__ int skst[kMaxTypes + 1];
    __shared__ double shs[kMaxTypes];
    for (int e = threadIdx.x; e < 4 * cy.SP; e += blockDim.x) scol[e] = cy.col[e], sw[e] = cy.w[e];
    for (int e = threadIdx.x; e < cls.ncls; e += blockDim.x) chs[e] = cls.hs[e], clen[e] = cls.len[e];
    for (int e = threadIdx.x; e < cls.ncls * cls.W; e += blockDim.x) cmask[e] = cls.mask[e], cpre[e] = cls.pre[e];
    for (int e = threadIdx.x; e < 2 * cy.LW; e += blockDim.x) {
        const int x = (e < cy.LW) ? e : e - cy.LW + 1;  // copy 1 starts one entry later
        wrep[e] = cy.w[x % cy.S];
    }
    if (threadIdx.x <= kMaxTypes) skst[threadIdx.x] = m.kstart[threadIdx.x];
    if (threadIdx.x < kMaxTypes) shs[threadIdx.x] = m.hs_full[threadIdx.x];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // wrep -> TMA (async proxy) reads
    __syncthreads();
    const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;
    const int S = cy.S, SP = cy.SP;
    const bool bulk = cy.LW > 0;
    bool issued = false;
    const int lane = threadIdx.x & 31;
    // Tasks: CH consecutive rows (CH = 32 * RPL); the flat path needs only the chunk's first and
    // end row pointers, the per-row path all of them (RPL per lane)
    constexpr int RPL = kLatRPL, CH = 32 * RPL;
    const int64_t ntasks = (m.n + CH - 1) / CH;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t task = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5;
    // row pointers of the chunk (lane l, slot u: rowptr[r0 + 32u + l]; all: rowptr[r0 + nr]),
    // loaded one task ahead so the stores never wait on them
    int64_t rp_lane[RPL], rp_end = 0;
    auto load_rp = [&](int64_t tk, int64_t *pl, int64_t &pe) {
        if (tk < ntasks) {
            const int64_t q0 = tk * CH;
            const int cnt = (int)(m.n - q0 < CH ? m.n - q0 : CH);
#pragma unroll
            for (int u = 0; u < RPL; ++u)
                if (32 * u + lane < cnt) pl[u] = rowptr[q0 + 32 * u + lane];
            pe = rowptr[q0 + cnt];
        }
    };
    load_rp(task, rp_lane, rp_end);
    for (; task < ntasks; task += wstride) {
        const int64_t r0 = task * CH;
        const int nr = (int)(m.n - r0 < CH ? m.n - r0 : CH);
        int64_t cur_lane[RPL];
#pragma unroll
        for (int u = 0; u < RPL; ++u) cur_lane[u] = rp_lane[u];
        const int64_t cur_end = rp_end;
        load_rp(task + wstride, rp_lane, rp_end);
        // row pointer of task row q (warp-uniform q; q == nr: the task's end)
        auto rp = [&](int q) -> int64_t {
            if (q >= nr) return cur_end;
            int64_t v = 0;
#pragma unroll
            for (int u = 0; u < RPL; ++u) {  // (warp-uniform slot selection)
                const int64_t b_u = __shfl_sync(0xffffffffu, cur_lane[u], q & 31);
                if ((q >> 5) == u) v = b_u;
            }
            return v;
        };
        // rows [qa, qb) of the task that lie in one x-line of interior cubes: their entries are a
        // window of the periodic cycle sequence, written flat
        auto flat = [&](int qa, int qb) {
            const int64_t base = rp(qa), end = rp(qb);
            const int64_t rs = r0 + qa;
            const int cnt = qb - qa, t = (int)((uint32_t)rs % (uint32_t)m.T);
            const int64_t rowc = rs - t;  // first row of the segment's first cycle
            const int P0 = skst[t];       // cycle position of the chunk's first entry
            auto scalar_at = [&](int64_t g, bool with_w) {  // head / tail entries (small chunk offsets)
                const int P = P0 + (int)(g - base);
                const int mc = P / S, cc = P - mc * S;
                cols[g] = (int32_t)(rowc + (int64_t)mc * m.T + scol[cc]);
                if (with_w) vals[g] = sw[cc];
            };
            if (bulk) {
                // weights: the window [P0, P0 + total) of the periodic weight sequence, as bulk
                // stores of <= LP entries over its 16-byte-aligned middle, one per lane (source
                // copy chosen per piece so both sides align); a short replica keeps shared memory
                // small enough for two blocks per SM
                const int64_t a0 = base + (base & 1), a1 = end & ~(int64_t)1;
                for (int64_t p0 = a0 + (int64_t)lane * cy.LP; p0 < a1; p0 += 32 * (int64_t)cy.LP) {
                    const int64_t len = (a1 - p0 < cy.LP) ? a1 - p0 : cy.LP;
                    const int Pp = (P0 + (int)(p0 - base)) % S, sh = Pp & 1;
                    TF_DCHECK(Pp - sh + len <= cy.LW && (len & 1) == 0);
                    const uint32_t src = (uint32_t)__cvta_generic_to_shared(wrep + sh * cy.LW + (Pp - sh));
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(vals + p0),
                                 "r"(src), "r"((uint32_t)(len * 8))
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    issued = true;
                }
                if (lane == 1 && (base & 1)) vals[base] = sw[P0 % S];
                if (lane == 2 && (end & 1) && end - 1 >= a0) vals[end - 1] = sw[(P0 + (int)(end - 1 - base)) % S];
                if (lane == 3 && a1 <= a0)
                    for (int64_t g = base; g < end; ++g) vals[g] = sw[(P0 + (int)(g - base)) % S];
            }
            const int64_t g0 = (base + 3) & ~(int64_t)3, g1 = end & ~(int64_t)3;
            TF_DCHECK(end >= base && end - base <= (int64_t)CH * S);
            if (g0 >= g1) {  // no aligned group (tiny tables only)
                for (int64_t g = base + lane; g < end; g += 32) scalar_at(g, !bulk);
            } else {
                if (base + lane < g0) scalar_at(base + lane, !bulk);
                if (g1 + lane < end) scalar_at(g1 + lane, !bulk);
                // per 128-entry group G: lane l writes columns G+4l..G+4l+3 (one int4) and, without
                // the bulk path, weights G+2l, G+2l+1 and G+64+2l, G+64+2l+1 (two double2): every
                // store instruction covers 512 contiguous bytes, whole sectors. Cycle positions
                // stay < S + 195: no division.
                const int PG = P0 + (int)(g0 - base);
                int mc = 0, cc = PG + 4 * lane, ca = PG + 2 * lane, cb = PG + 64 + 2 * lane;
                while (cc >= S) cc -= S, ++mc;
                while (ca >= S) ca -= S;
                while (cb >= S) cb -= S;
                // four groups per iteration: all shared-memory reads first, then all stores (ILP);
                // table positions stay inside the padded table, so the reads need no predicate
#ifndef TF_LAT_U
#define TF_LAT_U 4
#endif
                constexpr int U = TF_LAT_U;
                if (bulk) {
                    for (int64_t G = g0; G < g1; G += 128 * U) {
                        int4 co[U];
                        int32_t rb[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int shc = cc & 3;
                            TF_DCHECK(cc >= 0 && cc < S && cc - shc + 4 <= SP);
                            co[u] = *reinterpret_cast<const int4 *>(scol + shc * SP + (cc - shc));
                            rb[u] = (int32_t)(rowc + (int64_t)mc * m.T);
                            cc += 128;
                            while (cc >= S) cc -= S, ++mc;
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int64_t Gu = G + 128 * u;
                            if (Gu + 4 * lane < g1)
                                *reinterpret_cast<int4 *>(cols + Gu + 4 * lane) =
                                    make_int4(rb[u] + co[u].x, rb[u] + co[u].y, rb[u] + co[u].z, rb[u] + co[u].w);
                        }
                    }
                } else {
                    for (int64_t G = g0; G < g1; G += 128 * U) {
                        int4 co[U];
                        double2 wa[U], wb[U];
                        int32_t rb[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int shc = cc & 3, sha = ca & 1, shb = cb & 1;
                            co[u] = *reinterpret_cast<const int4 *>(scol + shc * SP + (cc - shc));
                            wa[u] = *reinterpret_cast<const double2 *>(sw + sha * SP + (ca - sha));
                            wb[u] = *reinterpret_cast<const double2 *>(sw + shb * SP + (cb - shb));
                            rb[u] = (int32_t)(rowc + (int64_t)mc * m.T);
                            cc += 128, ca += 128, cb += 128;
                            while (cc >= S) cc -= S, ++mc;
                            while (ca >= S) ca -= S;
                            while (cb >= S) cb -= S;
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int64_t Gu = G + 128 * u;
                            if (Gu + 4 * lane < g1)
                                *reinterpret_cast<int4 *>(cols + Gu + 4 * lane) =
                                    make_int4(rb[u] + co[u].x, rb[u] + co[u].y, rb[u] + co[u].z, rb[u] + co[u].w);
                            if (Gu + 2 * lane < g1) *reinterpret_cast<double2 *>(vals + Gu + 2 * lane) = wa[u];
                            if (Gu + 64 + 2 * lane < g1)
                                *reinterpret_cast<double2 *>(vals + Gu + 64 + 2 * lane) = wb[u];
                        }
                    }
                }
            }
            int expect = 0;
            for (int q = lane; q < cnt; q += 32) {
                const int tl = (t + q) % m.T;
                hs[rs + q] = shs[tl];
                expect += skst[tl + 1] - skst[tl];
            }
            for (int o = 16; o > 0; o >>= 1) expect += __shfl_xor_sync(0xffffffffu, expect, o);
            if (lane == 0 && expect != end - base) atomicOr(flag, 1);
        };
        // rows [qa, qb) one by one: a copy of each row's boundary class
        auto rows = [&](int qa, int qb) {
            if (qa >= qb) return;
            int t, i, j, k;
            lat_decode(r0 + qa, m, t, i, j, k);
            int64_t end = rp(qa);
            for (int q = qa; q < qb; ++q) {
                const int64_t r = r0 + q;
                const int64_t base = end;
                end = rp(q + 1);
                // a copy of the row's class: the type table entries flagged in its mask, scattered to
                // their ranks (ascending order kept), all from shared memory
                const int cid = lat_class_id<DIM>(m, t, i, j, k);
                TF_DCHECK(cid >= 0 && cid < cls.ncls);
                const int ks = skst[t], K = skst[t + 1] - ks;
                TF_DCHECK(ks >= 0 && ks + K <= S && (K + 31) / 32 <= cls.W);
                int32_t *cq = cols + base;
                double *vq = vals + base;
                const int64_t rowc = r - t;
                for (int e0 = 0; e0 < K; e0 += 32) {
                    const int wd = cid * cls.W + (e0 >> 5);
                    const uint32_t word = cmask[wd];
                    if (e0 + lane < K && ((word >> lane) & 1u)) {
                        const int pos = cpre[wd] + __popc(word & lt);
                        TF_DCHECK(pos >= 0 && base + pos < end);
                        cq[pos] = (int32_t)(rowc + scol[ks + e0 + lane]);
                        vq[pos] = sw[ks + e0 + lane];
                    }
                }
                if (lane == 0) {
                    hs[r] = chs[cid];
                    if (base + clen[cid] != end) atomicOr(flag, 1);
                }
                if (++t == m.T) {
                    t = 0;
                    if (++i == m.nx) {
                        i = 0;
                        if (++j == m.ny) j = 0, ++k;
                    }
                }
            }
        };
        // split the task at x-line ends; inside an x-line of interior (j, k), the rows of interior
        // cubes go flat and only the rows of the R end cubes go row by row (whole tasks went row by
        // row before whenever any of their rows was a boundary row)
        for (int q = 0; q < nr;) {
            const int64_t r = r0 + q;
            int t, i, j, k;
            lat_decode(r, m, t, i, j, k);
            const int64_t lb = r - t - (int64_t)i * m.T;  // first row of the x-line
            const int qe = (int)((lb + (int64_t)m.nx * m.T - r0 < nr) ? lb + (int64_t)m.nx * m.T - r0 : nr);
            if (m.nx > 2 * m.R[0] && lat_interior<DIM>(m, m.R[0], j, k)) {
                const int64_t fa = lb + (int64_t)m.R[0] * m.T - r0, fb = lb + (int64_t)(m.nx - m.R[0]) * m.T - r0;
                const int qa = (int)(fa > q ? fa : q), qb = (int)(fb < qe ? fb : qe);
                if (qa < qb) {
                    rows(q, qa);
                    flat(qa, qb);
                    rows(qb, qe);
                } else {
                    rows(q, qe);
                }
            } else {
                rows(q, qe);
            }
            q = qe;
        }
    }
    // bulk stores complete (and their shared-memory source stays allocated) before the CTA exits
    if (issued) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Tested mode: warp per 32 consecutive rows (decoded once, then stepped), lanes over the row's
// table candidates, each decided by the exact fp64 pair test on the caller's coordinates.
// FILL = false: row lengths; FILL = true: cols / vals / Hs at rowptr.
template <int DIM, bool FILL>
__global__ void __launch_bounds__(256) k_lat_rows(const double *__restrict__ c, LatDev m,
                                                  const LatEntry *__restrict__ gtab, int ntab,
                                                  const int64_t *__restrict__ rowptr, int32_t *__restrict__ counts,
                                                  int32_t *__restrict__ cols, double *__restrict__ vals,
                                                  double *__restrict__ hs, int32_t *__restrict__ flag) {
    extern __shared__ __align__(16) unsigned char lat_smem[];
    LatEntry *stab = reinterpret_cast<LatEntry *>(lat_smem);
    __shared__ int skst[kMaxTypes + 1];
    for (int e = threadIdx.x; e < ntab; e += blockDim.x) stab[e] = gtab[e];
    if (threadIdx.x <= kMaxTypes) skst[threadIdx.x] = m.kstart[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t ntasks = (m.n + 31) / 32;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t task = (((int64_t)blockIdx.x * blockDim.x) + threadIdx.x) >> 5; task < ntasks; task += wstride) {
        const int64_t r0 = task * 32;
        const int nr = (int)(m.n - r0 < 32 ? m.n - r0 : 32);
        int t, i, j, k;
        lat_decode(r0, m, t, i, j, k);
        int64_t rp_lane = 0, rp_end = 0;
        if (FILL) {
            if (lane < nr) rp_lane = rowptr[r0 + lane];
            rp_end = rowptr[r0 + nr];
        }
        for (int q = 0; q < nr; ++q) {
            const int64_t r = r0 + q;
            int64_t base = 0, end = 0;
            if (FILL) {
                base = __shfl_sync(0xffffffffu, rp_lane, q);
                const int64_t nxt = __shfl_sync(0xffffffffu, rp_lane, (q + 1) & 31);
                end = (q + 1 < nr) ? nxt : rp_end;
            }
            const int ks = skst[t], K = skst[t + 1] - ks;
            const bool interior = lat_interior<DIM>(m, i, j, k);
            const double qx = c[r * DIM], qy = c[r * DIM + 1], qz = (DIM == 3) ? c[r * DIM + 2] : 0.0;
            int wpos = 0;
            double hsum = 0.0;
            for (int e0 = 0; e0 < K; e0 += 32) {
                const int e = e0 + lane;
                bool ok = e < K;
                LatEntry en{0, 0, 0.0};
                if (ok) en = stab[ks + e];
                if (ok && !interior) ok = lat_in_grid<DIM>(m, en.off, i, j, k);
                double d2 = 0.0;
                if (ok) {
                    const int64_t p = r + en.delta;
                    TF_DCHECK(p >= 0 && p < m.n);
                    d2 = pair_d2<DIM>(qx, qy, qz, c[p * DIM], c[p * DIM + 1], (DIM == 3) ? c[p * DIM + 2] : 0.0);
                    ok = d2 < m.r2;
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                if (FILL && ok) {
                    const double w = weight_of(m.rmin, d2);
                    const int64_t kk = base + wpos + __popc(bal & lt);
                    TF_DCHECK(kk < end);
                    cols[kk] = (int32_t)(r + en.delta);
                    vals[kk] = w;
                    hsum += w;
                }
                wpos += __popc(bal);
            }
            if (FILL) {
                for (int o = 16; o > 0; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
                if (lane == 0) {
                    hs[r] = hsum;
                    if (base + wpos != end) atomicOr(flag, 1);
                }
            } else if (lane == 0) {
                counts[r] = wpos;
            }
            if (++t == m.T) {
                t = 0;
                if (++i == m.nx) {
                    i = 0;
                    if (++j == m.ny) j = 0, ++k;
                }
            }
        }
    }
}

// ------------------------------------------------------------------ host: detection
struct LatModel {
    int dim = 0, T = 0;
    int64_t nx = 0, ny = 1, nz = 1;
    double c0[kMaxTypes][3] = {};
    double h[3] = {0, 0, 0};
};

// Row structure from a prefix A[P x dim]: T cells per cube, nx cubes per row with spacing hx
// along x, and the step D from row 0 to row 1 (along y, or along z when ny = 1). Returns 1 on
// success, 0 if the input is not lattice-ordered, -1 if the prefix is too short to decide.
int detect_rows(const double *A, int64_t P, int64_t n, int dim, LatModel *M, double D[3]) {
    auto at = [&](int64_t id, int d) { return A[id * dim + d]; };
    bool need_more = false;
    for (int T = 1; T <= kMaxTypes; ++T) {
        if (2 * T > n) break;
        if (2 * T > P) {
            need_more = true;
            break;
        }
        const double hx = at(T, 0) - at(0, 0);
        if (!(hx > 0.0) || !isfinite(hx)) continue;
        const double tol = 1e-6 * hx;
        // cube m of row 0 matches cube 0 shifted by m*hx along x
        auto cube_on_row = [&](int64_t base, const double *shift) {
            for (int t = 0; t < T; ++t)
                for (int d = 0; d < dim; ++d)
                    if (!(fabs(at(base + t, d) - (at(t, d) + shift[d])) <= tol)) return false;
            return true;
        };
        int64_t m = 1;
        const int64_t lim = std::min(P, n);
        bool ok = true;
        for (; T * (m + 1) <= lim; ++m) {
            const double sh[3] = {(double)m * hx, 0.0, 0.0};
            if (!cube_on_row(T * m, sh)) break;
        }
        int64_t nx;
        if (T * m == n) {
            nx = m;  // a single row
        } else if (T * (m + 1) > lim) {
            if (lim < n) need_more = true;  // prefix exhausted inside row 0
            continue;
        } else {
            nx = m;
        }
        if (nx < 2 || n % (T * nx) != 0) continue;
        D[0] = D[1] = D[2] = 0.0;
        if (n > T * nx) {
            if (2 * T * nx > P) {
                need_more = true;
                continue;
            }
            for (int d = 0; d < dim; ++d) D[d] = at(T * nx, d) - at(0, d);
            const bool along_y = D[1] > 0.0 && fabs(D[0]) <= tol && (dim == 2 || fabs(D[2]) <= tol);
            const bool along_z = dim == 3 && D[2] > 0.0 && fabs(D[0]) <= tol && fabs(D[1]) <= tol;
            if (!along_y && !along_z) continue;
            if (along_y) D[0] = D[2] = 0.0;
            else D[0] = D[1] = 0.0;
            for (int64_t i = 0; i < nx && ok; ++i) {
                const double sh[3] = {(double)i * hx + D[0], D[1], D[2]};
                ok = cube_on_row(T * nx + T * i, sh);
            }
            if (!ok) continue;
        }
        M->dim = dim;
        M->T = T;
        M->nx = nx;
        M->h[0] = hx;
        for (int t = 0; t < T; ++t)
            for (int d = 0; d < dim; ++d) M->c0[t][d] = at(t, d);
        return 1;
    }
    return need_more ? -1 : 0;
}

// Where detection reads centroids from: a prefix and a few gathered points (3 doubles each).
struct PointSource {
    virtual tf_status prefix(int64_t P, std::vector<double> &A) = 0;
    // the prefix and the last point (3 doubles, zero-padded) in one round trip
    virtual tf_status prefix_last(int64_t P, int64_t n, std::vector<double> &A, double last[3]) = 0;
    virtual tf_status gather(const std::vector<int64_t> &idx, std::vector<double> &pts) = 0;
    virtual ~PointSource() = default;
};

struct DevicePoints final : PointSource {  // the caller's device array (copies on `s`)
    const double *c;
    int dim;
    cudaStream_t s;
    DevicePoints(const double *c_, int dim_, cudaStream_t s_) : c(c_), dim(dim_), s(s_) {}
    tf_status prefix(int64_t P, std::vector<double> &A) override {
        A.resize((size_t)P * dim);
        TF_CUDA_TRY(cudaMemcpyAsync(A.data(), c, (size_t)P * dim * sizeof(double), cudaMemcpyDeviceToHost, s));
        TF_CUDA_TRY(cudaStreamSynchronize(s));
        return TF_OK;
    }
    tf_status prefix_last(int64_t P, int64_t n, std::vector<double> &A, double last[3]) override {
        A.resize((size_t)P * dim);
        last[0] = last[1] = last[2] = 0.0;
        TF_CUDA_TRY(cudaMemcpyAsync(A.data(), c, (size_t)P * dim * sizeof(double), cudaMemcpyDeviceToHost, s));
        TF_CUDA_TRY(cudaMemcpyAsync(last, c + (n - 1) * dim, (size_t)dim * sizeof(double), cudaMemcpyDeviceToHost, s));
        TF_CUDA_TRY(cudaStreamSynchronize(s));
        return TF_OK;
    }
    tf_status gather(const std::vector<int64_t> &idx, std::vector<double> &pts) override {
        const int m = (int)idx.size();
        pts.assign((size_t)m * 3, 0.0);
        if (m == 0) return TF_OK;
        DevBuf<int64_t> didx;
        DevBuf<double> dout;
        TF_TRY(didx.alloc(m, s, "lattice probes"));
        TF_TRY(dout.alloc((size_t)m * 3, s, "lattice probe points"));
        TF_CUDA_TRY(cudaMemsetAsync(dout.p, 0, (size_t)m * 3 * sizeof(double), s));
        TF_CUDA_TRY(cudaMemcpyAsync(didx.p, idx.data(), m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        k_lat_probe<<<(m + 127) / 128, 128, 0, s>>>(c, dim, didx.p, m, dout.p);
        TF_LAUNCH_CHECK();
        TF_CUDA_TRY(cudaMemcpyAsync(pts.data(), dout.p, (size_t)m * 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
        TF_CUDA_TRY(cudaStreamSynchronize(s));
        return TF_OK;
    }
};

struct HostPoints final : PointSource {  // a host array (tf_lattice_detect_host: CPU-testable)
    const double *c;
    int dim;
    HostPoints(const double *c_, int dim_) : c(c_), dim(dim_) {}
    tf_status prefix(int64_t P, std::vector<double> &A) override {
        A.assign(c, c + (size_t)P * dim);
        return TF_OK;
    }
    tf_status prefix_last(int64_t P, int64_t n, std::vector<double> &A, double last[3]) override {
        A.assign(c, c + (size_t)P * dim);
        last[0] = last[1] = last[2] = 0.0;
        for (int d = 0; d < dim; ++d) last[d] = c[(n - 1) * dim + d];
        return TF_OK;
    }
    tf_status gather(const std::vector<int64_t> &idx, std::vector<double> &pts) override {
        pts.assign(idx.size() * 3, 0.0);
        for (size_t p = 0; p < idx.size(); ++p)
            for (int d = 0; d < dim; ++d) pts[p * 3 + d] = c[idx[p] * dim + d];
        return TF_OK;
    }
};

// Full model (T, nx, ny, nz, spacings) or found = false.
tf_status detect_model(PointSource &src, int64_t n, int dim, LatModel *M, bool *found) {
    *found = false;
    std::vector<double> A;
    double D[3];
    int64_t P = std::min<int64_t>(n, 4096);
    double last[3];
    TF_TRY(src.prefix_last(P, n, A, last));
    int st = detect_rows(A.data(), P, n, dim, M, D);
    if (st < 0 && P < n) {
        P = std::min<int64_t>(n, 1 << 16);
        TF_TRY(src.prefix(P, A));
        st = detect_rows(A.data(), P, n, dim, M, D);
    }
    if (st <= 0) return TF_OK;
    const int64_t rowlen = (int64_t)M->T * M->nx;
    const int64_t rows = n / rowlen;  // ny*nz
    const double tol = 1e-6 * M->h[0];
    if (rows == 1) {
        M->ny = M->nz = 1;
        M->h[1] = M->h[2] = M->h[0];
    } else if (dim == 2) {
        M->ny = rows;
        M->nz = 1;
        M->h[1] = D[1];
        M->h[2] = M->h[0];
    } else if (D[2] > 0.0) {  // 3D with one row per layer
        M->ny = 1;
        M->nz = rows;
        M->h[1] = M->h[0];
        M->h[2] = D[2];
    } else {
        // 3D: the last point is c0[T-1] + ((nx-1) hx, (ny-1) hy, (nz-1) hz) on a complete lattice:
        // it gives ny (and with it nz, hz) without a second round trip; anything inconsistent falls
        // back to probing rows T*nx*d for the divisors d of rows (one more round trip)
        M->h[1] = D[1];
        {
            const double *cl = M->c0[M->T - 1];
            const double fy = (last[1] - cl[1]) / D[1];
            const int64_t ny = (int64_t)llround(fy) + 1;
            const double ex = last[0] - (cl[0] + (double)(M->nx - 1) * M->h[0]);
            if (fabs(fy - (double)(ny - 1)) <= 1e-6 * std::max(1.0, fabs(fy)) && fabs(ex) <= tol && ny >= 1 &&
                ny <= rows && rows % ny == 0) {
                const int64_t nz = rows / ny;
                const double hz = (nz > 1) ? (last[2] - cl[2]) / (double)(nz - 1) : M->h[0];
                if (nz == 1 || hz > 0.0) {
                    M->ny = ny;
                    M->nz = nz;
                    M->h[2] = hz;
                    if (M->nx * M->ny * M->nz * M->T == n) *found = true;
                    return TF_OK;  // the device verification checks every point against this model
                }
            }
        }
        std::vector<int64_t> divs;
        for (int64_t d = 2; d * d <= rows; ++d)
            if (rows % d == 0) {
                divs.push_back(d);
                if (d * d != rows) divs.push_back(rows / d);
            }
        std::sort(divs.begin(), divs.end());
        if (divs.size() > 512) return TF_OK;
        int64_t ny = rows;
        double hz = M->h[0];
        std::vector<int64_t> idx(divs.size());
        for (size_t p = 0; p < divs.size(); ++p) idx[p] = rowlen * divs[p];
        std::vector<double> pts;
        TF_TRY(src.gather(idx, pts));
        for (size_t p = 0; p < divs.size(); ++p) {
            const double *q = &pts[p * 3];
            const double dx = q[0] - M->c0[0][0], dy = q[1] - M->c0[0][1], dz = q[2] - M->c0[0][2];
            const bool on_y = fabs(dx) <= tol && fabs(dy - (double)divs[p] * D[1]) <= tol && fabs(dz) <= tol;
            if (on_y) continue;
            if (!(fabs(dx) <= tol && fabs(dy) <= tol && dz > 0.0)) return TF_OK;  // not a lattice
            ny = divs[p];
            hz = dz;
            break;
        }
        M->ny = ny;
        M->nz = rows / ny;
        M->h[2] = hz;
    }
    if (M->nx * M->ny * M->nz * M->T != n) return TF_OK;
    *found = true;
    return TF_OK;
}

// Smallest e <= 60 with v * 2^e an integer for every v (0 if none): the dyadic grid candidate.
double dyadic_scale(const std::vector<double> &vs) {
    for (int e = 0; e <= 60; ++e) {
        const double q = ldexp(1.0, e);
        bool ok = true;
        for (double v : vs) {
            const double s = v * q;
            if (!(s == rint(s)) || fabs(s) > 9007199254740992.0) {
                ok = false;
                break;
            }
        }
        if (ok) return q;
    }
    return 0.0;
}

}  // namespace

tf_status build_lattice_csr(const double *c, int64_t n, int dim, double rmin, cudaStream_t s, tf_filter_s *h,
                            bool *used, bool speculate) {
    *used = false;
    if (n < 4) return TF_OK;
    NvtxRange r_det("tf_build/lattice detect + verify");
    LatModel M;
    bool found = false;
    DevicePoints src(c, dim, s);
    TF_TRY(detect_model(src, n, dim, &M, &found));
    if (!found) return TF_OK;
    build_trace().mark("lattice detect", s);

    // ---- verify every centroid against the model
    LatVerifyArgs va{};
    va.dim = dim;
    va.T = M.T;
    va.nx = (uint32_t)M.nx;
    va.ny = (uint32_t)M.ny;
    for (int t = 0; t < M.T; ++t)
        for (int d = 0; d < 3; ++d) va.c0[t][d] = (d < dim) ? M.c0[t][d] : 0.0;
    for (int d = 0; d < 3; ++d) va.h[d] = M.h[d];
    {
        std::vector<double> vs;
        for (int t = 0; t < M.T; ++t)
            for (int d = 0; d < dim; ++d) vs.push_back(M.c0[t][d]);
        for (int d = 0; d < dim; ++d) vs.push_back(M.h[d]);
        va.q = dyadic_scale(vs);
    }
    DeviceInfo di;
    TF_TRY(device_info(&di));
    DevBuf<unsigned long long> vout;
    TF_TRY(vout.alloc(2, s, "lattice verify"));
    TF_CUDA_TRY(cudaMemsetAsync(vout.p, 0, 2 * sizeof(unsigned long long), s));
    const unsigned vgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(M.ny * M.nz, (int64_t)di.sms * 8));
    if (dim == 3) k_lat_verify<3><<<vgrid, 256, 0, s>>>(c, n, va, vout.p);
    else k_lat_verify<2><<<vgrid, 256, 0, s>>>(c, n, va, vout.p);
    TF_LAUNCH_CHECK();
    // ---- per-type tables (bounds need the deviation; the exact-mode tables do not, so they are
    // built on the host while the verification pass runs, and discarded if it rules them out)
    const int64_t nd[3] = {M.nx, M.ny, M.nz};
    double cmax = 0.0, spread[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) {
        double lo = M.c0[0][d], hi = M.c0[0][d];
        for (int t = 1; t < M.T; ++t) lo = std::min(lo, M.c0[t][d]), hi = std::max(hi, M.c0[t][d]);
        spread[d] = hi - lo;
        cmax = std::max(cmax, std::max(fabs(lo), fabs(hi)) + (double)nd[d] * M.h[d]);
    }
    // tested mode: a true neighbour's nominal distance is < rmin + 2 sqrt(dim) (dev + rounding of L)
    const double slack = 8.0 * 2.220446049250313e-16 * cmax;
    double margin = 0.0;
    int R[3] = {0, 0, 0}, Rb[3] = {0, 0, 0};  // trimmed reach, enumeration bound
    auto set_bounds = [&](double dv) -> bool {
        margin = 2.0 * sqrt((double)dim) * (dv + slack) + 1e-9 * rmin + slack;
        int64_t span = 1;
        for (int d = 0; d < 3; ++d) Rb[d] = 0;
        for (int d = 0; d < dim; ++d) {
            const double reach = ceil((rmin + margin + spread[d]) / M.h[d]);
            if (!(reach <= (double)kLatMaxReach)) return false;
            Rb[d] = (int)std::min<int64_t>((int64_t)reach, nd[d] - 1);
            span *= 2 * Rb[d] + 1;
        }
        return span * M.T * M.T <= ((int64_t)4 << 20);
    };
    const double r2 = rmin * rmin;
    std::vector<LatEntry> tab;
    LatDev L{};
    L.n = n;
    L.T = M.T;
    L.nx = (int)M.nx;
    L.ny = (int)M.ny;
    L.nz = (int)M.nz;
    L.rmin = rmin;
    L.r2 = r2;
    int maxK = 0;
    // per-type tables sorted by column delta; exact: accepted entries with their weights, tested:
    // candidates. Returns false if over the table capacity.
    auto build_tables = [&](bool ex) -> bool {
        tab.clear();
        maxK = 0;
        for (int sty = 0; sty < M.T; ++sty) {
            L.kstart[sty] = (int)tab.size();
            std::vector<LatEntry> row;
            for (int dz = -Rb[2]; dz <= Rb[2]; ++dz)
                for (int dy = -Rb[1]; dy <= Rb[1]; ++dy)
                    for (int dx = -Rb[0]; dx <= Rb[0]; ++dx)
                        for (int tt = 0; tt < M.T; ++tt) {
                            const int dd[3] = {dx, dy, dz};
                            double v[3] = {0, 0, 0};
                            for (int d = 0; d < dim; ++d) v[d] = (M.c0[tt][d] - M.c0[sty][d]) + (double)dd[d] * M.h[d];
                            // the oracle's expression, never contracted: in exact mode v is exactly the
                            // pair difference, so this is the d2 the oracle computes (R22)
                            volatile double p0 = v[0] * v[0], p1 = v[1] * v[1], p2 = v[2] * v[2];
                            double d2 = p0 + p1;
                            if (dim == 3) d2 = d2 + p2;
                            LatEntry en;
                            en.delta = (int32_t)((int64_t)M.T * (((int64_t)dz * M.ny + dy) * M.nx + dx) + (tt - sty));
                            en.off = (dx + 128) | ((dy + 128) << 8) | ((dz + 128) << 16);
                            en.w = 0.0;
                            if (ex) {
                                if (!(d2 < r2)) continue;
                                double w = (d2 > 0.0) ? rmin - sqrt(d2) : rmin;
                                en.w = w < 0.0 ? 0.0 : w;
                            } else {
                                if (!(sqrt(d2) < rmin + margin)) continue;
                            }
                            row.push_back(en);
                        }
            std::sort(row.begin(), row.end(), [](const LatEntry &x, const LatEntry &y) { return x.delta < y.delta; });
            double hsf = 0.0;
            for (const LatEntry &e : row) hsf += e.w;  // ascending column order
            L.hs_full[sty] = hsf;
            maxK = std::max(maxK, (int)row.size());
            tab.insert(tab.end(), row.begin(), row.end());
            if ((int64_t)tab.size() > kLatMaxTable) return false;
        }
        L.kstart[M.T] = (int)tab.size();
        for (int t = M.T + 1; t <= kMaxTypes; ++t) L.kstart[t] = L.kstart[M.T];
        // the reach that matters is the largest cube offset in the tables (the enumeration bound is
        // conservative): it sets the interior test and the boundary classes
        for (int d = 0; d < 3; ++d) R[d] = 0;
        for (const LatEntry &e : tab) {
            const int dd[3] = {(e.off & 255) - 128, ((e.off >> 8) & 255) - 128, ((e.off >> 16) & 255) - 128};
            for (int d = 0; d < dim; ++d) R[d] = std::max(R[d], std::abs(dd[d]));
        }
        for (int d = 0; d < 3; ++d) L.R[d] = R[d];
        return true;
    };
    // One upload: [tested: the candidate table] or [exact: cycle table (4 shifted copies) +
    // boundary classes]. Exact-mode boundary classes (per axis C_d = min(n_d, 2R_d + 1); see
    // lat_axis_class): each (class, type) list is the type table restricted to the offsets in the
    // grid at a representative position; Hs summed in ascending column order (the oracle's order).
    std::vector<unsigned char> blob;
    std::vector<int32_t> cls_len;  // exact mode: row length of every (boundary class, type)
    size_t o_tab = 0, o_ccol = 0, o_cw = 0, o_mask = 0, o_pre = 0, o_len = 0, o_hs = 0;
    int ntab = 0, SP = 0;
    int64_t ncls = 0;
    int Wc = 0;
    auto make_blob = [&](bool ex) {
        blob.clear();
        ntab = (int)tab.size();
        // One upload: [tested: the candidate table] or [exact: cycle table (4 shifted copies) +
        // boundary classes]. Exact-mode boundary classes (per axis C_d = min(n_d, 2R_d + 1); see
        // lat_axis_class): each (class, type) list is the type table restricted to the offsets in the
        // grid at a representative position; Hs summed in ascending column order (the oracle's order).
        auto put = [&](const void *src, size_t bytes) -> size_t {
            const size_t at = (blob.size() + 15) & ~(size_t)15;
            blob.resize(at + bytes);
            if (bytes) memcpy(blob.data() + at, src, bytes);
            return at;
        };
        SP = (ntab + 3 + 3) & ~3;
        if (!ex) {
            o_tab = put(tab.data(), (size_t)ntab * sizeof(LatEntry));
        } else {
            std::vector<int32_t> ccol((size_t)4 * SP);
            std::vector<double> cw((size_t)4 * SP);
            std::vector<int32_t> seqc(ntab);
            std::vector<double> seqw(ntab);
            for (int sty = 0; sty < M.T; ++sty)
                for (int e = L.kstart[sty]; e < L.kstart[sty + 1]; ++e) seqc[e] = sty + tab[e].delta, seqw[e] = tab[e].w;
            for (int sh = 0; sh < 4; ++sh)
                for (int x = 0; x < SP; ++x) {
                    const int p = x + sh;  // extended cycle position
                    ccol[(size_t)sh * SP + x] = seqc[p % ntab] + M.T * (p / ntab);
                    cw[(size_t)sh * SP + x] = seqw[p % ntab];
                }
            o_ccol = put(ccol.data(), ccol.size() * sizeof(int32_t));
            o_cw = put(cw.data(), cw.size() * sizeof(double));
            auto rep = [&](int cl, int d) -> int64_t {  // a position of class cl on axis d
                if (nd[d] < 2 * R[d] + 1 || cl <= R[d]) return cl;
                return nd[d] - 1 - (2 * R[d] - cl);
            };
            std::vector<uint32_t> c_mask((size_t)ncls * Wc, 0u);
            std::vector<int32_t> c_pre((size_t)ncls * Wc, 0), c_len(ncls, 0);
            std::vector<double> c_hs(ncls, 0.0);
            int64_t cid = 0;
            for (int cz = 0; cz < L.C[2]; ++cz)
                for (int cy = 0; cy < L.C[1]; ++cy)
                    for (int cx = 0; cx < L.C[0]; ++cx) {
                        const int64_t pos[3] = {rep(cx, 0), rep(cy, 1), rep(cz, 2)};
                        for (int sty = 0; sty < M.T; ++sty, ++cid) {
                            double hsum = 0.0;
                            int cnt = 0;
                            for (int e = L.kstart[sty]; e < L.kstart[sty + 1]; ++e) {
                                const int el = e - L.kstart[sty];
                                if (el % 32 == 0) c_pre[cid * Wc + el / 32] = cnt;
                                const int off = tab[e].off;
                                const int dd[3] = {(off & 255) - 128, ((off >> 8) & 255) - 128, ((off >> 16) & 255) - 128};
                                bool in = true;
                                for (int d = 0; d < dim; ++d) in = in && pos[d] + dd[d] >= 0 && pos[d] + dd[d] < nd[d];
                                if (!in) continue;
                                c_mask[cid * Wc + el / 32] |= 1u << (el % 32);
                                hsum += tab[e].w;
                                ++cnt;
                            }
                            c_len[cid] = cnt;
                            c_hs[cid] = hsum;
                        }
                    }
            o_mask = put(c_mask.data(), c_mask.size() * sizeof(uint32_t));
            o_pre = put(c_pre.data(), c_pre.size() * sizeof(int32_t));
            o_len = put(c_len.data(), c_len.size() * sizeof(int32_t));
            cls_len = c_len;
            o_hs = put(c_hs.data(), c_hs.size() * sizeof(double));
        }
    };
    // exact mode needs the cycle table and the boundary-class masks in shared memory; otherwise
    // (large reach) the same input is built in tested mode. The exact tables do not depend on the
    // deviation, so they are built on the host while k_lat_verify runs.
    const auto th0 = std::chrono::steady_clock::now();
    const bool spec_ok = set_bounds(0.0) && build_tables(true);
    bool spec_fits = false;
    if (spec_ok) {
        for (int d = 0; d < 3; ++d) L.C[d] = (d < dim) ? (int)std::min<int64_t>(nd[d], 2 * R[d] + 1) : 1;
        ncls = (int64_t)L.C[0] * L.C[1] * L.C[2] * M.T;
        Wc = std::max(1, (maxK + 31) / 32);
        const int SPx = ((int)tab.size() + 6) & ~3;
        const size_t need = (size_t)4 * SPx * 12 + (ncls <= (1 << 16) ? LatClasses::smem_bytes((int)ncls, Wc) : SIZE_MAX / 2);
        spec_fits = need <= (size_t)160 * 1024;
        if (spec_fits) make_blob(true);
    }
    if (speculate && spec_ok && spec_fits && va.q != 0.0 && (h->lat_check || (h->lat_check = pinned_slot_acquire()))) {
        // ---- speculative exact build: no round trip for the verification or for nnz. nnz follows
        // from the host tables (rows per boundary class x class length); the verification result,
        // the fill's agreement flag and the scanned nnz land in pinned memory by the build's final
        // synchronisation and are checked then (lattice_check_ok); a failed check rebuilds without
        // speculation (tf_build_filter, api.cu)
        int64_t nnz_h = 0;
        auto axis_count = [&](int d, int cl) -> int64_t {
            if (nd[d] < 2 * R[d] + 1) return 1;
            return (cl == R[d]) ? nd[d] - 2 * R[d] : 1;
        };
        int64_t cid = 0;
        for (int cz = 0; cz < L.C[2]; ++cz)
            for (int cy = 0; cy < L.C[1]; ++cy)
                for (int cx = 0; cx < L.C[0]; ++cx) {
                    const int64_t rows = axis_count(0, cx) * (dim >= 2 ? axis_count(1, cy) : 1) *
                                         (dim == 3 ? axis_count(2, cz) : 1);
                    for (int sty = 0; sty < M.T; ++sty, ++cid) nnz_h += rows * (int64_t)cls_len[cid];
                }
        build_trace().mark("lattice tables (speculative)", s);
        DevBuf<unsigned char> dblob;
        TF_TRY(dblob.alloc(blob.size(), s, "lattice tables"));
        TF_CUDA_TRY(cudaMemcpyAsync(dblob.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, s));
        auto at = [&](size_t o) { return dblob.p + o; };
        const int ntab_ = (int)tab.size();
        const int LP = (std::max(1024, ntab_) + 1) & ~1;
        int LW = (ntab_ + LP + 2 + 1) & ~1;
        if ((size_t)2 * LW * sizeof(double) > (size_t)96 * 1024) LW = 0;
        // the replica must fit beside the cycle table and the class masks (found by tools/lattice_soak.py:
        // large tables passed the 160 KB check above and then overflowed the block's shared memory)
        if ((size_t)2 * LW * sizeof(double) + (size_t)4 * SP * (sizeof(int32_t) + sizeof(double)) +
                LatClasses::smem_bytes((int)ncls, Wc) + 4096 > di.smem_optin)
            LW = 0;
#ifdef TF_LAT_NO_BULK
        LW = 0;
#endif
        const LatCycle cyc{reinterpret_cast<const int32_t *>(at(o_ccol)), reinterpret_cast<const double *>(at(o_cw)),
                           ntab_, SP, LW, LP};
        const LatClasses cls{reinterpret_cast<const uint32_t *>(at(o_mask)),
                             reinterpret_cast<const int32_t *>(at(o_pre)), reinterpret_cast<const int32_t *>(at(o_len)),
                             reinterpret_cast<const double *>(at(o_hs)), (int)ncls, Wc};
        DevBuf<int32_t> flag;
        TF_TRY(flag.alloc(1, s, "lattice fill flag"));
        TF_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int32_t), s));
        // row pointers in closed form (k_lat_rowptr_exact): per-axis class prefixes of the class lengths
        DevBuf<int64_t> rpt;
        {
            const int C0 = L.C[0], C1 = L.C[1], C2 = L.C[2], T = M.T;
            auto axis_total = [&](int d, const int64_t *P, int64_t SR) -> int64_t {
                return (nd[d] < 2 * R[d] + 1) ? P[nd[d]] : P[L.C[d]] + (int64_t)(nd[d] - 2 * R[d] - 1) * SR;
            };
            const size_t o_tp = 0, o_px = o_tp + ncls, o_sxr = o_px + (size_t)C2 * C1 * (C0 + 1),
                         o_py = o_sxr + (size_t)C2 * C1, o_syr = o_py + (size_t)C2 * (C1 + 1), o_pz = o_syr + C2,
                         o_end = o_pz + C2 + 1;
            std::vector<int64_t> rt(o_end, 0);
            int64_t szr = 0;
            for (int cz = 0; cz < C2; ++cz) {
                for (int cy = 0; cy < C1; ++cy) {
                    const int yz = cz * C1 + cy;
                    int64_t *px = &rt[o_px + (size_t)yz * (C0 + 1)];
                    for (int cx = 0; cx < C0; ++cx) {
                        int64_t cube = 0;
                        for (int t = 0; t < T; ++t) {
                            const size_t c = ((size_t)yz * C0 + cx) * T + t;
                            rt[o_tp + c] = cube;
                            cube += cls_len[c];
                        }
                        px[cx + 1] = px[cx] + cube;
                        if (cx == R[0]) rt[o_sxr + yz] = cube;
                    }
                    int64_t *py = &rt[o_py + (size_t)cz * (C1 + 1)];
                    const int64_t line = axis_total(0, px, rt[o_sxr + yz]);
                    py[cy + 1] = py[cy] + line;
                    if (cy == R[1]) rt[o_syr + cz] = line;
                }
                const int64_t plane = (dim >= 2) ? axis_total(1, &rt[o_py + (size_t)cz * (C1 + 1)], rt[o_syr + cz])
                                                 : rt[o_py + (size_t)cz * (C1 + 1) + 1];
                rt[o_pz + cz + 1] = rt[o_pz + cz] + plane;
                if (cz == R[2]) szr = plane;
            }
            const int64_t total = (dim == 3) ? axis_total(2, &rt[o_pz], szr) : rt[o_pz + 1];
            if (total != nnz_h) {
                set_error("internal: lattice row-pointer tables disagree with nnz (%lld vs %lld)", (long long)total,
                          (long long)nnz_h);
                return TF_ERR_CUDA;
            }
            TF_TRY(rpt.alloc(o_end, s, "lattice row-pointer tables"));
            TF_CUDA_TRY(cudaMemcpyAsync(rpt.p, rt.data(), o_end * sizeof(int64_t), cudaMemcpyHostToDevice, s));
            TF_TRY(dalloc(&h->rowptr, n + 3, s, "rowptr (+2 padding for 16-byte bulk copies)"));
            const LatRowptrTabs tb{rpt.p + o_tp, rpt.p + o_px, rpt.p + o_sxr, rpt.p + o_py, rpt.p + o_syr,
                                   rpt.p + o_pz, szr, total};
            const unsigned g = (unsigned)std::min<int64_t>((n + 256) / 256, (int64_t)di.sms * 16);
            if (dim == 3) k_lat_rowptr_exact<3><<<g, 256, 0, s>>>(L, tb, h->rowptr);
            else k_lat_rowptr_exact<2><<<g, 256, 0, s>>>(L, tb, h->rowptr);
            TF_LAUNCH_CHECK();
        }
        TF_TRY(dalloc(&h->cols, nnz_h + 4, s, "cols (nnz int32, +4 padding for 16-byte bulk copies)"));
        TF_TRY(dalloc(&h->vals, nnz_h + 4, s, "vals (nnz fp64, +4 padding)"));
        TF_TRY(dalloc(&h->hs, n, s, "Hs"));
        {
            const size_t smem_cyc = (size_t)2 * LW * sizeof(double) + (size_t)4 * SP * (sizeof(int32_t) + sizeof(double)) +
                                    LatClasses::smem_bytes((int)ncls, Wc);
            auto kern = (dim == 3) ? k_lat_fill_exact<3> : k_lat_fill_exact<2>;
            TF_TRY(allow_dynamic_smem(kern, smem_cyc));
            int per_sm = 0;
            TF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem_cyc));
            const int64_t warps_needed = (n + 31) / 32;
            const unsigned grid = (unsigned)std::max<int64_t>(
                1, std::min<int64_t>((int64_t)di.sms * std::max(1, per_sm), (warps_needed + 7) / 8));
            kern<<<grid, 256, smem_cyc, s>>>(L, cyc, cls, h->rowptr, h->cols, h->vals, h->hs, flag.p);
            TF_LAUNCH_CHECK();
        }
        if (!h->lat_check) h->lat_check = pinned_slot_acquire();
        if (!h->lat_check) {
            set_error("internal: no pinned slot for the speculative lattice build");
            return TF_ERR_NOMEM;
        }
        memset(h->lat_check, 0xff, 4 * sizeof(unsigned long long));
        TF_CUDA_TRY(cudaMemcpyAsync(h->lat_check, vout.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        h->lat_check[2] = 0;
        TF_CUDA_TRY(cudaMemcpyAsync(&h->lat_check[2], flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        TF_CUDA_TRY(cudaMemcpyAsync(&h->lat_check[3], h->rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        build_trace().mark("lattice count + scan + fill (speculative)", s);
        h->lat_pending = true;
        h->lat_nnz_host = nnz_h;
        h->nnz = nnz_h;
        h->info.bin_side = 0.0;
        for (int d = 0; d < 3; ++d) h->info.bins[d] = nd[d];
        h->info.nbins = M.nx * M.ny * M.nz;
        h->info.max_candidates = maxK;
        h->max_row_hint = maxK;
        h->info.large_rows = 0;
        h->info.radix_passes = 0;
        h->info.path = TF_PATH_LATTICE_EXACT;
        *used = true;
        return TF_OK;
    }
    unsigned long long vres[2];
    TF_CUDA_TRY(cudaMemcpyAsync(vres, vout.p, sizeof(vres), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    build_trace().mark("lattice verify + tables", s);
    if (vres[1] & 1ull) return TF_OK;  // non-finite: the cell-list path reports it
    double dev;
    memcpy(&dev, &vres[0], sizeof(dev));
    double hmin = M.h[0];
    if (dim >= 2 && M.ny > 1) hmin = std::min(hmin, M.h[1]);
    if (dim == 3 && M.nz > 1) hmin = std::min(hmin, M.h[2]);
    if (!(dev <= 0.05 * hmin)) return TF_OK;
    bool exact = (vres[1] & 2ull) == 0;  // implies dev == 0
    if (exact && !spec_ok) return TF_OK;
    if (exact && !spec_fits) exact = false;
    if (!exact) {
        if (!set_bounds(dev) || !build_tables(false)) return TF_OK;
        ncls = 0;
        Wc = 0;
        make_blob(false);
    }
    const auto th1 = std::chrono::steady_clock::now();
    DevBuf<unsigned char> dblob;
    TF_TRY(dblob.alloc(blob.size(), s, "lattice tables"));
    TF_CUDA_TRY(cudaMemcpyAsync(dblob.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, s));
    if (PhaseTrace::enabled()) {
        const auto th2 = std::chrono::steady_clock::now();
        fprintf(stderr, "[topofilt trace] lattice host: tables %.3f ms, upload %zu B %.3f ms\n",
                std::chrono::duration<double, std::milli>(th1 - th0).count(), blob.size(),
                std::chrono::duration<double, std::milli>(th2 - th1).count());
    }
    auto at = [&](size_t o) { return dblob.p + o; };
    const LatEntry *dtab = reinterpret_cast<const LatEntry *>(at(o_tab));
    // weight-cycle replica for the bulk weight stores: enough for a chunk window starting anywhere
    // in the cycle (two copies, 16 bytes per entry); off if it would crowd shared memory
    // (pieces of LP entries: the replica needs S + LP entries, not a whole chunk's window -- config
    // 5: 25 KB instead of 98 KB, which lets two fill blocks share an SM)
    const int LP = (std::max(1024, (int)ntab) + 1) & ~1;
    int LW = ((int)ntab + LP + 2 + 1) & ~1;
    if (!exact || (size_t)2 * LW * sizeof(double) > (size_t)96 * 1024) LW = 0;
    if (exact && (size_t)2 * LW * sizeof(double) + (size_t)4 * SP * (sizeof(int32_t) + sizeof(double)) +
                         LatClasses::smem_bytes((int)ncls, Wc) + 4096 > di.smem_optin)
        LW = 0;
#ifdef TF_LAT_NO_BULK
    LW = 0;
#endif
    const LatCycle cyc{reinterpret_cast<const int32_t *>(at(o_ccol)), reinterpret_cast<const double *>(at(o_cw)), ntab,
                       SP, LW, LP};
    const LatClasses cls{reinterpret_cast<const uint32_t *>(at(o_mask)), reinterpret_cast<const int32_t *>(at(o_pre)),
                         reinterpret_cast<const int32_t *>(at(o_len)), reinterpret_cast<const double *>(at(o_hs)),
                         (int)ncls, Wc};
    build_trace().mark("lattice table", s);

    // ---- count -> scan -> nnz
    NvtxRange r_rows("tf_build/lattice count + scan + fill");
    DevBuf<int32_t> counts, flag;
    TF_TRY(counts.alloc(n, s, "row counts"));
    TF_TRY(flag.alloc(1, s, "lattice fill flag"));
    TF_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int32_t), s));
    auto grid_for = [&](auto kern, size_t smem, unsigned *grid) -> tf_status {
        TF_TRY(allow_dynamic_smem(kern, smem));
        int per_sm = 0;
        TF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
        const int64_t warps_needed = (n + 31) / 32;
        *grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)di.sms * std::max(1, per_sm),
                                                                 (warps_needed + 7) / 8));
        return TF_OK;
    };
    const size_t smem_tab = (size_t)ntab * sizeof(LatEntry);
    const size_t smem_cyc = (size_t)2 * LW * sizeof(double) + (size_t)4 * SP * (sizeof(int32_t) + sizeof(double)) +
                            LatClasses::smem_bytes((int)ncls, Wc);
    unsigned grid = 0;
    if (exact) {
        const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)di.sms * 16);
        if (dim == 3) k_lat_count_exact<3><<<g, 256, 0, s>>>(L, cls, counts.p);
        else k_lat_count_exact<2><<<g, 256, 0, s>>>(L, cls, counts.p);
        TF_LAUNCH_CHECK();
    } else {
        auto kern = (dim == 3) ? k_lat_rows<3, false> : k_lat_rows<2, false>;
        TF_TRY(grid_for(kern, smem_tab, &grid));
        kern<<<grid, 256, smem_tab, s>>>(c, L, dtab, ntab, nullptr, counts.p, nullptr, nullptr, nullptr, flag.p);
        TF_LAUNCH_CHECK();
    }
    build_trace().mark("lattice count", s);
    TF_TRY(dalloc(&h->rowptr, n + 3, s, "rowptr (+2 padding for 16-byte bulk copies)"));
    TF_TRY(exclusive_scan_i32_i64(counts.p, h->rowptr, n, s));
    int64_t nnz = 0;
    TF_CUDA_TRY(cudaMemcpyAsync(&nnz, h->rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    if (nnz < n) {
        set_error("internal: lattice nnz %lld < n %lld", (long long)nnz, (long long)n);
        return TF_ERR_CUDA;
    }
    h->nnz = nnz;
    build_trace().mark("scan+sync", s);

    // ---- fill
    TF_TRY(dalloc(&h->cols, nnz + 4, s, "cols (nnz int32, +4 padding for 16-byte bulk copies)"));
    TF_TRY(dalloc(&h->vals, nnz + 4, s, "vals (nnz fp64, +4 padding)"));
    TF_TRY(dalloc(&h->hs, n, s, "Hs"));
    build_trace().mark("alloc_csr", s);
    if (exact) {
        auto kern = (dim == 3) ? k_lat_fill_exact<3> : k_lat_fill_exact<2>;
        TF_TRY(grid_for(kern, smem_cyc, &grid));
        kern<<<grid, 256, smem_cyc, s>>>(L, cyc, cls, h->rowptr, h->cols, h->vals, h->hs, flag.p);
        TF_LAUNCH_CHECK();
    } else {
        auto kern = (dim == 3) ? k_lat_rows<3, true> : k_lat_rows<2, true>;
        TF_TRY(grid_for(kern, smem_tab, &grid));
        kern<<<grid, 256, smem_tab, s>>>(c, L, dtab, ntab, h->rowptr, nullptr, h->cols, h->vals, h->hs, flag.p);
        TF_LAUNCH_CHECK();
    }
    build_trace().mark("lattice fill", s);
    int32_t hflag = 0;
    TF_CUDA_TRY(cudaMemcpyAsync(&hflag, flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    if (hflag != 0) {
        set_error("internal: lattice fill disagreed with its count pass (row lengths)");
        return TF_ERR_CUDA;
    }
    h->info.bin_side = 0.0;
    for (int d = 0; d < 3; ++d) h->info.bins[d] = nd[d];
    h->info.nbins = M.nx * M.ny * M.nz;
    h->info.max_candidates = maxK;
    if (exact) h->max_row_hint = maxK;  // exact mode: the longest class list is the longest row
    h->info.large_rows = 0;
    h->info.radix_passes = 0;
    h->info.path = exact ? TF_PATH_LATTICE_EXACT : TF_PATH_LATTICE_TESTED;
    *used = true;
    return TF_OK;
}

bool lattice_check_ok(const tf_filter_s *h) {
    const unsigned long long *k = h->lat_check;
    if (!k) return false;
    double dev;
    memcpy(&dev, &k[0], sizeof(dev));
    const bool verified = (k[1] & 3ull) == 0 && dev == 0.0;  // finite, exact, on the lattice
    const int32_t fill_flag = (int32_t)(k[2] & 0xffffffffull);
    return verified && fill_flag == 0 && (int64_t)k[3] == h->lat_nnz_host;
}

tf_status lattice_detect_host(const double *c, int64_t n, int dim, int32_t *T, int64_t cubes[3], double spacing[3]) {
    *T = 0;
    for (int d = 0; d < 3; ++d) cubes[d] = 0, spacing[d] = 0.0;
    if (n < 4) return TF_OK;
    LatModel M;
    bool found = false;
    HostPoints src(c, dim);
    TF_TRY(detect_model(src, n, dim, &M, &found));
    if (!found) return TF_OK;
    *T = M.T;
    cubes[0] = M.nx, cubes[1] = M.ny, cubes[2] = M.nz;
    for (int d = 0; d < 3; ++d) spacing[d] = M.h[d];
    return TF_OK;
}

}  // namespace tf
