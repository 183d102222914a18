// cl_build.cu -- the cell-list build's pair decisions and CSR fill, by query GROUPS (round 2).
//
// Method (sec. 3.2.2 / 4.5; Eq. filter_cond, listing PAPER.md:442-445):
// W_ij = max(0, rmin - |c_i - c_j|) for the pairs with d^2 < rmin^2, columns ascending, Hs = row
// sums. build.cu has already binned the centroids (a2-a4: bbox, keys, radix sort, cell start,
// sorted SoA); this file does a5 (count), a7 (fill) on top of that, and hands the row lengths to
// the a6 scan in between.
//
// Design. A GROUP is <= kGroupQ (32) consecutive points of the cell-sorted order
// inside one "unit" (a bin row cut into blocks of kUnitBins bins), i.e. a compact run along x:
//   k_cl_groups  group records and the size of each group's UNION neighbourhood -- the 3^(dim-1)
//                contiguous x-runs [bx0-1, bx1+1] of the bin rows around it;
//   k_cl_count   block per group: (1) stages the union, (2) sorts it by point id with the block
//                radix sort (smem_sort.cuh), so the union is in ascending COLUMN order, (3) writes
//                that sorted list (sorted-SoA positions) for the fill, (4) sweeps it: lane = query,
//                every union candidate tested with packed fp32x2 math in EDM form (R4c), one sign
//                bit per test funnel-shifted (SHF.L.W) into a per-query 32-bit mask word, band
//                candidates caught by a running unsigned minimum (VIMNMX3) and decided by the
//                exact fp64 test; (5) stores the words (coalesced, word k of query q at [k][q]) and
//                the row length = popcount;
//   k_cl_fill    warp per group: lane = query walks its mask words (branch-free, two bits per
//                step) into a list of candidate indices, then lane = entry writes each row: exact
//                fp64 coordinates, the oracle's d^2 and weight, coalesced int32 / fp64 stores, Hs by
//                a fixed-order lane reduction. No pair is tested twice: the set bits ARE the
//                accepted pairs.
// The per-bin kernels of build.cu (k_count / k_fill) stay as TF_BUILD_CELL_LIST_BINS and as the
// fallback for unions beyond kMaxUnion. Measured: both group kernels are bound
// by L1 wavefronts -- the sweep's broadcast candidate loads and the sort in the count, the
// per-entry coordinate gathers in the fill.
//
// Exactness (R2-R4, R4c): a bit is set only if the fp32 value proves d^2 < r^2 with
// the derived error bound, or the exact fp64 test (pair_d2, uncontracted) says so; the fill's
// weight is the oracle's expression on the caller's bytes. The CSR is therefore bitwise the
// per-bin path's and the oracle's.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "tf_internal.cuh"
#include "smem_sort.cuh"

namespace tf {
namespace {

constexpr int kUnitBins = 32;     // bins per unit along x: a group spans at most this many bins
#ifndef TF_CL_GROUPQ
#define TF_CL_GROUPQ 32
#endif
constexpr int kGroupQ = TF_CL_GROUPQ;  // queries per group (they share one sorted union); 32 per fill warp
constexpr int kHalves = kGroupQ / 32;
constexpr int kMaxUnion = 6144;   // largest union (candidates) the group kernels take
constexpr float kFarCC = 1e30f;   // |c|^2 of padding candidates / q of idle lanes: never "in"

struct GroupRec {
    int32_t q0, q1;    // sorted positions [q0, q1), q1 - q0 <= kGroupQ
    int32_t bx0, bx1;  // bin x-range of the group's queries
    int32_t row;       // bin row index by + bz * nb[1]
    int32_t L;         // union size (candidates)
};

// ---- packed fp32x2 (sm_100a FADD2 / FFMA2)
typedef unsigned long long f2u;
__device__ __forceinline__ f2u f2_pack(float a, float b) {
    return ((f2u)__float_as_uint(b) << 32) | (f2u)__float_as_uint(a);
}
__device__ __forceinline__ uint32_t f2_lo_bits(f2u v) { return (uint32_t)(v & 0xffffffffull); }
__device__ __forceinline__ uint32_t f2_hi_bits(f2u v) { return (uint32_t)(v >> 32); }
__device__ __forceinline__ f2u f2_add(f2u a, f2u b) {
    f2u r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2u f2_fma(f2u a, f2u b, f2u c) {
    f2u r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// ---- one sorted point (x, y, z, id) as a single 256-bit load of its 32-byte AoS record
struct PtRec {
    double x, y, z;
    int32_t id;
};
__device__ __forceinline__ PtRec load_pt(const double4 *a, int p) {
    PtRec r;
    double w;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(w) : "l"(a + p));
    r.id = (int32_t)__double_as_longlong(w);
    return r;
}

// ---- units and groups
// Unit u = (bin row, x block of kUnitBins bins); its points are one contiguous sorted range.
__device__ __forceinline__ void unit_range(int64_t u, const Grid &g, int nxb, const int32_t *cs, int32_t &s,
                                           int32_t &e) {
    const int64_t row = u / nxb;
    const int xb = (int)(u % nxb);
    const int64_t b0 = row * g.nb[0] + (int64_t)xb * kUnitBins;
    const int64_t b1 = row * g.nb[0] + std::min<int64_t>((int64_t)xb * kUnitBins + kUnitBins, g.nb[0]);
    s = cs[b0];
    e = cs[b1];
}

// ng[u] = groups of unit u (ceil(points / kGroupQ)); ng[U] = 0 (the scan's total slot)
__global__ void __launch_bounds__(256) k_cl_units(const int32_t *__restrict__ cs, Grid g, int nxb, int64_t U,
                                                  int32_t *__restrict__ ng) {
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= U; u += (int64_t)gridDim.x * blockDim.x) {
        if (u == U) {
            ng[u] = 0;
            continue;
        }
        int32_t s, e;
        unit_range(u, g, nxb, cs, s, e);
        ng[u] = (e - s + kGroupQ - 1) / kGroupQ;
    }
}

// Union runs of a group: lane r < NR gets run r = bin row (by + dy, bz + dz), x-bins
// [bx0 - 1, bx1 + 1] clipped to the grid, as the contiguous sorted range [s, s + len).
template <int DIM>
__device__ __forceinline__ void group_run(int r, const GroupRec &G, const Grid &g, const int32_t *cs, int &s,
                                          int &len) {
    s = 0;
    len = 0;
    const int by = G.row % g.nb[1], bz = G.row / g.nb[1];
    const int dz = (DIM == 3) ? (r / 3 - 1) : 0;
    const int dy = r % 3 - 1;
    const int yy = by + dy, zz = bz + dz;
    if (yy < 0 || yy >= g.nb[1] || zz < 0 || zz >= g.nb[2]) return;
    const int xl = max(G.bx0 - 1, 0), xh = min(G.bx1 + 1, g.nb[0] - 1);
    const int64_t rb = ((int64_t)zz * g.nb[1] + yy) * g.nb[0];
    s = cs[rb + xl];
    len = cs[rb + xh + 1] - s;
}

// Thread per unit: the unit's group records and padded union sizes; stats[0] = max union.
template <int DIM>
__global__ void __launch_bounds__(256) k_cl_groups(const int32_t *__restrict__ cs, const uint32_t *__restrict__ keys,
                                                   Grid g, int nxb, int64_t U, const int32_t *__restrict__ goff,
                                                   GroupRec *__restrict__ rec, int32_t *__restrict__ lp,
                                                   int32_t *__restrict__ stats) {
    constexpr int NR = (DIM == 3) ? 9 : 3;
    int best = 0;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
        int32_t s, e;
        unit_range(u, g, nxb, cs, s, e);
        const int32_t row = (int32_t)(u / nxb);
        int32_t gi = goff[u];
        for (int32_t q0 = s; q0 < e; q0 += kGroupQ, ++gi) {
            GroupRec G;
            G.q0 = q0;
            G.q1 = min(q0 + kGroupQ, e);
            G.bx0 = (int32_t)(keys[G.q0] % (uint32_t)g.nb[0]);
            G.bx1 = (int32_t)(keys[G.q1 - 1] % (uint32_t)g.nb[0]);
            G.row = row;
            int L = 0;
            for (int r = 0; r < NR; ++r) {
                int rs, rl;
                group_run<DIM>(r, G, g, cs, rs, rl);
                L += rl;
            }
            G.L = L;
            rec[gi] = G;
            lp[gi] = (L + 31) & ~31;
            best = max(best, L);
        }
    }
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best > 0) atomicMax(&stats[0], best);
}

// Per-group origin and the R4c error band. o = centre of the union box; Mx, My, Mz bound
// |c - o| per component over the union (x: (bx1 - bx0 + 3)/2 bins, y/z: 1.5 bins; 1e-4 margin for
// the binning's rounding). With S = Mx^2 + My^2 + Mz^2 the EDM-form fp32 value u of
// d^2 - t_in errs by at most E_r + E_conv <= 1.6e-6 S + 3e-7 r2 (R4c); E = 4e-6 S + 1e-6 r2.
struct GroupFrame {
    double ox, oy, oz;
    double t_in;     // r2 - 2E: u < 0 proves d^2 < r2
    float delta;     // fp32 >= 4E, rounded up: u > delta proves d^2 >= r2
};

template <int DIM>
__device__ __forceinline__ GroupFrame group_frame(const GroupRec &G, const Grid &g) {
    GroupFrame f;
    const int by = G.row % g.nb[1], bz = G.row / g.nb[1];
    f.ox = g.lo[0] + 0.5 * (double)(G.bx0 + G.bx1 + 1) * g.s;
    f.oy = g.lo[1] + ((double)by + 0.5) * g.s;
    f.oz = (DIM == 3) ? g.lo[2] + ((double)bz + 0.5) * g.s : 0.0;
    const double mx = 0.5 * (double)(G.bx1 - G.bx0 + 3) * g.s * (1.0 + 1e-4);
    const double my = 1.5 * g.s * (1.0 + 1e-4);
    const double S = mx * mx + my * my + (DIM == 3 ? my * my : 0.0);
    const double E = 4e-6 * S + 1e-6 * g.r2;
    f.t_in = g.r2 - 2.0 * E;
    f.delta = __double2float_ru(4.0 * E);
    return f;
}

// ------------------------------------------------------------------ a5: count (group kernel)
// One block of kCountWarps warps per group. Shared memory (dynamic): 5 arrays of LPmax uint32:
//   sort: block radix sort ping-pong (Q3 keys, Q4 vals) <-> (Q0 keys, Q1 vals), staged so the
//         sorted vals (sorted-SoA positions) end in Q4;
//   sweep: A = (Q0, Q1) as float4 (x0, x1, y0, y1) per candidate pair, B = (Q2, Q3) as float4
//          (z0, z1, cc0, cc1) [2D: float2 (cc0, cc1) in Q2]; Q4 keeps the positions.
// The sweep splits the union's mask words over the warps (word k -> warp k mod kCountWarps); every
// warp runs the same 32 queries (lane = query) and the row length is summed over the warps.
#ifndef TF_CL_COUNT_WARPS
#define TF_CL_COUNT_WARPS 4
#endif
constexpr int kCountWarps = TF_CL_COUNT_WARPS;

template <int DIM>
__global__ void __launch_bounds__(kCountWarps * 32) k_cl_count(SortedPtsView P, Grid g, const GroupRec *__restrict__ rec,
                                                                const int64_t *__restrict__ loff, int LPmax,
                                                                int32_t *__restrict__ list, uint32_t *__restrict__ mask,
                                                                int32_t *__restrict__ counts,
                                                                int32_t *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int32_t wc[kCountWarps][256];
    __shared__ int32_t wsum[kCountWarps];
    __shared__ int run_s[9], run_x[10];
    __shared__ int lohi[2];
    __shared__ int wcnt[kCountWarps][kGroupQ];
    constexpr int NR = (DIM == 3) ? 9 : 3;
    constexpr int T = kCountWarps * 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t *Q0 = reinterpret_cast<uint32_t *>(smem_raw), *Q1 = Q0 + LPmax, *Q2 = Q0 + 2 * LPmax,
             *Q3 = Q0 + 3 * LPmax, *Q4 = Q0 + 4 * LPmax;
    const GroupRec R = rec[blockIdx.x];
    const int L = R.L, LP = (L + 31) & ~31;
    const int64_t base = loff[blockIdx.x];

    // (1) union runs (warp 0) -> shared run starts, exclusive offsets and bin-row bases
    __shared__ int64_t run_rb[9];
    if (warp == 0) {
        int rs = 0, rl = 0;
        int64_t rb = -1;
        if (lane < NR) {
            group_run<DIM>(lane, R, g, P.cs, rs, rl);
            const int by = R.row % g.nb[1], bz = R.row / g.nb[1];
            const int yy = by + lane % 3 - 1, zz = bz + ((DIM == 3) ? lane / 3 - 1 : 0);
            if (yy >= 0 && yy < g.nb[1] && zz >= 0 && zz < g.nb[2]) rb = ((int64_t)zz * g.nb[1] + yy) * g.nb[0];
        }
        int incl = rl;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane < NR) run_s[lane] = rs, run_x[lane] = incl - rl, run_rb[lane] = rb;
        if (lane == NR - 1) run_x[NR] = incl;
        if (lane == 0) lohi[0] = 0x7fffffff, lohi[1] = 0;
    }
    __syncthreads();
    // (2a) id range of the union from its bins' first and last points (ids ascend inside a bin)
    {
        const int xl = max(R.bx0 - 1, 0), xh = min(R.bx1 + 1, g.nb[0] - 1), nbr = xh - xl + 1;
        int lo = 0x7fffffff, hi = 0;
        for (int f = tid; f < NR * nbr; f += T) {
            const int r = f / nbr;
            if (run_rb[r] < 0) continue;
            const int64_t bin = run_rb[r] + xl + f % nbr;
            const int32_t a0 = P.cs[bin], a1 = P.cs[bin + 1];
            if (a1 > a0) lo = min(lo, P.id[a0]), hi = max(hi, P.id[a1 - 1]);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) atomicMin(&lohi[0], lo), atomicMax(&lohi[1], hi);
    }
    __syncthreads();
    const int lo = lohi[0];
    const int bits = (lohi[1] > lo) ? 32 - __clz((unsigned)(lohi[1] - lo)) : 0;
    // (sorting only the top 16 bits and repairing the equal-high-bit runs was measured slower at
    // config 5: Kuhn tets of one cube fall in different y/z bins, so most runs needed repair)
    const int s_lo = 0;
    const int passes = (bits - s_lo + 7) >> 3;
    // the sort ping-pongs (ka, va) -> (kb, vb) -> ...; sorted vals must end in Q4:
    //   even passes: ka = Q3, va = Q4, kb = Q0, vb = Q1;  odd: ka = Q0, va = Q1, kb = Q3, vb = Q4
    uint32_t *KA = (passes & 1) ? Q0 : Q3, *VA = (passes & 1) ? Q1 : Q4;
    uint32_t *KB = (passes & 1) ? Q3 : Q0, *VB = (passes & 1) ? Q4 : Q1;
    // (2b) stage (id - lo, sorted-SoA position) in run order
    {
        int r = 0;
        for (int t0 = 0; t0 < L; t0 += 4 * T) {
            int id[4], pp[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = t0 + u * T + tid;
                while (r < NR - 1 && t >= run_x[r + 1]) ++r;
                pp[u] = run_s[r] + (t - run_x[r]);
                id[u] = (t < L) ? P.id[pp[u]] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = t0 + u * T + tid;
                if (t < L) KA[t] = (uint32_t)(id[u] - lo), VA[t] = (uint32_t)pp[u];
            }
        }
    }
    __syncthreads();
    block_radix_sort_bits<kCountWarps>(KA, VA, KB, VB, L, s_lo, bits, wc, wsum);
    if (s_lo > 0) block_fix_low_bits(Q3, Q4, L, s_lo);
    // (3) the sorted union (ascending id) for the fill; (4) sweep operands in sorted order,
    // fp32 offsets from the group origin (R4c)
    const GroupFrame F = group_frame<DIM>(R, g);
    float4 *A = reinterpret_cast<float4 *>(Q0);
    float4 *B3 = reinterpret_cast<float4 *>(Q2);
    float2 *B2 = reinterpret_cast<float2 *>(Q2);
    for (int j0 = 0; j0 < LP / 2; j0 += 2 * T) {
        double xs[2][2], ys[2][2], zs[2][2];
        bool ok[2][2];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = j0 + u * T + tid, t = 2 * j + h;
                ok[u][h] = (j < LP / 2) && (t < L);
                xs[u][h] = ys[u][h] = zs[u][h] = 0.0;
                if (ok[u][h]) {
                    const int p = (int)Q4[t];
                    list[base + t] = p;
                    const PtRec c = load_pt(P.a, p);
                    xs[u][h] = c.x;
                    ys[u][h] = c.y;
                    if (DIM == 3) zs[u][h] = c.z;
                }
            }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = j0 + u * T + tid;
            if (j >= LP / 2) continue;
            float x[2], y[2], z[2], cc[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (ok[u][h]) {
                    x[h] = __double2float_rn(xs[u][h] - F.ox);
                    y[h] = __double2float_rn(ys[u][h] - F.oy);
                    z[h] = (DIM == 3) ? __double2float_rn(zs[u][h] - F.oz) : 0.f;
                    const double xx = x[h], yy = y[h], zz = z[h];
                    cc[h] = __double2float_rn(xx * xx + yy * yy + zz * zz);
                } else {
                    x[h] = y[h] = z[h] = 0.f;
                    cc[h] = kFarCC;
                }
            }
            A[j] = make_float4(x[0], x[1], y[0], y[1]);
            if (DIM == 3) B3[j] = make_float4(z[0], z[1], cc[0], cc[1]);
            else B2[j] = make_float2(cc[0], cc[1]);
        }
    }
    __syncthreads();
    // (5) sweep: every warp runs all kGroupQ queries -- lane = queries lane, lane + 32, ... (NQ per
    // lane, so one broadcast candidate load serves NQ * 32 tests) -- on its share of the union's mask
    // words (word k -> warp k mod kCountWarps); the row length is summed over the warps.
    constexpr int NQ = kHalves;
    int q[NQ];
    bool have[NQ];
    double qxd[NQ], qyd[NQ], qzd[NQ];
    f2u QX[NQ], QY[NQ], QZ[NQ], QQ[NQ];
#pragma unroll
    for (int h = 0; h < NQ; ++h) {
        q[h] = R.q0 + 32 * h + lane;
        have[h] = q[h] < R.q1;
        qxd[h] = qyd[h] = qzd[h] = 0.0;
        QX[h] = QY[h] = QZ[h] = 0;
        if (have[h]) {
            const PtRec c = load_pt(P.a, q[h]);
            qxd[h] = c.x;
            qyd[h] = c.y;
            qzd[h] = (DIM == 3) ? c.z : 0.0;
            const float bx = __double2float_rn(qxd[h] - F.ox), by = __double2float_rn(qyd[h] - F.oy),
                        bz = (DIM == 3) ? __double2float_rn(qzd[h] - F.oz) : 0.f;
            const double bb = (double)bx * bx + (double)by * by + (double)bz * bz;
            const float qq = __double2float_rn(bb - F.t_in);
            QX[h] = f2_pack(-2.f * bx, -2.f * bx);
            QY[h] = f2_pack(-2.f * by, -2.f * by);
            QZ[h] = f2_pack(-2.f * bz, -2.f * bz);
            QQ[h] = f2_pack(qq, qq);
        } else {
            QQ[h] = f2_pack(kFarCC, kFarCC);
        }
    }
    const uint32_t dbits = __float_as_uint(F.delta);
    const ulonglong2 *A2 = reinterpret_cast<const ulonglong2 *>(A);
    const ulonglong2 *B32 = reinterpret_cast<const ulonglong2 *>(B3);
    const f2u *B22 = reinterpret_cast<const f2u *>(B2);
    const double r2 = g.r2;
    int cnt[NQ];
#pragma unroll
    for (int h = 0; h < NQ; ++h) cnt[h] = 0;
    for (int k = warp; k < LP / 32; k += kCountWarps) {
        // four independent 8-candidate accumulators per query (shorter dependency chains), then combined
        uint32_t wq[NQ][4], bm[NQ][4];
#pragma unroll
        for (int h = 0; h < NQ; ++h)
#pragma unroll
            for (int u = 0; u < 4; ++u) wq[h][u] = 0u, bm[h][u] = 0xffffffffu;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const ulonglong2 a = A2[16 * k + j];
            ulonglong2 b;
            f2u cc;
            if (DIM == 3) {
                b = B32[16 * k + j];
                cc = b.y;
            } else {
                cc = B22[16 * k + j];
            }
#pragma unroll
            for (int h = 0; h < NQ; ++h) {
                f2u acc = f2_add(cc, QQ[h]);
                acc = f2_fma(QX[h], a.x, acc);
                acc = f2_fma(QY[h], a.y, acc);
                if (DIM == 3) acc = f2_fma(QZ[h], b.x, acc);
                const uint32_t u0 = f2_lo_bits(acc), u1 = f2_hi_bits(acc);
                wq[h][j >> 2] = __funnelshift_l(u0, wq[h][j >> 2], 1);
                wq[h][j >> 2] = __funnelshift_l(u1, wq[h][j >> 2], 1);
                bm[h][j >> 2] = min(min(bm[h][j >> 2], u0), u1);
            }
        }
#pragma unroll
        for (int h = 0; h < NQ; ++h) {
            uint32_t w = (wq[h][0] << 24) | (wq[h][1] << 16) | (wq[h][2] << 8) | wq[h][3];
            const uint32_t bmin = min(min(bm[h][0], bm[h][1]), min(bm[h][2], bm[h][3]));
            if (bmin <= dbits) {
                // band: some candidate of this word has 0 <= u <= delta -> decide it exactly
                // (bit 31 - b <-> candidate 32k + b); u recomputed with the same roundings
                const float *Af = reinterpret_cast<const float *>(A);
                const float *Bf = reinterpret_cast<const float *>(Q2);
                const float qq = __uint_as_float(f2_lo_bits(QQ[h]));
                const float mx = __uint_as_float(f2_lo_bits(QX[h])), my = __uint_as_float(f2_lo_bits(QY[h])),
                            mz = __uint_as_float(f2_lo_bits(QZ[h]));
                for (int b = 0; b < 32; ++b) {
                    const int t = 32 * k + b, j = t >> 1, hh = t & 1;
                    float u;
                    if (DIM == 3) {
                        u = __fadd_rn(Bf[4 * j + 2 + hh], qq);
                        u = __fmaf_rn(mx, Af[4 * j + hh], u);
                        u = __fmaf_rn(my, Af[4 * j + 2 + hh], u);
                        u = __fmaf_rn(mz, Bf[4 * j + hh], u);
                    } else {
                        u = __fadd_rn(Bf[2 * j + hh], qq);
                        u = __fmaf_rn(mx, Af[4 * j + hh], u);
                        u = __fmaf_rn(my, Af[4 * j + 2 + hh], u);
                    }
                    if (__float_as_uint(u) <= dbits && t < L) {
                        const PtRec c = load_pt(P.a, (int)Q4[t]);
                        if (pair_d2<DIM>(qxd[h], qyd[h], qzd[h], c.x, c.y, (DIM == 3) ? c.z : 0.0) < r2)
                            w |= 0x80000000u >> b;
                    }
                }
            }
            if (!have[h]) w = 0;
            mask[kHalves * base + kGroupQ * k + 32 * h + lane] = w;
            cnt[h] += __popc(w);
        }
    }
#pragma unroll
    for (int h = 0; h < NQ; ++h) wcnt[warp][32 * h + lane] = cnt[h];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int h = 0; h < NQ; ++h) {
            if (!have[h]) continue;
            int c = 0;
#pragma unroll
            for (int w = 0; w < kCountWarps; ++w) c += wcnt[w][32 * h + lane];
            counts[P.id[q[h]]] = c;
            if (c > stats[3]) atomicMax(&stats[3], c);  // longest row (apply plan)
        }
    }
}

// ------------------------------------------------------------------ a7: fill (group kernel)
// Warp per half group (32 queries), two phases.
//  expansion (lane = query): the half's mask words are staged in shared memory transposed to
//    [lane][word] (odd stride); each lane walks its own words -- up to two set bits or one word step
//    per iteration, independently of the other lanes -- and appends the candidate indices
//    (ascending = ascending column) to its list ent[lane][0..len);
//  emission (lane = entry): two rows per pass, their first kFillRounds 32-entry rounds in flight
//    together: sorted-SoA position from the group's union list, exact fp64 coordinates and id,
//    the oracle's d^2 and weight, coalesced int32 / fp64 stores, Hs by a fixed-order lane reduction.
// Shared memory per warp: masks [32][MS] uint32 (MS odd, > words) + lists [32][S] uint16.
#ifndef TF_CL_FILL_ROUNDS
#define TF_CL_FILL_ROUNDS 3
#endif
constexpr int kFillRounds = TF_CL_FILL_ROUNDS;
constexpr int kListCap = 256;  // per-lane list capacity; longer rows take the word-parallel path

template <int DIM, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_cl_fill(SortedPtsView P, Grid g, const GroupRec *__restrict__ rec,
                                                        const int64_t *__restrict__ loff, int32_t G, int MS, int S,
                                                        const int32_t *__restrict__ list,
                                                        const uint32_t *__restrict__ mask,
                                                        const int64_t *__restrict__ rowptr,
                                                        int32_t *__restrict__ cols, double *__restrict__ vals,
                                                        double *__restrict__ hs, int32_t *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t wi = (int32_t)blockIdx.x * WARPS + warp;
    const int32_t gi = wi / kHalves, half = wi % kHalves;
    if (gi >= G) return;
    const size_t per_warp = (size_t)32 * MS * 4 + (size_t)32 * S * 2;
    uint32_t *sm = reinterpret_cast<uint32_t *>(smem_raw + (size_t)warp * per_warp);  // [32][MS]
    uint16_t *ent = reinterpret_cast<uint16_t *>(sm + 32 * MS);                       // [32][S]
    GroupRec R = rec[gi];
    R.q0 += 32 * half;  // this warp's queries
    R.q1 = min(R.q1, R.q0 + 32);
    if (R.q0 >= R.q1) return;
    const int L = R.L, LP = (L + 31) & ~31, nw = LP >> 5;
    const int64_t base = loff[gi];
    const uint32_t *mk = mask + kHalves * base + 32 * half;
    for (int k0 = 0; k0 < MS; k0 += 4) {
        uint32_t m[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) m[u] = (k0 + u < nw) ? mk[kGroupQ * (k0 + u) + lane] : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (k0 + u < MS) sm[lane * MS + k0 + u] = m[u];
    }
    const int q = R.q0 + lane;
    const bool have = q < R.q1;
    int32_t qid = 0;
    int64_t rbase = 0;
    int len = 0;
    if (have) {
        qid = P.id[q];
        rbase = rowptr[qid];
        len = (int)(rowptr[qid + 1] - rbase);
    }
    __syncwarp();
    {
        // branch-free walk: every iteration either emits the lane's next set bit or steps to its
        // next word (mw has MS >= nw + 1 words per lane, the extra one zero)
        const uint32_t *mw = sm + lane * MS;
        uint16_t *my = ent + (size_t)lane * S;
        int n = 0, k = 0;
        uint32_t w = mw[0];
        const int kend = have ? nw : 0;
        while (__any_sync(0xffffffffu, k < kend)) {
#pragma unroll 2
            for (int u = 0; u < 2; ++u) {
                // up to two set bits of the current word, or one word step
                const bool z = (w == 0);
                const int b1 = __clz(w) & 31;
                const uint32_t w1 = w ^ (0x80000000u >> b1);
                const int b2 = __clz(w1) & 31;
                const bool two = !z && (w1 != 0);
                my[min(n, S - 1)] = (uint16_t)(32 * k + b1);
                my[min(n + 1, S - 1)] = (uint16_t)(32 * k + b2);
                n += z ? 0 : (two ? 2 : 1);
                const uint32_t wn = mw[min(k + 1, MS - 1)];
                w = z ? wn : (two ? (w1 ^ (0x80000000u >> b2)) : 0u);
                k = z ? min(k + 1, nw) : k;
            }
        }
        if (have && n != len) atomicOr(&stats[2], 1);  // count/fill agreement (always-on invariant)
    }
    __syncwarp();
    const double rmin = g.rmin;
#ifdef TF_DEBUG_CHECKS
    const double r2 = g.r2;
#endif
    const int nq = R.q1 - R.q0;
    for (int i0 = 0; i0 < nq; i0 += 2) {
        int li[2];
        bool longrow[2];
        int32_t qi[2];
        int64_t bi[2];
        double qx[2], qy[2], qz[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = min(i0 + h, nq - 1);
            li[h] = (i0 + h < nq) ? __shfl_sync(0xffffffffu, len, i) : 0;
            longrow[h] = li[h] > S - 2;
            if (longrow[h]) li[h] = 0;
            bi[h] = __shfl_sync(0xffffffffu, rbase, i);
            qi[h] = __shfl_sync(0xffffffffu, qid, i);
            qx[h] = P.x[R.q0 + i];
            qy[h] = P.y[R.q0 + i];
            qz[h] = (DIM == 3) ? P.z[R.q0 + i] : 0.0;
        }
        double cx[2][kFillRounds], cy[2][kFillRounds], cz[2][kFillRounds];
        int32_t cid[2][kFillRounds];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int r = 0; r < kFillRounds; ++r) {
                const int e = 32 * r + lane;
                const int p = (e < li[h]) ? list[base + ent[(size_t)(i0 + h) * S + e]] : list[base];
                const PtRec c = load_pt(P.a, p);
                cx[h][r] = c.x;
                cy[h][r] = c.y;
                cz[h][r] = (DIM == 3) ? c.z : 0.0;
                cid[h][r] = c.id;
            }
        double hsum[2] = {0.0, 0.0};
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int r = 0; r < kFillRounds; ++r) {
                const int e = 32 * r + lane;
                if (e < li[h]) {
                    const double d2 = pair_d2<DIM>(qx[h], qy[h], qz[h], cx[h][r], cy[h][r], cz[h][r]);
                    const double w = weight_of(rmin, d2);
                    cols[bi[h] + e] = cid[h][r];
                    vals[bi[h] + e] = w;
                    hsum[h] += w;
                    TF_DCHECK(d2 < r2);
                }
            }
#pragma unroll
        for (int h = 0; h < 2; ++h)
            for (int e = 32 * kFillRounds + lane; e < li[h]; e += 32) {
                const int p = list[base + ent[(size_t)(i0 + h) * S + e]];
                const PtRec c = load_pt(P.a, p);
                const double d2 = pair_d2<DIM>(qx[h], qy[h], qz[h], c.x, c.y, (DIM == 3) ? c.z : 0.0);
                const double w = weight_of(rmin, d2);
                cols[bi[h] + e] = c.id;
                vals[bi[h] + e] = w;
                hsum[h] += w;
                TF_DCHECK(d2 < r2);
            }
        // rows longer than the lists (dense clusters): lane = mask word of the row, positions from
        // a warp scan of the words' popcounts, each lane emits its word's bits
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!longrow[h]) continue;
            const int i = i0 + h;
            int done = 0;
            for (int k0 = 0; k0 < nw; k0 += 32) {
                const int k = k0 + lane;
                uint32_t w = (k < nw) ? sm[i * MS + k] : 0u;
                const int c = __popc(w);
                int inc = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += v;
                }
                int e = done + inc - c;
                while (w) {
                    const int b = __clz(w);
                    const int p = list[base + 32 * k + b];
                    const double d2 = pair_d2<DIM>(qx[h], qy[h], qz[h], P.x[p], P.y[p], (DIM == 3) ? P.z[p] : 0.0);
                    const double wt = weight_of(rmin, d2);
                    cols[bi[h] + e] = P.id[p];
                    vals[bi[h] + e] = wt;
                    hsum[h] += wt;
                    TF_DCHECK(d2 < r2);
                    ++e;
                    w ^= 0x80000000u >> b;
                }
                done += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            hsum[0] += __shfl_xor_sync(0xffffffffu, hsum[0], o);
            hsum[1] += __shfl_xor_sync(0xffffffffu, hsum[1], o);
        }
        if (lane == 0) {
            hs[qi[0]] = hsum[0];
            if (i0 + 1 < nq) hs[qi[1]] = hsum[1];
        }
    }
}

// ------------------------------------------------------------------ a7: fill, warp per group, row by row
// The default fill (round 2, second version). Warp per group; the rows of the group's queries are
// written one after the other, and the expansion of a row's mask words into its candidate list is
// done by the whole warp, right before the row is written:
//  expansion (lane = mask word of the row): popcount, warp scan of the counts -> each lane appends
//    the bit positions of its own word at its offset of the row's list (ascending = ascending
//    column). Lists are double-buffered per warp ([2][S] uint16), so the list of row i + 1 is built
//    while the candidate points of row i are in flight;
//  emission (lane = entry): ROUNDS 32-entry rounds in flight: sorted position from the group's
//    union list, the whole point in one 256-bit load, the oracle's d^2 and weight, coalesced
//    int32 / fp64 stores, Hs by a fixed-order lane reduction.
// Against k_cl_fill this keeps no transposed mask copy and no per-query lists in shared memory
// (10.5 KB -> < 0.5 KB per warp at config 5) and has no serial per-lane walk at the start of a group;
// the occupancy limit becomes the register count (launch bounds: kFill2MinBlocks blocks of 4 warps).
#ifndef TF_CL_FILL2_MINB
#define TF_CL_FILL2_MINB 8
#endif
constexpr int kFill2Warps = 4;
constexpr int kFill2MinBlocks = TF_CL_FILL2_MINB;

// list of query i of the group: expand the set bits of its mask words (mk[32 * k + i], k < nw) into
// dst[0..n) (candidate indices, ascending); returns n (uniform). Entries beyond cap are dropped.
__device__ __forceinline__ int expand_row(const uint32_t *__restrict__ mk, int i, int nw, uint16_t *dst, int cap,
                                          int lane) {
    int done = 0;
    for (int k0 = 0; k0 < nw; k0 += 32) {
        const int k = k0 + lane;
        uint32_t w = (k < nw) ? mk[32 * k + i] : 0u;
        const int c = __popc(w);
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        int e = done + inc - c;
        const int t0 = 32 * k;
        while (w) {
            const int b = __clz(w);
            if (e < cap) dst[e] = (uint16_t)(t0 + b);
            ++e;
            w ^= 0x80000000u >> b;
        }
        done += __shfl_sync(0xffffffffu, inc, 31);
    }
    return done;
}

template <int DIM, int ROUNDS>
__global__ void __launch_bounds__(kFill2Warps * 32, kFill2MinBlocks)
    k_cl_fill2(SortedPtsView P, Grid g, const GroupRec *__restrict__ rec, const int64_t *__restrict__ loff, int32_t G,
               int S, const int32_t *__restrict__ list, const uint32_t *__restrict__ mask,
               const int64_t *__restrict__ rowptr, int32_t *__restrict__ cols, double *__restrict__ vals,
               double *__restrict__ hs, int32_t *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t gi = (int32_t)blockIdx.x * kFill2Warps + warp;
    if (gi >= G) return;
    uint16_t *ent = reinterpret_cast<uint16_t *>(smem_raw) + (size_t)warp * 2 * S;  // [2][S]
    const GroupRec R = rec[gi];
    const int nq = R.q1 - R.q0;
    const int L = R.L, nw = (L + 31) >> 5;
    const int64_t base = loff[gi];
    const uint32_t *mk = mask + base;
    const int32_t *ul = list + base;
    const int q = R.q0 + lane;
    const bool have = lane < nq;
    int32_t qid = 0;
    int64_t rbase = 0;
    int len = 0;
    double qxl = 0.0, qyl = 0.0, qzl = 0.0;
    if (have) {
        const PtRec c = load_pt(P.a, q);
        qid = c.id;
        qxl = c.x, qyl = c.y, qzl = c.z;
        rbase = rowptr[qid];
        len = (int)(rowptr[qid + 1] - rbase);
    }
    const double rmin = g.rmin;
#ifdef TF_DEBUG_CHECKS
    const double r2 = g.r2;
#endif
    int bad = 0;
    int n_next = expand_row(mk, 0, nw, ent, S, lane);
    __syncwarp();
    for (int i = 0; i < nq; ++i) {
        const uint16_t *my = ent + (size_t)(i & 1) * S;
        const int li = __shfl_sync(0xffffffffu, len, i);
        const int64_t bi = __shfl_sync(0xffffffffu, rbase, i);
        const int32_t qi = __shfl_sync(0xffffffffu, qid, i);
        const double qx = __shfl_sync(0xffffffffu, qxl, i), qy = __shfl_sync(0xffffffffu, qyl, i);
        const double qz = (DIM == 3) ? __shfl_sync(0xffffffffu, qzl, i) : 0.0;
        bad |= (n_next != li);  // count/fill agreement (always-on invariant)
        const bool longrow = li > S;
        const int lr = longrow ? 0 : li;
        // candidate points of the first ROUNDS rounds: loads first
        PtRec c[ROUNDS];
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int e = 32 * r + lane;
            const int p = ul[(e < lr) ? my[e] : 0];
            c[r] = load_pt(P.a, p);
        }
        // the next row's list, while those are in flight
        if (i + 1 < nq) n_next = expand_row(mk, i + 1, nw, ent + (size_t)((i + 1) & 1) * S, S, lane);
        double hsum = 0.0;
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int e = 32 * r + lane;
            if (e < lr) {
                const double d2 = pair_d2<DIM>(qx, qy, qz, c[r].x, c[r].y, c[r].z);
                const double w = weight_of(rmin, d2);
                cols[bi + e] = c[r].id;
                vals[bi + e] = w;
                hsum += w;
                TF_DCHECK(d2 < r2);
            }
        }
        for (int e = 32 * ROUNDS + lane; e < lr; e += 32) {
            const PtRec cc = load_pt(P.a, ul[my[e]]);
            const double d2 = pair_d2<DIM>(qx, qy, qz, cc.x, cc.y, cc.z);
            const double w = weight_of(rmin, d2);
            cols[bi + e] = cc.id;
            vals[bi + e] = w;
            hsum += w;
            TF_DCHECK(d2 < r2);
        }
        if (longrow) {
            // rows longer than the list (dense clusters): lane = mask word, each lane emits its bits
            int done = 0;
            for (int k0 = 0; k0 < nw; k0 += 32) {
                const int k = k0 + lane;
                uint32_t w = (k < nw) ? mk[32 * k + i] : 0u;
                const int cnt = __popc(w);
                int inc = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += v;
                }
                int e = done + inc - cnt;
                while (w) {
                    const int b = __clz(w);
                    const PtRec cc = load_pt(P.a, ul[32 * k + b]);
                    const double d2 = pair_d2<DIM>(qx, qy, qz, cc.x, cc.y, cc.z);
                    const double wt = weight_of(rmin, d2);
                    cols[bi + e] = cc.id;
                    vals[bi + e] = wt;
                    hsum += wt;
                    TF_DCHECK(d2 < r2);
                    ++e;
                    w ^= 0x80000000u >> b;
                }
                done += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
        if (lane == 0) hs[qi] = hsum;
        __syncwarp();
    }
    if (bad) atomicOr(&stats[2], 1);
}

template <int DIM, int ROUNDS>
tf_status launch_cl_fill2(const SortedPtsView &P, const Grid &g, const GroupRec *rec, const int64_t *loff, int32_t G,
                          int S, const int32_t *list, const uint32_t *mask, tf_filter_s *h, int32_t *stats,
                          cudaStream_t s) {
    const size_t smem = (size_t)kFill2Warps * 2 * S * sizeof(uint16_t);
    auto kern = k_cl_fill2<DIM, ROUNDS>;
    kern<<<(unsigned)(((int64_t)G + kFill2Warps - 1) / kFill2Warps), kFill2Warps * 32, smem, s>>>(
        P, g, rec, loff, G, S, list, mask, h->rowptr, h->cols, h->vals, h->hs, stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

// ------------------------------------------------------------------ a7: fill, warp per group, masks from L1
// k_cl_fill with two changes for occupancy (the fill is latency-bound at 5 blocks of 4 warps per SM):
// the walk reads each lane's mask words straight from global memory (word k of query q at [k][q]:
// the group's words stay L1-resident; the next word is loaded one step ahead), so no transposed mask
// copy in shared memory (10.5 -> 5.8 KB per warp at config 5); rows are written one at a time with
// ROUNDS rounds in flight, which fits 64 registers (8 blocks per SM).
#ifndef TF_CL_FILL3_MINB
#define TF_CL_FILL3_MINB 8
#endif
template <int DIM, int ROUNDS>
__global__ void __launch_bounds__(128, TF_CL_FILL3_MINB)
    k_cl_fill3(SortedPtsView P, Grid g, const GroupRec *__restrict__ rec, const int64_t *__restrict__ loff, int32_t G,
               int S, const int32_t *__restrict__ list, const uint32_t *__restrict__ mask,
               const int64_t *__restrict__ rowptr, int32_t *__restrict__ cols, double *__restrict__ vals,
               double *__restrict__ hs, int32_t *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t wi = (int32_t)blockIdx.x * 4 + warp;
    const int32_t gi = wi / kHalves, half = wi % kHalves;  // this warp's 32 queries of the group
    if (gi >= G) return;
    uint16_t *ent = reinterpret_cast<uint16_t *>(smem_raw) + (size_t)warp * 32 * S;  // [32][S]
    GroupRec R = rec[gi];
    R.q0 += 32 * half;
    R.q1 = min(R.q1, R.q0 + 32);
    if (R.q0 >= R.q1) return;
    const int nq = R.q1 - R.q0;
    const int L = R.L, nw = (L + 31) >> 5;
    const int64_t base = loff[gi];
    constexpr int WS = kGroupQ;  // words of one query are WS apart
    const uint32_t *mk = mask + kHalves * base + 32 * half + lane;  // word k of this lane's query at mk[WS * k]
    const int32_t *ul = list + base;
    const bool have = lane < nq;
    int32_t qid = 0;
    int64_t rbase = 0;
    int len = 0;
    double qxl = 0.0, qyl = 0.0, qzl = 0.0;
    if (have) {
        const PtRec c = load_pt(P.a, R.q0 + lane);
        qid = c.id;
        qxl = c.x, qyl = c.y, qzl = c.z;
        rbase = rowptr[qid];
        len = (int)(rowptr[qid + 1] - rbase);
    }
    {
        // branch-free walk: every step either emits up to two set bits of the current word or moves
        // to the next word (loaded one step ahead)
        uint16_t *my = ent + (size_t)lane * S;
        const int kend = have ? nw : 0;
        int n = 0, k = 0;
        uint32_t w = (kend > 0) ? mk[0] : 0u;
        uint32_t wnext = (kend > 1) ? mk[WS] : 0u;
        while (__any_sync(0xffffffffu, k < kend)) {
#pragma unroll 2
            for (int u = 0; u < 2; ++u) {
                const bool z = (w == 0);
                const int b1 = __clz(w) & 31;
                const uint32_t w1 = w ^ (0x80000000u >> b1);
                const int b2 = __clz(w1) & 31;
                const bool two = !z && (w1 != 0);
                my[min(n, S - 1)] = (uint16_t)(32 * k + b1);
                my[min(n + 1, S - 1)] = (uint16_t)(32 * k + b2);
                n += z ? 0 : (two ? 2 : 1);
                const bool step = z && (k < kend);
                const uint32_t wl = (step && k + 2 < kend) ? mk[WS * (k + 2)] : 0u;
                w = z ? wnext : (two ? (w1 ^ (0x80000000u >> b2)) : 0u);
                wnext = step ? wl : wnext;
                k = step ? k + 1 : k;
            }
        }
        if (have && n != len) atomicOr(&stats[2], 1);  // count/fill agreement (always-on invariant)
    }
    __syncwarp();
    const double rmin = g.rmin;
#ifdef TF_DEBUG_CHECKS
    const double r2 = g.r2;
#endif
    for (int i = 0; i < nq; ++i) {
        const uint16_t *my = ent + (size_t)i * S;
        const int li = __shfl_sync(0xffffffffu, len, i);
        const int64_t bi = __shfl_sync(0xffffffffu, rbase, i);
        const int32_t qi = __shfl_sync(0xffffffffu, qid, i);
        const double qx = __shfl_sync(0xffffffffu, qxl, i), qy = __shfl_sync(0xffffffffu, qyl, i);
        const double qz = (DIM == 3) ? __shfl_sync(0xffffffffu, qzl, i) : 0.0;
        const bool longrow = li > S - 2;
        const int lr = longrow ? 0 : li;
        PtRec c[ROUNDS];
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int e = 32 * r + lane;
            c[r] = load_pt(P.a, ul[(e < lr) ? my[e] : 0]);
        }
        double hsum = 0.0;
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int e = 32 * r + lane;
            if (e < lr) {
                const double d2 = pair_d2<DIM>(qx, qy, qz, c[r].x, c[r].y, c[r].z);
                const double w = weight_of(rmin, d2);
                cols[bi + e] = c[r].id;
                vals[bi + e] = w;
                hsum += w;
                TF_DCHECK(d2 < r2);
            }
        }
        for (int e = 32 * ROUNDS + lane; e < lr; e += 32) {
            const PtRec cc = load_pt(P.a, ul[my[e]]);
            const double d2 = pair_d2<DIM>(qx, qy, qz, cc.x, cc.y, cc.z);
            const double w = weight_of(rmin, d2);
            cols[bi + e] = cc.id;
            vals[bi + e] = w;
            hsum += w;
            TF_DCHECK(d2 < r2);
        }
        if (longrow) {
            // rows longer than the lists (dense clusters): lane = mask word, each lane emits its bits
            int done = 0;
            for (int k0 = 0; k0 < nw; k0 += 32) {
                const int k = k0 + lane;
                uint32_t w = (k < nw) ? mk[WS * k + i - lane] : 0u;
                const int cnt = __popc(w);
                int inc = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += v;
                }
                int e = done + inc - cnt;
                while (w) {
                    const int b = __clz(w);
                    const PtRec cc = load_pt(P.a, ul[32 * k + b]);
                    const double d2 = pair_d2<DIM>(qx, qy, qz, cc.x, cc.y, cc.z);
                    const double wt = weight_of(rmin, d2);
                    cols[bi + e] = cc.id;
                    vals[bi + e] = wt;
                    hsum += wt;
                    TF_DCHECK(d2 < r2);
                    ++e;
                    w ^= 0x80000000u >> b;
                }
                done += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
        if (lane == 0) hs[qi] = hsum;
    }
}

template <int DIM, int ROUNDS>
tf_status launch_cl_fill3(const SortedPtsView &P, const Grid &g, const GroupRec *rec, const int64_t *loff, int32_t G,
                          int S, const int32_t *list, const uint32_t *mask, tf_filter_s *h, int32_t *stats,
                          cudaStream_t s) {
    const size_t smem = (size_t)4 * 32 * S * sizeof(uint16_t);
    auto kern = k_cl_fill3<DIM, ROUNDS>;
    TF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)(((int64_t)G * kHalves + 3) / 4), 128, smem, s>>>(P, g, rec, loff, G, S, list, mask, h->rowptr,
                                                                       h->cols, h->vals, h->hs, stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

// ------------------------------------------------------------------ a7: fill, block per group, split walk
// Block of 4 warps per group. (1) Each warp walks one quarter of every query's mask words (lane =
// query; the quarter's list offset = popcount of the words before it), so the serial walk is a
// quarter as long and no warp idles; (2) all threads stage the group's sorted union -- exact fp64
// coordinates and ids, one 256-bit load per point -- in shared memory; (3) warp w writes the rows of
// queries w, w + 4, ...: lane = entry, ROUNDS rounds in flight, candidate data from shared memory
// (each union point is fetched from L2 once per group instead of once per entry: 3.7x fewer L2
// sectors at config 5).
template <int DIM, int ROUNDS>
__global__ void __launch_bounds__(128) k_cl_fill4(SortedPtsView P, Grid g, const GroupRec *__restrict__ rec,
                                                  const int64_t *__restrict__ loff, int LPmax, int S,
                                                  const int32_t *__restrict__ list, const uint32_t *__restrict__ mask,
                                                  const int64_t *__restrict__ rowptr, int32_t *__restrict__ cols,
                                                  double *__restrict__ vals, double *__restrict__ hs,
                                                  int32_t *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double *ux = reinterpret_cast<double *>(smem_raw);
    double *uy = ux + LPmax;
    double *uz = uy + LPmax;
    int32_t *uid = reinterpret_cast<int32_t *>(uz + ((DIM == 3) ? LPmax : 0));
    uint16_t *ent = reinterpret_cast<uint16_t *>(uid + LPmax);  // [32][S]
    const GroupRec R = rec[blockIdx.x];
    const int nq = R.q1 - R.q0;
    const int L = R.L, nw = (L + 31) >> 5;
    const int64_t base = loff[blockIdx.x];
    const uint32_t *mk = mask + base + lane;  // word k of this lane's query at mk[32 * k]
    const int32_t *ul = list + base;
    const bool have = lane < nq;
    int32_t qid = 0;
    int64_t rbase = 0;
    int len = 0;
    double qxl = 0.0, qyl = 0.0, qzl = 0.0;
    if (have) {
        const PtRec c = load_pt(P.a, R.q0 + lane);
        qid = c.id;
        qxl = c.x, qyl = c.y, qzl = c.z;
        rbase = rowptr[qid];
        len = (int)(rowptr[qid + 1] - rbase);
    }
    // (2) staging loads first (they overlap the walk)
    constexpr int SU = 3;
    PtRec sp[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) {
        const int t = u * 128 + tid;
        sp[u] = load_pt(P.a, ul[t < L ? t : 0]);
    }
    {
        // (1) this warp's quarter of the words
        const int k0 = (nw * warp) >> 2, k1 = (nw * (warp + 1)) >> 2;
        uint16_t *my = ent + (size_t)lane * S;
        int n = 0;
        if (have)
            for (int k = 0; k < k0; ++k) n += __popc(mk[32 * k]);
        const int kend = have ? k1 : k0;
        int k = k0;
        uint32_t w = (k < kend) ? mk[32 * k] : 0u;
        uint32_t wnext = (k + 1 < kend) ? mk[32 * (k + 1)] : 0u;
        while (__any_sync(0xffffffffu, k < kend)) {
#pragma unroll 2
            for (int u = 0; u < 2; ++u) {
                const bool z = (w == 0);
                const int b1 = __clz(w) & 31;
                const uint32_t w1 = w ^ (0x80000000u >> b1);
                const int b2 = __clz(w1) & 31;
                const bool two = !z && (w1 != 0);
                // (predicated: the next quarter's warp owns the slots past this quarter's end)
                if (!z) my[min(n, S - 1)] = (uint16_t)(32 * k + b1);
                if (two) my[min(n + 1, S - 1)] = (uint16_t)(32 * k + b2);
                n += z ? 0 : (two ? 2 : 1);
                const bool step = z && (k < kend);
                const uint32_t wl = (step && k + 2 < kend) ? mk[32 * (k + 2)] : 0u;
                w = z ? wnext : (two ? (w1 ^ (0x80000000u >> b2)) : 0u);
                wnext = step ? wl : wnext;
                k = step ? k + 1 : k;
            }
        }
        if (warp == 3 && have && n != len) atomicOr(&stats[2], 1);  // count/fill agreement (always-on invariant)
    }
#pragma unroll
    for (int u = 0; u < SU; ++u) {
        const int t = u * 128 + tid;
        if (t < L) {
            ux[t] = sp[u].x;
            uy[t] = sp[u].y;
            if (DIM == 3) uz[t] = sp[u].z;
            uid[t] = sp[u].id;
        }
    }
    for (int t0 = SU * 128; t0 < L; t0 += 4 * 128) {
        PtRec c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = t0 + u * 128 + tid;
            c[u] = load_pt(P.a, ul[t < L ? t : 0]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = t0 + u * 128 + tid;
            if (t < L) {
                ux[t] = c[u].x;
                uy[t] = c[u].y;
                if (DIM == 3) uz[t] = c[u].z;
                uid[t] = c[u].id;
            }
        }
    }
    __syncthreads();
    const double rmin = g.rmin;
#ifdef TF_DEBUG_CHECKS
    const double r2 = g.r2;
#endif
    for (int i = warp; i < nq; i += 4) {
        const uint16_t *my = ent + (size_t)i * S;
        const int li = __shfl_sync(0xffffffffu, len, i);
        const int64_t bi = __shfl_sync(0xffffffffu, rbase, i);
        const int32_t qi = __shfl_sync(0xffffffffu, qid, i);
        const double qx = __shfl_sync(0xffffffffu, qxl, i), qy = __shfl_sync(0xffffffffu, qyl, i);
        const double qz = (DIM == 3) ? __shfl_sync(0xffffffffu, qzl, i) : 0.0;
        const bool longrow = li > S - 2;
        const int lr = longrow ? 0 : li;
        double cx[ROUNDS], cy[ROUNDS], cz[ROUNDS];
        int32_t cid[ROUNDS];
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int e = 32 * r + lane;
            const int t = (e < lr) ? my[e] : 0;
            cx[r] = ux[t];
            cy[r] = uy[t];
            cz[r] = (DIM == 3) ? uz[t] : 0.0;
            cid[r] = uid[t];
        }
        double hsum = 0.0;
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int e = 32 * r + lane;
            if (e < lr) {
                const double d2 = pair_d2<DIM>(qx, qy, qz, cx[r], cy[r], cz[r]);
                const double w = weight_of(rmin, d2);
                cols[bi + e] = cid[r];
                vals[bi + e] = w;
                hsum += w;
                TF_DCHECK(d2 < r2);
            }
        }
        for (int e = 32 * ROUNDS + lane; e < lr; e += 32) {
            const int t = my[e];
            const double d2 = pair_d2<DIM>(qx, qy, qz, ux[t], uy[t], (DIM == 3) ? uz[t] : 0.0);
            const double w = weight_of(rmin, d2);
            cols[bi + e] = uid[t];
            vals[bi + e] = w;
            hsum += w;
            TF_DCHECK(d2 < r2);
        }
        if (longrow) {
            // rows longer than the lists (dense clusters): lane = mask word, each lane emits its bits
            int done = 0;
            for (int k0 = 0; k0 < nw; k0 += 32) {
                const int k = k0 + lane;
                uint32_t w = (k < nw) ? mask[base + 32 * k + i] : 0u;
                const int cnt = __popc(w);
                int inc = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += v;
                }
                int e = done + inc - cnt;
                while (w) {
                    const int b = __clz(w);
                    const int t = 32 * k + b;
                    const double d2 = pair_d2<DIM>(qx, qy, qz, ux[t], uy[t], (DIM == 3) ? uz[t] : 0.0);
                    const double wt = weight_of(rmin, d2);
                    cols[bi + e] = uid[t];
                    vals[bi + e] = wt;
                    hsum += wt;
                    TF_DCHECK(d2 < r2);
                    ++e;
                    w ^= 0x80000000u >> b;
                }
                done += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
        if (lane == 0) hs[qi] = hsum;
    }
}

template <int DIM, int ROUNDS>
tf_status launch_cl_fill4(const SortedPtsView &P, const Grid &g, const GroupRec *rec, const int64_t *loff, int32_t G,
                          int LPmax, int S, const int32_t *list, const uint32_t *mask, tf_filter_s *h, int32_t *stats,
                          cudaStream_t s) {
    const size_t smem = (size_t)LPmax * ((DIM == 3 ? 24 : 16) + 4) + (size_t)32 * S * sizeof(uint16_t);
    auto kern = k_cl_fill4<DIM, ROUNDS>;
    TF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)G, 128, smem, s>>>(P, g, rec, loff, LPmax, S, list, mask, h->rowptr, h->cols, h->vals, h->hs,
                                        stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

// ------------------------------------------------------------------ a7: fill, block per group
// One block of kFillBWarps warps per group (kGroupQ = 32 queries). The group's sorted union is
// staged in shared memory once -- exact fp64 coordinates and ids --, so every entry's candidate
// data is a shared-memory load instead of a global gather (the warp-per-group fill was bound by
// the L1 wavefronts of those gathers). Warp 0 expands the lanes' mask words into candidate lists
// (lane = query, as k_cl_fill) while the other warps stage the union; then warp w writes the rows
// of queries w, w + kFillBWarps, ... (lane = entry; two rows per pass, kFillRounds rounds each in
// flight): the oracle's d^2 and weight, coalesced int32 / fp64 stores, Hs by a fixed-order lane
// reduction. Shared memory: union x, y, z [LPmax] fp64 + ids [LPmax] int32 + masks [32][MS] + lists
// [32][S] uint16.
constexpr int kFillBWarps = 4;

template <int DIM>
__global__ void __launch_bounds__(kFillBWarps * 32) k_cl_fill_b(SortedPtsView P, Grid g,
                                                                const GroupRec *__restrict__ rec,
                                                                const int64_t *__restrict__ loff, int LPmax, int MS,
                                                                int S, const int32_t *__restrict__ list,
                                                                const uint32_t *__restrict__ mask,
                                                                const int64_t *__restrict__ rowptr,
                                                                int32_t *__restrict__ cols, double *__restrict__ vals,
                                                                double *__restrict__ hs, int32_t *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int T = kFillBWarps * 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double *ux = reinterpret_cast<double *>(smem_raw);
    double *uy = ux + LPmax;
    double *uz = uy + LPmax;
    int32_t *uid = reinterpret_cast<int32_t *>(uz + ((DIM == 3) ? LPmax : 0));
    uint32_t *sm = reinterpret_cast<uint32_t *>(uid + LPmax);  // [32][MS]
    uint16_t *ent = reinterpret_cast<uint16_t *>(sm + 32 * MS);  // [32][S]
    __shared__ int32_t s_len[32];
    __shared__ int64_t s_base[32];
    __shared__ int32_t s_qid[32];
    const GroupRec R = rec[blockIdx.x];
    const int L = R.L, LP = (L + 31) & ~31, nw = LP >> 5;
    const int64_t base = loff[blockIdx.x];
    const int nq = R.q1 - R.q0;
    if (warp == 0) {
        // masks of the group, transposed to [lane][word] (odd stride MS > nw, the padding zero)
        for (int k0 = 0; k0 < MS; k0 += 4) {
            uint32_t m[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) m[u] = (k0 + u < nw) ? mask[base + 32 * (k0 + u) + lane] : 0u;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k0 + u < MS) sm[lane * MS + k0 + u] = m[u];
        }
        const int q = R.q0 + lane;
        const bool have = lane < nq;
        int32_t qid = 0;
        int64_t rbase = 0;
        int len = 0;
        if (have) {
            qid = P.id[q];
            rbase = rowptr[qid];
            len = (int)(rowptr[qid + 1] - rbase);
        }
        s_len[lane] = len;
        s_base[lane] = rbase;
        s_qid[lane] = qid;
        __syncwarp();
        // branch-free walk of the lane's words (two set bits or one word step per iteration)
        const uint32_t *mw = sm + lane * MS;
        uint16_t *my = ent + (size_t)lane * S;
        int n = 0, k = 0;
        uint32_t w = mw[0];
        const int kend = have ? nw : 0;
        while (__any_sync(0xffffffffu, k < kend)) {
#pragma unroll 2
            for (int u = 0; u < 2; ++u) {
                const bool z = (w == 0);
                const int b1 = __clz(w) & 31;
                const uint32_t w1 = w ^ (0x80000000u >> b1);
                const int b2 = __clz(w1) & 31;
                const bool two = !z && (w1 != 0);
                my[min(n, S - 1)] = (uint16_t)(32 * k + b1);
                my[min(n + 1, S - 1)] = (uint16_t)(32 * k + b2);
                n += z ? 0 : (two ? 2 : 1);
                const uint32_t wn = mw[min(k + 1, MS - 1)];
                w = z ? wn : (two ? (w1 ^ (0x80000000u >> b2)) : 0u);
                k = z ? min(k + 1, nw) : k;
            }
        }
        if (have && n != len) atomicOr(&stats[2], 1);  // count/fill agreement (always-on invariant)
    } else {
        // the union's exact coordinates and ids, staged once for the whole group
        for (int t0 = (warp - 1) * 32; t0 < L; t0 += 4 * (T - 32)) {
            int p[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = t0 + u * (T - 32) + lane;
                p[u] = (t < L) ? list[base + t] : -1;
            }
            double xv[4], yv[4], zv[4];
            int32_t iv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int pp = p[u] < 0 ? 0 : p[u];
                xv[u] = P.x[pp];
                yv[u] = P.y[pp];
                zv[u] = (DIM == 3) ? P.z[pp] : 0.0;
                iv[u] = P.id[pp];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = t0 + u * (T - 32) + lane;
                if (t < L) {
                    ux[t] = xv[u];
                    uy[t] = yv[u];
                    if (DIM == 3) uz[t] = zv[u];
                    uid[t] = iv[u];
                }
            }
        }
    }
    __syncthreads();
    const double rmin = g.rmin;
#ifdef TF_DEBUG_CHECKS
    const double r2 = g.r2;
#endif
    for (int i0 = 2 * warp; i0 < nq; i0 += 2 * kFillBWarps) {
        int li[2];
        bool longrow[2];
        int32_t qi[2];
        int64_t bi[2];
        double qx[2], qy[2], qz[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = min(i0 + h, nq - 1);
            li[h] = (i0 + h < nq) ? s_len[i] : 0;
            longrow[h] = li[h] > S - 2;
            if (longrow[h]) li[h] = 0;
            bi[h] = s_base[i];
            qi[h] = s_qid[i];
            qx[h] = P.x[R.q0 + i];
            qy[h] = P.y[R.q0 + i];
            qz[h] = (DIM == 3) ? P.z[R.q0 + i] : 0.0;
        }
        double cx[2][kFillRounds], cy[2][kFillRounds], cz[2][kFillRounds];
        int32_t cid[2][kFillRounds];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int r = 0; r < kFillRounds; ++r) {
                const int e = 32 * r + lane;
                const int t = (e < li[h]) ? ent[(size_t)(i0 + h) * S + e] : 0;
                cx[h][r] = ux[t];
                cy[h][r] = uy[t];
                cz[h][r] = (DIM == 3) ? uz[t] : 0.0;
                cid[h][r] = uid[t];
            }
        double hsum[2] = {0.0, 0.0};
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int r = 0; r < kFillRounds; ++r) {
                const int e = 32 * r + lane;
                if (e < li[h]) {
                    const double d2 = pair_d2<DIM>(qx[h], qy[h], qz[h], cx[h][r], cy[h][r], cz[h][r]);
                    const double w = weight_of(rmin, d2);
                    cols[bi[h] + e] = cid[h][r];
                    vals[bi[h] + e] = w;
                    hsum[h] += w;
                    TF_DCHECK(d2 < r2);
                }
            }
#pragma unroll
        for (int h = 0; h < 2; ++h)
            for (int e = 32 * kFillRounds + lane; e < li[h]; e += 32) {
                const int t = ent[(size_t)(i0 + h) * S + e];
                const double d2 = pair_d2<DIM>(qx[h], qy[h], qz[h], ux[t], uy[t], (DIM == 3) ? uz[t] : 0.0);
                const double w = weight_of(rmin, d2);
                cols[bi[h] + e] = uid[t];
                vals[bi[h] + e] = w;
                hsum[h] += w;
                TF_DCHECK(d2 < r2);
            }
        // rows longer than the lists: lane = mask word of the row (word-parallel path)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!longrow[h]) continue;
            const int i = i0 + h;
            int done = 0;
            for (int k0 = 0; k0 < nw; k0 += 32) {
                const int k = k0 + lane;
                uint32_t w = (k < nw) ? sm[i * MS + k] : 0u;
                const int c = __popc(w);
                int inc = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += v;
                }
                int e = done + inc - c;
                while (w) {
                    const int b = __clz(w);
                    const int t = 32 * k + b;
                    const double d2 = pair_d2<DIM>(qx[h], qy[h], qz[h], ux[t], uy[t], (DIM == 3) ? uz[t] : 0.0);
                    const double wt = weight_of(rmin, d2);
                    cols[bi[h] + e] = uid[t];
                    vals[bi[h] + e] = wt;
                    hsum[h] += wt;
                    ++e;
                    w ^= 0x80000000u >> b;
                }
                done += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            hsum[0] += __shfl_xor_sync(0xffffffffu, hsum[0], o);
            hsum[1] += __shfl_xor_sync(0xffffffffu, hsum[1], o);
        }
        if (lane == 0) {
            hs[qi[0]] = hsum[0];
            if (i0 + 1 < nq) hs[qi[1]] = hsum[1];
        }
    }
}

template <int DIM>
tf_status launch_cl_fill_b(const SortedPtsView &P, const Grid &g, const GroupRec *rec, const int64_t *loff, int32_t G,
                           int LPmax, int MS, int S, const int32_t *list, const uint32_t *mask, tf_filter_s *h,
                           int32_t *stats, cudaStream_t s) {
    const size_t smem = (size_t)LPmax * ((DIM == 3 ? 24 : 16) + 4) + (size_t)32 * MS * 4 + (size_t)32 * S * 2;
    auto kern = k_cl_fill_b<DIM>;
    TF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)G, kFillBWarps * 32, smem, s>>>(P, g, rec, loff, LPmax, MS, S, list, mask, h->rowptr, h->cols,
                                                     h->vals, h->hs, stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

template <int DIM>
tf_status launch_cl_count(const SortedPtsView &P, const Grid &g, const GroupRec *rec, const int64_t *loff, int32_t G,
                          int LPmax, int32_t *list, uint32_t *mask, int32_t *counts, int32_t *stats, cudaStream_t s) {
    const size_t smem = (size_t)5 * LPmax * sizeof(uint32_t);
    auto kern = k_cl_count<DIM>;
    TF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)G, kCountWarps * 32, smem, s>>>(P, g, rec, loff, LPmax, list, mask, counts, stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

template <int DIM, int WARPS>
tf_status launch_cl_fill(const SortedPtsView &P, const Grid &g, const GroupRec *rec, const int64_t *loff, int32_t G,
                         int MS, int S, const int32_t *list, const uint32_t *mask, tf_filter_s *h, int32_t *stats,
                         cudaStream_t s) {
    const size_t smem = (size_t)WARPS * ((size_t)32 * MS * 4 + (size_t)32 * S * 2);
    auto kern = k_cl_fill<DIM, WARPS>;
    TF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)(((int64_t)G * kHalves + WARPS - 1) / WARPS), WARPS * 32, smem, s>>>(P, g, rec, loff, G, MS, S, list, mask,
                                                                     h->rowptr, h->cols, h->vals, h->hs, stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

}  // namespace

// The group path of the cell-list build (rows a5-a7 after build.cu's a2-a4). *done = false
// (TF_OK) when the largest union exceeds kMaxUnion: the caller then runs the per-bin kernels.
tf_status build_cell_list_groups(const SortedPtsView &P, const uint32_t *sorted_keys, const Grid &g, int64_t n,
                                 cudaStream_t s, tf_filter_s *h, bool *done) {
    *done = false;
    const int dim = g.dim;
    const int nxb = (g.nb[0] + kUnitBins - 1) / kUnitBins;
    const int64_t U = (int64_t)g.nb[1] * g.nb[2] * nxb;
    const int64_t Gmax = U + n / 32 + 1;
    if (Gmax >= (int64_t)INT32_MAX) return TF_OK;
    DeviceInfo di;
    TF_TRY(device_info(&di));
    const int threads = 256;
    const unsigned gridU = (unsigned)std::min<int64_t>((U + threads) / threads, (int64_t)di.sms * 8);

    // units -> group offsets -> group records + padded union sizes -> union offsets
    DevBuf<int32_t> ng, goff, lp, stats;
    DevBuf<GroupRec> rec;
    DevBuf<int64_t> loff;
    TF_TRY(ng.alloc(U + 1, s, "unit group counts"));
    TF_TRY(goff.alloc(U + 2, s, "unit group offsets"));
    TF_TRY(rec.alloc(Gmax, s, "group records"));
    TF_TRY(lp.alloc(Gmax, s, "group union sizes"));
    TF_TRY(loff.alloc(Gmax + 1, s, "group union offsets"));
    TF_TRY(stats.alloc(4, s, "build stats"));
    TF_CUDA_TRY(cudaMemsetAsync(stats.p, 0, 4 * sizeof(int32_t), s));
    TF_CUDA_TRY(cudaMemsetAsync(lp.p, 0, Gmax * sizeof(int32_t), s));
    k_cl_units<<<gridU, threads, 0, s>>>(P.cs, g, nxb, U, ng.p);
    TF_LAUNCH_CHECK();
    TF_TRY(exclusive_scan_i32_i32(ng.p, goff.p, U + 1, s));
    if (dim == 3) k_cl_groups<3><<<gridU, threads, 0, s>>>(P.cs, sorted_keys, g, nxb, U, goff.p, rec.p, lp.p, stats.p);
    else k_cl_groups<2><<<gridU, threads, 0, s>>>(P.cs, sorted_keys, g, nxb, U, goff.p, rec.p, lp.p, stats.p);
    TF_LAUNCH_CHECK();
    TF_TRY(exclusive_scan_i32_i64(lp.p, loff.p, Gmax, s));
    int32_t hG = 0, hmax = 0;
    int64_t hTot = 0;
    TF_CUDA_TRY(cudaMemcpyAsync(&hG, goff.p + U, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaMemcpyAsync(&hmax, stats.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaMemcpyAsync(&hTot, loff.p + Gmax, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    build_trace().mark("groups+sync", s);
    h->info.max_candidates = hmax;
    if (hmax > kMaxUnion || hG <= 0) return TF_OK;  // per-bin kernels take it
    const int LPmax = (hmax + 31) & ~31;

    // a5 count: sorted unions + mask words + row lengths
    DevBuf<int32_t> list, counts;
    DevBuf<uint32_t> mask;
    TF_TRY(list.alloc(hTot, s, "group unions"));
    TF_TRY(mask.alloc((size_t)kHalves * hTot, s, "group masks"));
    TF_TRY(counts.alloc(n, s, "row counts"));
    if (dim == 3) TF_TRY((launch_cl_count<3>(P, g, rec.p, loff.p, hG, LPmax, list.p, mask.p, counts.p, stats.p, s)));
    else TF_TRY((launch_cl_count<2>(P, g, rec.p, loff.p, hG, LPmax, list.p, mask.p, counts.p, stats.p, s)));
    build_trace().mark("count", s);

    // a6 row pointers + nnz readback
    TF_TRY(dalloc(&h->rowptr, n + 3, s, "rowptr (+2 padding for 16-byte bulk copies)"));
    TF_TRY(exclusive_scan_i32_i64(counts.p, h->rowptr, n, s));
    int64_t nnz = 0;
    int32_t maxrow = 0;
    TF_CUDA_TRY(cudaMemcpyAsync(&nnz, h->rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaMemcpyAsync(&maxrow, stats.p + 3, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    build_trace().mark("scan+sync", s);
    if (nnz < n || nnz < 0) {
        set_error("internal: nnz %lld < n %lld", (long long)nnz, (long long)n);
        return TF_ERR_CUDA;
    }
    h->nnz = nnz;
    h->max_row_hint = maxrow;

    // a7 fill
    TF_TRY(dalloc(&h->cols, nnz + 4, s, "cols (nnz int32, +4 padding for 16-byte bulk copies)"));
    TF_TRY(dalloc(&h->vals, nnz + 4, s, "vals (nnz fp64, +4 padding)"));
    TF_TRY(dalloc(&h->hs, n, s, "Hs"));
    build_trace().mark("alloc_csr", s);
    // per-lane list stride S >= longest row (capped: longer rows take the word-parallel path),
    // S = 2 mod 4 uint16 so lanes at equal list positions hit different banks; mask stride MS odd
    int S = std::max(2, (std::min(maxrow, kListCap) + 3) & ~1);  // +2 slots for the walk's idle writes
    if ((S & 3) == 0) S += 2;
    const int MS = (LPmax / 32 + 1) | 1;
    const size_t per_warp = (size_t)32 * MS * 4 + (size_t)32 * S * 2;
    // the block-per-group fill (union staged in shared memory) measured 8.90 vs 8.60 ms at config 5
    // and 0.42 vs 0.47 ms at config 4: opt-in (TOPOFILT_CL_FILL=block, benchmarks and tests)
    const char *fk = getenv("TOPOFILT_CL_FILL");
    const size_t smem4 = (size_t)LPmax * ((dim == 3 ? 24 : 16) + 4) + (size_t)32 * S * 2;
    // block-per-group fill with the union staged in shared memory: measured faster only for small
    // unions (config 4: 366 vs 402 us; config 5: 8.9 vs 6.65 ms), so it takes the builds whose blocks
    // need <= 12 KB (2D neighbourhoods); TOPOFILT_CL_FILL=split / walk3 force either kernel
    const bool want4 = fk ? !strcmp(fk, "split") : (smem4 <= 12 * 1024);
    if (kGroupQ == 32 && want4 && smem4 <= di.smem_optin) {
        const int rounds = std::min(3, (std::min(maxrow, 96) + 31) / 32);
#define TF_FILL4(D, R) TF_TRY((launch_cl_fill4<D, R>(P, g, rec.p, loff.p, hG, LPmax, S, list.p, mask.p, h, stats.p, s)))
        if (dim == 3) {
            if (rounds >= 3) TF_FILL4(3, 3);
            else if (rounds == 2) TF_FILL4(3, 2);
            else TF_FILL4(3, 1);
        } else {
            if (rounds >= 3) TF_FILL4(2, 3);
            else if (rounds == 2) TF_FILL4(2, 2);
            else TF_FILL4(2, 1);
        }
#undef TF_FILL4
    } else if (!(fk && (!strcmp(fk, "block") || !strcmp(fk, "walk") || !strcmp(fk, "rows")))) {
        // default: the walk fill with the mask words read from L1 and one row at a time in flight
        const int rounds = std::min(3, (std::min(maxrow, 96) + 31) / 32);
#define TF_FILL3(D, R) TF_TRY((launch_cl_fill3<D, R>(P, g, rec.p, loff.p, hG, S, list.p, mask.p, h, stats.p, s)))
        if (dim == 3) {
            if (rounds >= 3) TF_FILL3(3, 3);
            else if (rounds == 2) TF_FILL3(3, 2);
            else TF_FILL3(3, 1);
        } else {
            if (rounds >= 3) TF_FILL3(2, 3);
            else if (rounds == 2) TF_FILL3(2, 2);
            else TF_FILL3(2, 1);
        }
#undef TF_FILL3
    } else if (kGroupQ == 32 && fk && !strcmp(fk, "rows")) {
        // default: row-by-row fill; list stride = longest row rounded up to 32 (capped), rounds in
        // flight from the longest row
        const int S2 = std::max(32, (std::min(maxrow, 1024) + 31) & ~31);
        const int rounds = std::min(3, (std::min(maxrow, 96) + 31) / 32);
#define TF_FILL2(D, R) TF_TRY((launch_cl_fill2<D, R>(P, g, rec.p, loff.p, hG, S2, list.p, mask.p, h, stats.p, s)))
        if (dim == 3) {
            if (rounds >= 3) TF_FILL2(3, 3);
            else if (rounds == 2) TF_FILL2(3, 2);
            else TF_FILL2(3, 1);
        } else {
            if (rounds >= 3) TF_FILL2(2, 3);
            else if (rounds == 2) TF_FILL2(2, 2);
            else TF_FILL2(2, 1);
        }
#undef TF_FILL2
    } else {
    const size_t smem_b = (size_t)LPmax * ((dim == 3 ? 24 : 16) + 4) + (size_t)32 * MS * 4 + (size_t)32 * S * 2;
    if (kGroupQ == 32 && fk && !strcmp(fk, "block") && smem_b <= di.smem_optin) {
        if (dim == 3) TF_TRY((launch_cl_fill_b<3>(P, g, rec.p, loff.p, hG, LPmax, MS, S, list.p, mask.p, h, stats.p, s)));
        else TF_TRY((launch_cl_fill_b<2>(P, g, rec.p, loff.p, hG, LPmax, MS, S, list.p, mask.p, h, stats.p, s)));
    } else {
    int fw = env_int("TOPOFILT_CL_FILL_WARPS", 4);  // tuning knob (benchmarks only)
    while (fw > 1 && (size_t)fw * per_warp > di.smem_optin) fw >>= 1;
    if (dim == 3) {
        if (fw >= 4) TF_TRY((launch_cl_fill<3, 4>(P, g, rec.p, loff.p, hG, MS, S, list.p, mask.p, h, stats.p, s)));
        else if (fw >= 2) TF_TRY((launch_cl_fill<3, 2>(P, g, rec.p, loff.p, hG, MS, S, list.p, mask.p, h, stats.p, s)));
        else TF_TRY((launch_cl_fill<3, 1>(P, g, rec.p, loff.p, hG, MS, S, list.p, mask.p, h, stats.p, s)));
    } else {
        if (fw >= 4) TF_TRY((launch_cl_fill<2, 4>(P, g, rec.p, loff.p, hG, MS, S, list.p, mask.p, h, stats.p, s)));
        else if (fw >= 2) TF_TRY((launch_cl_fill<2, 2>(P, g, rec.p, loff.p, hG, MS, S, list.p, mask.p, h, stats.p, s)));
        else TF_TRY((launch_cl_fill<2, 1>(P, g, rec.p, loff.p, hG, MS, S, list.p, mask.p, h, stats.p, s)));
    }
    }
    }
    build_trace().mark("fill", s);
    int32_t flag = 0;
    TF_CUDA_TRY(cudaMemcpyAsync(&flag, stats.p + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    build_trace().mark("stats+sync", s);
    if (flag != 0) {
        set_error("internal: group fill disagreed with the count pass (flag %d)", flag);
        return TF_ERR_CUDA;
    }
    h->info.groups = hG;
    *done = true;
    return TF_OK;
}

}  // namespace tf
