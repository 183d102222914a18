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
//                that sorted list for the fill as 16-bit run codes (run << 12 | offset in the run:
//                sorted position = run start + offset), (4) sweeps it: lane = query, every union
//                candidate tested with packed fp32x2 math in EDM form (R4c), one sign bit per test
//                funnel-shifted (SHF.L.W) into a per-query 32-bit mask word, band candidates caught
//                by a running unsigned minimum (VIMNMX3) and decided by the exact fp64 test; (5)
//                stores the words (coalesced, word k of query q at [k][q]) and the row length =
//                popcount;
//   k_cl_fill3   warp per group (the default for 3D-sized unions): lane = query walks its mask
//                words straight from L1 (branch-free, two bits per step, next word loaded a step
//                ahead) into a list of candidate indices, then lane = entry writes the rows one at a
//                time: the candidate's whole point (x, y, z, id) in ONE 256-bit load of the AoS copy
//                of the sorted centroids, the oracle's d^2 and weight, coalesced int32 / fp64 stores,
//                Hs by a fixed-order lane reduction. 64 registers, 5.8 KB of shared memory per warp:
//                8 blocks of 4 warps per SM;
//   k_cl_fill4   block per group (small unions, i.e. 2D): the walk is split over the four warps (a
//                quarter of every query's words each), the union's exact coordinates are staged in
//                shared memory once, warp w writes rows w, w + 4, ...
// No pair is tested twice: the set bits ARE the accepted pairs.
// The per-bin kernels of build.cu (k_count / k_fill) stay as TF_BUILD_CELL_LIST_BINS and as the
// fallback for unions beyond kMaxUnion (or runs beyond kMaxRun). Measured: the
// count is bound by shared-memory wavefronts (the sweep's broadcast candidate loads and the sort),
// the fill by the L2 -> L1 sectors of its per-entry point gathers (one 32-byte sector per entry).
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
constexpr int kListCap = 256;     // per-lane list capacity of the fills; longer rows take the word-parallel path
// The sorted union handed from the count to the fill is a list of 16-bit codes (run << kRunShift) |
// offset-in-run (sorted position = run start + offset): half the bytes and sectors of a position list.
constexpr int kRunShift = 12;
constexpr int kMaxRun = 1 << kRunShift;  // longest union run the codes can address
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

// Warp per unit, lane per group: the unit's group records and padded union sizes; stats[0] = max union,
// stats[1] = longest union run.
template <int DIM>
__global__ void __launch_bounds__(256) k_cl_groups(const int32_t *__restrict__ cs, const uint32_t *__restrict__ keys,
                                                   Grid g, int nxb, int64_t U, const int32_t *__restrict__ goff,
                                                   GroupRec *__restrict__ rec, int32_t *__restrict__ lp,
                                                   int32_t *__restrict__ stats) {
    constexpr int NR = (DIM == 3) ? 9 : 3;
    int best = 0, longest = 0;
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = wid; u < U; u += nwarp) {
        int32_t s, e;
        unit_range(u, g, nxb, cs, s, e);
        const int32_t row = (int32_t)(u / nxb);
        // warp per unit, lane per group of the unit
        for (int32_t q0 = s + lane * kGroupQ; q0 < e; q0 += 32 * kGroupQ) {
            const int32_t gi = goff[u] + (q0 - s) / kGroupQ;
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
                longest = max(longest, rl);
            }
            G.L = L;
            rec[gi] = G;
            lp[gi] = (L + 31) & ~31;
            best = max(best, L);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
        longest = max(longest, __shfl_xor_sync(0xffffffffu, longest, o));
    }
    if ((threadIdx.x & 31) == 0 && best > 0) atomicMax(&stats[0], best), atomicMax(&stats[1], longest);
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
                                                                uint16_t *__restrict__ list, uint32_t *__restrict__ mask,
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
    // (2b) stage (id - lo, run code of the sorted-SoA position) in run order
    {
        int r = 0;
        for (int t0 = 0; t0 < L; t0 += 4 * T) {
            int id[4];
            uint32_t cd[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = t0 + u * T + tid;
                while (r < NR - 1 && t >= run_x[r + 1]) ++r;
                cd[u] = ((uint32_t)r << kRunShift) | (uint32_t)(t - run_x[r]);
                id[u] = (t < L) ? P.id[run_s[r] + (t - run_x[r])] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = t0 + u * T + tid;
                if (t < L) KA[t] = (uint32_t)(id[u] - lo), VA[t] = cd[u];
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
                    const uint32_t cd = Q4[t];
                    list[base + t] = (uint16_t)cd;
                    const PtRec c = load_pt(P.a, run_s[cd >> kRunShift] + (int)(cd & (kMaxRun - 1)));
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
                        const uint32_t cd = Q4[t];
                        const PtRec c = load_pt(P.a, run_s[cd >> kRunShift] + (int)(cd & (kMaxRun - 1)));
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

// ------------------------------------------------------------------ a7: fill, warp per group, masks from L1
// k_cl_fill with two changes for occupancy (the fill is latency-bound at 5 blocks of 4 warps per SM):
// the walk reads each lane's mask words straight from global memory (word k of query q at [k][q]:
// the group's words stay L1-resident; the next word is loaded one step ahead), so no transposed mask
// copy in shared memory (10.5 -> 5.8 KB per warp at config 5); rows are written one at a time with
// ROUNDS rounds in flight, which fits 64 registers (8 blocks per SM).
#ifndef TF_CL_FILL3_WARPS
#define TF_CL_FILL3_WARPS 4
#endif
constexpr int kFill3Warps = TF_CL_FILL3_WARPS;  // warps per block: consecutive groups, i.e. neighbours along x
#ifndef TF_CL_FILL3_PREFETCH
#define TF_CL_FILL3_PREFETCH 1
#endif
#ifndef TF_CL_FILL3_MINB
#define TF_CL_FILL3_MINB (32 / TF_CL_FILL3_WARPS)
#endif
template <int DIM, int ROUNDS>
__global__ void __launch_bounds__(kFill3Warps * 32, TF_CL_FILL3_MINB)
    k_cl_fill3(SortedPtsView P, Grid g, const GroupRec *__restrict__ rec, const int64_t *__restrict__ loff, int32_t G,
               int S, const uint16_t *__restrict__ list, const uint32_t *__restrict__ mask,
               const int64_t *__restrict__ rowptr, int32_t *__restrict__ cols, double *__restrict__ vals,
               double *__restrict__ hs, int32_t *__restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t wi = (int32_t)blockIdx.x * kFill3Warps + warp;
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
    const uint16_t *ul = list + base;
    // run starts of the union (code -> sorted position)
    __shared__ int32_t s_run[kFill3Warps][16];
    int32_t *srun = s_run[warp];
    {
        constexpr int NR = (DIM == 3) ? 9 : 3;
        int rs = 0, rl = 0;
        if (lane < NR) group_run<DIM>(lane, R, g, P.cs, rs, rl);
        if (lane < 16) srun[lane] = rs;
    }
    auto pos_of = [&](uint32_t cd) { return srun[cd >> kRunShift] + (int)(cd & (kMaxRun - 1)); };
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
#if TF_CL_FILL3_PREFETCH
    // the group's mask block ([word][query], 128 bytes per word) comes from DRAM: touch every word
    // line now, all in flight at once, instead of meeting the misses one by one along the walk
    for (int k = lane; k < nw; k += 32)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(mask + kHalves * base + (size_t)WS * k + 32 * half));
    for (int t = 64 * lane; t < L; t += 64 * 32)  // and the union's code list (128 bytes = 64 codes per line)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(ul + t));
#endif
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
            c[r] = load_pt(P.a, pos_of(ul[(e < lr) ? my[e] : 0]));
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
            const PtRec cc = load_pt(P.a, pos_of(ul[my[e]]));
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
                    const PtRec cc = load_pt(P.a, pos_of(ul[32 * k + b]));
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
                          int S, const uint16_t *list, const uint32_t *mask, tf_filter_s *h, int32_t *stats,
                          cudaStream_t s) {
    const size_t smem = (size_t)kFill3Warps * 32 * S * sizeof(uint16_t);
    auto kern = k_cl_fill3<DIM, ROUNDS>;
    TF_TRY(allow_dynamic_smem(kern, smem));
    kern<<<(unsigned)(((int64_t)G * kHalves + kFill3Warps - 1) / kFill3Warps), kFill3Warps * 32, smem, s>>>(
        P, g, rec, loff, G, S, list, mask, h->rowptr, h->cols, h->vals, h->hs, stats);
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
                                                  const uint16_t *__restrict__ list, const uint32_t *__restrict__ mask,
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
    const uint16_t *ul = list + base;
    // run starts of the union (code -> sorted position), one copy per warp (no block barrier)
    __shared__ int32_t s_run[4][16];
    int32_t *srun = s_run[warp];
    {
        constexpr int NR = (DIM == 3) ? 9 : 3;
        int rs = 0, rl = 0;
        if (lane < NR) group_run<DIM>(lane, R, g, P.cs, rs, rl);
        if (lane < 16) srun[lane] = rs;
        __syncwarp();
    }
    auto pos_of = [&](uint32_t cd) { return srun[cd >> kRunShift] + (int)(cd & (kMaxRun - 1)); };
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
    for (int k = tid; k < nw; k += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(mask + base + 32 * k));
    // (2) staging loads first (they overlap the walk)
    constexpr int SU = 3;
    PtRec sp[SU];
#pragma unroll
    for (int u = 0; u < SU; ++u) {
        const int t = u * 128 + tid;
        sp[u] = load_pt(P.a, pos_of(ul[t < L ? t : 0]));
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
            c[u] = load_pt(P.a, pos_of(ul[t < L ? t : 0]));
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
    // Hs: the lanes' partial sums of a warp's (up to 8) rows are parked in shared memory and reduced
    // together after the rows are written (a 5-step shuffle tree per row was 15% of the kernel's
    // instructions on short 2D rows); fixed order, so Hs is reproducible run to run
    __shared__ double s_hs[4][8][33];
    for (int i = warp; i < nq; i += 4) {
        const uint16_t *my = ent + (size_t)i * S;
        const int li = __shfl_sync(0xffffffffu, len, i);
        const int64_t bi = __shfl_sync(0xffffffffu, rbase, i);
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
        s_hs[warp][i >> 2][lane] = hsum;
    }
    __syncwarp();
    {
        // lane = (row j of this warp, quarter): 8 partials in lane order, then the four quarters
        const int j = lane >> 2, part = lane & 3, i = warp + 4 * j;
        double t = 0.0;
        if (i < nq) {
#pragma unroll
            for (int k = 0; k < 8; ++k) t += s_hs[warp][j][8 * part + k];
        }
        t += __shfl_xor_sync(0xffffffffu, t, 1);
        t += __shfl_xor_sync(0xffffffffu, t, 2);
        const int32_t qi = __shfl_sync(0xffffffffu, qid, min(i, 31));
        if (part == 0 && i < nq) hs[qi] = t;
    }
}

template <int DIM, int ROUNDS>
tf_status launch_cl_fill4(const SortedPtsView &P, const Grid &g, const GroupRec *rec, const int64_t *loff, int32_t G,
                          int LPmax, int S, const uint16_t *list, const uint32_t *mask, tf_filter_s *h, int32_t *stats,
                          cudaStream_t s) {
    const size_t smem = (size_t)LPmax * ((DIM == 3 ? 24 : 16) + 4) + (size_t)32 * S * sizeof(uint16_t);
    auto kern = k_cl_fill4<DIM, ROUNDS>;
    TF_TRY(allow_dynamic_smem(kern, smem));
    kern<<<(unsigned)G, 128, smem, s>>>(P, g, rec, loff, LPmax, S, list, mask, h->rowptr, h->cols, h->vals, h->hs,
                                        stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
}

template <int DIM>
tf_status launch_cl_count(const SortedPtsView &P, const Grid &g, const GroupRec *rec, const int64_t *loff, int32_t G,
                          int LPmax, uint16_t *list, uint32_t *mask, int32_t *counts, int32_t *stats, cudaStream_t s) {
    const size_t smem = (size_t)5 * LPmax * sizeof(uint32_t);
    auto kern = k_cl_count<DIM>;
    TF_TRY(allow_dynamic_smem(kern, smem));
    kern<<<(unsigned)G, kCountWarps * 32, smem, s>>>(P, g, rec, loff, LPmax, list, mask, counts, stats);
    TF_LAUNCH_CHECK();
    return TF_OK;
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
    const unsigned gridG = (unsigned)std::min<int64_t>((U * 32 + threads - 1) / threads, (int64_t)di.sms * 32);
    if (dim == 3) k_cl_groups<3><<<gridG, threads, 0, s>>>(P.cs, sorted_keys, g, nxb, U, goff.p, rec.p, lp.p, stats.p);
    else k_cl_groups<2><<<gridG, threads, 0, s>>>(P.cs, sorted_keys, g, nxb, U, goff.p, rec.p, lp.p, stats.p);
    TF_LAUNCH_CHECK();
    TF_TRY(exclusive_scan_i32_i64(lp.p, loff.p, Gmax, s));
    int32_t hG = 0, hmax = 0, hrun = 0;
    int64_t hTot = 0;
    TF_CUDA_TRY(cudaMemcpyAsync(&hG, goff.p + U, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaMemcpyAsync(&hmax, stats.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaMemcpyAsync(&hrun, stats.p + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaMemcpyAsync(&hTot, loff.p + Gmax, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    build_trace().mark("groups+sync", s);
    h->info.max_candidates = hmax;
    if (hmax > kMaxUnion || hrun >= kMaxRun || hG <= 0) return TF_OK;  // per-bin kernels take it
    const int LPmax = (hmax + 31) & ~31;

    // a5 count: sorted unions + mask words + row lengths
    DevBuf<uint16_t> list;
    DevBuf<int32_t> counts;
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
    // S = 2 mod 4 uint16 so lanes at equal list positions hit different banks
    int S = std::max(2, (std::min(maxrow, kListCap) + 3) & ~1);  // +2 slots for the walk's idle writes
    if ((S & 3) == 0) S += 2;
    const int rounds = std::min(3, (std::min(maxrow, 96) + 31) / 32);  // 32-entry rounds in flight per row
    // k_cl_fill4 (block per group, union staged in shared memory) measured faster only for small
    // unions (config 4: 366 vs 402 us; config 5: 8.9 vs 6.65 ms), so it takes the builds whose blocks
    // need <= 12 KB (2D neighbourhoods); k_cl_fill3 (warp per group) takes the rest.
    // TOPOFILT_CL_FILL=split / walk3 force either kernel (tests, benchmarks).
    const char *fk = getenv("TOPOFILT_CL_FILL");
    const size_t smem4 = (size_t)LPmax * ((dim == 3 ? 24 : 16) + 4) + (size_t)32 * S * 2;
    const bool want4 = (fk && *fk) ? !strcmp(fk, "split") : (smem4 <= 12 * 1024);
    if (kGroupQ == 32 && want4 && smem4 <= di.smem_optin) {
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
    } else {
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
