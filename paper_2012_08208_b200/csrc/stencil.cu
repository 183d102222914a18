// stencil.cu -- matrix-free filter apply for regular grids (BASELINE.json
// north_star: "a matrix-free stencil variant for structured grids, kept only if ncu shows it
// beats stored CSR").
//
// For cells on a regular grid (index (k*ny + j)*nx + i, centroid origin + ((i,j,k)+1/2)*h) the
// weight of Eq. filter_cond depends only on the integer offset (a,b,c):
//   d2 = ((a*h)*(a*h) + (b*h)*(b*h)) + (c*h)*(c*h)  (same fp64 expression and order as the CSR
//   build; exact for the configs' h = 1), stored iff d2 < rmin^2, w = max(0, rmin - sqrt(d2)),
// so H never needs to be stored: out_i = sum_o w_o t[i + o] over in-grid neighbours, and
// Hs_i = sum_o w_o over the same neighbours (boundary truncation), recomputed on the fly.
// HBM traffic per apply: x and dc read once, out written once (24 N bytes for the
// sensitivity filter, 16 N for density) instead of 12 nnz + ... for the CSR.
//
// Kernel: one block per (32 x TY x TZ) tile; the block stages t = x*dc (or x) of the tile
// plus its halo of radius R in shared memory with coalesced loads (0 outside the grid), then
// each thread sums its cell's K offsets from shared memory (offset table: handle-owned device
// memory, broadcast reads). Row sums: the full offset-order sum for cells whose neighbours are
// all in the grid, the truncated sum built once per handle (k_lattice_hs) near the boundary.
#include <math.h>

#include <algorithm>
#include <new>
#include <vector>

#include "tf_internal.cuh"

namespace tf {
namespace {

constexpr int kMaxOffsets = 4096;

constexpr int kTX = 32;

// RC = compile-time halo radius (1..4) or 0 for a runtime radius (general fallback)
template <bool SENS, int DIM, int RC>
__global__ void __launch_bounds__(256) k_stencil(StencilGeom sg, const int4 *__restrict__ offs,
                                                 const double *__restrict__ wts, const double *__restrict__ hs_cell,
                                                 const double *__restrict__ x, const double *__restrict__ dc,
                                                 double *__restrict__ out) {
    extern __shared__ double tile[];
    // 32 x TY x TZ cells per block, two per thread (the second kStHalf rows further along the
    // last axis), so each broadcast offset/weight read serves two tile reads
    constexpr int TY = (DIM == 3) ? 4 : 16, TZ = (DIM == 3) ? 4 : 1;
    const int R = RC ? RC : sg.R;
    const int HX = kTX + 2 * R, HY = TY + 2 * R, HZ = (DIM == 3) ? TZ + 2 * R : 1;
    const int bx0 = blockIdx.x * kTX, by0 = blockIdx.y * TY, bz0 = (DIM == 3) ? blockIdx.z * TZ : 0;
    const int nx = (int)sg.nx, ny = (int)sg.ny, nz = (int)sg.nz;
    // stage t over the haloed tile, one x-row per warp iteration (coalesced; no divisions);
    // out-of-grid neighbours stage 0 and add fma(w, 0, acc) = acc exactly
    const int rows = HY * HZ;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int row = warp; row < rows; row += 8) {
        const int hy = row % HY, hz = row / HY;
        const int gy = by0 + hy - R, gz = (DIM == 3) ? bz0 + hz - R : 0;
        const bool rok = gy >= 0 && gy < ny && gz >= 0 && gz < nz;
        const int64_t rbase = ((int64_t)gz * ny + gy) * nx;
        for (int hx = lane; hx < HX; hx += 32) {
            const int gx = bx0 + hx - R;
            double t = 0.0;
            if (rok && gx >= 0 && gx < nx) {
                const int64_t g = rbase + gx;
                t = SENS ? __ldg(x + g) * __ldg(dc + g) : __ldg(x + g);
            }
            tile[row * HX + hx] = t;
        }
    }
    // offset table -> shared memory as tile-index deltas
    int *s_delta = reinterpret_cast<int *>(tile + rows * HX);
    double *s_w = reinterpret_cast<double *>(s_delta + ((sg.K + 1) & ~1));
    for (int o = threadIdx.x; o < sg.K; o += 256) {
        const int4 off = __ldg(offs + o);
        s_delta[o] = ((DIM == 3) ? off.z * HY * HX : 0) + off.y * HX + off.x;
        s_w[o] = __ldg(wts + o);
    }
    __syncthreads();
    // two cells per thread: (lx, ly, lz) and the cell half a tile further along the last axis
    const int lx = threadIdx.x & 31;
    const int ly = (DIM == 3) ? (threadIdx.x >> 5) % TY : (threadIdx.x >> 5);
    const int lz = (DIM == 3) ? (threadIdx.x >> 5) / TY : 0;
    const int step = (DIM == 3) ? (TZ / 2) * HY * HX : (TY / 2) * HX;  // tile offset of the 2nd cell
    const int center = (((DIM == 3) ? lz + R : 0) * HY + (ly + R)) * HX + (lx + R);
    double a0 = 0.0, a1 = 0.0;
#pragma unroll 9
    for (int o = 0; o < sg.K; ++o) {
        const double w = s_w[o];
        const int si = center + s_delta[o];
        a0 = fma(w, tile[si], a0);
        a1 = fma(w, tile[si + step], a1);
    }
    const int gx = bx0 + lx;
    for (int q = 0; q < 2; ++q) {
        const int gy = by0 + ly + ((DIM == 2 && q) ? TY / 2 : 0);
        const int gz = bz0 + lz + ((DIM == 3 && q) ? TZ / 2 : 0);
        if (gx >= nx || gy >= ny || gz >= nz) continue;
        const int64_t g = ((int64_t)gz * ny + gy) * nx + gx;
        // row sum: the full offset-order sum for cells with every neighbour in the grid, else the
        // truncated offset-order sum built once per handle (k_lattice_hs) -- bitwise the same
        const bool inner = gx >= R && gx + R < nx && gy >= R && gy + R < ny && (DIM == 2 || (gz >= R && gz + R < nz));
        const double hs = inner ? sg.hs_full : __ldg(hs_cell + g);
        const double acc = q ? a1 : a0;
        out[g] = SENS ? acc / (hs * fmax(1e-3, __ldg(x + g))) : acc / hs;
    }
}

// ------------------------------------------------------------------ periodic lattices (T types)
// Cells T*cube + s at h*((i,j,k) + o_s) (BoxMesh-style tetrahedra: T = 6; triangulated squares:
// T = 2). The weight between type s at cube c and type t at cube c + d depends only on
// (s, t, d), so per source type a table of (d, t, w) replaces the stored rows. The block stages
// t = x*dc of its haloed tile ONE ARRAY PER TYPE ([T][HZ][HY][HX]: a warp's lanes read 32
// consecutive cubes of one type, conflict-free), and each warp computes one (row, type) item
// of 32 cubes at a time, so every lane of the warp walks the same offset list (broadcast
// shared-memory reads). Tiles away from the grid boundary skip the in-grid mask: their row sum
// is the type's full sum hs_full_t, bitwise the masked offset-order sum (fma(w, 1, h) = h + w).
// One 16-byte entry per offset (tile index delta = type * plane + cube delta, cube delta for the
// mask, weight), precomputed at build for the tile shape: every lane of a warp reads the same
// entry, so each offset costs one broadcast shared-memory wavefront besides the tile read.
constexpr int kLatMaxOffs = 4096;
#ifndef TF_LAT_TZ
#define TF_LAT_TZ 4   // lattice tile depth (cubes) in 3D (swept: 2/4/8 x rows 2/4/8 -> 4, 4)
#endif
#ifndef TF_LAT_RPI
#define TF_LAT_RPI 4  // rows per warp item (one table read serves this many tile reads)
#endif
constexpr int kLatTZ = TF_LAT_TZ, kLatRPI = TF_LAT_RPI;
struct __align__(16) LatEntry {
    int delta, mdelta;
    double w;
};

template <bool SENS, int DIM, int RC, int TT>
__global__ void __launch_bounds__(256) k_lattice(StencilGeom sg, const LatEntry *__restrict__ tab,
                                                 const double *__restrict__ hs_cell, const double *__restrict__ x,
                                                 const double *__restrict__ dc, double *__restrict__ out) {
    extern __shared__ double tile[];
    constexpr int TY = (DIM == 3) ? 4 : 8, TZ = (DIM == 3) ? kLatTZ : 1;
    const int T = TT ? TT : sg.T;
    const int R = RC ? RC : sg.R;
    const int HX = kTX + 2 * R, HY = TY + 2 * R, HZ = (DIM == 3) ? TZ + 2 * R : 1;
    const int plane = HX * HY * HZ;
    const int bx0 = blockIdx.x * kTX, by0 = blockIdx.y * TY, bz0 = (DIM == 3) ? blockIdx.z * TZ : 0;
    const int nx = (int)sg.nx, ny = (int)sg.ny, nz = (int)sg.nz;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows = HY * HZ;
    // stage t (0 outside the grid: out-of-grid neighbours add fma(w, 0, acc) = acc exactly)
    for (int row = warp; row < rows; row += 8) {
        const int hy = row % HY, hz = row / HY;
        const int gy = by0 + hy - R, gz = (DIM == 3) ? bz0 + hz - R : 0;
        const bool rok = gy >= 0 && gy < ny && gz >= 0 && gz < nz;
        const int64_t rbase = ((int64_t)gz * ny + gy) * nx;
        // the row's HX cubes x T types are contiguous in global memory: coalesced
        for (int e = lane; e < HX * T; e += 32) {
            const int hx = e / T, t = e - hx * T;
            const int gx = bx0 + hx - R;
            double v = 0.0;
            if (rok && gx >= 0 && gx < nx) {
                const int64_t g = (rbase + gx) * T + t;
                v = SENS ? __ldg(x + g) * __ldg(dc + g) : __ldg(x + g);
            }
            tile[(size_t)t * plane + row * HX + hx] = v;
        }
    }
    LatEntry *s_tab = reinterpret_cast<LatEntry *>(tile + (((size_t)T * plane + 1) & ~(size_t)1));
    for (int o = threadIdx.x; o < sg.K; o += 256) s_tab[o] = tab[o];
    __syncthreads();
    // items: (kLatRPI rows, type); one table read serves the rows' tile reads
    constexpr int RPI = kLatRPI;
    constexpr int NP = TY * TZ / RPI;
    for (int item = warp; item < NP * T; item += 8) {
        const int s = item % T, p = item / T;
        int ly[RPI], lz[RPI], c[RPI];
        double a[RPI];
#pragma unroll
        for (int q = 0; q < RPI; ++q) {
            const int ri = RPI * p + q;
            ly[q] = ri % TY, lz[q] = ri / TY;
            c[q] = (((DIM == 3) ? lz[q] + R : 0) * HY + (ly[q] + R)) * HX + (lane + R);
            a[q] = 0.0;
        }
        const int o0 = sg.kstart[s], o1 = sg.kstart[s + 1];
#pragma unroll 4
        for (int o = o0; o < o1; ++o) {
            const LatEntry e = s_tab[o];
#pragma unroll
            for (int q = 0; q < RPI; ++q) a[q] = fma(e.w, tile[c[q] + e.delta], a[q]);
        }
        const int gx = bx0 + lane;
#pragma unroll
        for (int q = 0; q < RPI; ++q) {
            const int gy = by0 + ly[q], gz = bz0 + lz[q];
            if (gx >= nx || gy >= ny || gz >= nz) continue;
            const int64_t g = (((int64_t)gz * ny + gy) * nx + gx) * T + s;
            // interior cells: the type's full row sum; near the boundary: the truncated sum built once
            const bool inner = gx >= R && gx + R < nx && gy >= R && gy + R < ny && (DIM == 2 || (gz >= R && gz + R < nz));
            const double hs = inner ? sg.hs_full_t[s] : __ldg(hs_cell + g);
            out[g] = SENS ? a[q] / (hs * fmax(1e-3, __ldg(x + g))) : a[q] / hs;
        }
    }
}

// Row sums with boundary truncation, once per lattice handle: in offset order, only in-grid
// neighbours (bitwise the interior full sum where nothing is truncated).
template <int DIM>
__global__ void k_lattice_hs(StencilGeom sg, const int4 *__restrict__ offs, const double *__restrict__ w,
                             double *__restrict__ hs) {
    const int64_t n = sg.nx * sg.ny * sg.nz * sg.T;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cube = g / sg.T;
        const int s = (int)(g - cube * sg.T);
        const int64_t cx = cube % sg.nx, cy = (cube / sg.nx) % sg.ny, cz = cube / (sg.nx * sg.ny);
        const int R = sg.R;
        if (cx >= R && cx + R < sg.nx && cy >= R && cy + R < sg.ny && (DIM == 2 || (cz >= R && cz + R < sg.nz))) {
            hs[g] = sg.hs_full_t[s];  // nothing truncated: the full offset-order sum
            continue;
        }
        double h = 0.0;
        for (int o = sg.kstart[s]; o < sg.kstart[s + 1]; ++o) {
            const int4 q = offs[o];
            const int64_t ax = cx + q.x, ay = cy + q.y, az = cz + q.z;
            if (ax >= 0 && ax < sg.nx && ay >= 0 && ay < sg.ny && az >= 0 && az < sg.nz) h += w[o];
        }
        hs[g] = h;
    }
}

}  // namespace

tf_status build_lattice(int dim, int64_t nx, int64_t ny, int64_t nz, double h, int ntypes, const double *o,
                        double rmin, cudaStream_t s, tf_filter_s *f) {
    // per source type s: every (target type t, cube offset d) with d2 < rmin^2, the same fp64
    // pair expression as the CSR build on centroids h*(cube + o): delta = h*(d + o_t - o_s)
    const double r2 = rmin * rmin;
    const int Rs = (int)floor(rmin / h) + 2;
    std::vector<int4> off;
    std::vector<double> w;
    StencilGeom &sg = f->stencil;
    sg.T = ntypes;
    // one type per cube is a regular grid: k_stencil is faster there (config 3: 34.8 vs 41.0 us,
    // bitwise the same result; tools/stencil_vs_lattice.py) and reads the same offset table
    sg.lattice = ntypes > 1;
    const int zr = (dim == 3) ? Rs : 0;
    for (int st = 0; st < ntypes; ++st) {
        sg.kstart[st] = (int)off.size();
        double hsum = 0.0;
        for (int tt = 0; tt < ntypes; ++tt)
            for (int c = -zr; c <= zr; ++c)
                for (int b = -Rs; b <= Rs; ++b)
                    for (int a = -Rs; a <= Rs; ++a) {
                        const double ox = o[tt * dim + 0] - o[st * dim + 0], oy = o[tt * dim + 1] - o[st * dim + 1];
                        const double oz = (dim == 3) ? o[tt * dim + 2] - o[st * dim + 2] : 0.0;
                        const volatile double dx = ((double)a + ox) * h, dy = ((double)b + oy) * h;
                        const volatile double dz = ((double)c + oz) * h;
                        const volatile double dxx = dx * dx, dyy = dy * dy, dzz = dz * dz;
                        const volatile double s2 = dxx + dyy;
                        const double d2 = (dim == 3) ? (double)(s2 + dzz) : (double)s2;
                        if (!(d2 < r2)) continue;
                        double ww = rmin;
                        if (d2 > 0.0) {
                            const volatile double sq = sqrt(d2);
                            ww = rmin - sq;
                        }
                        if (ww < 0) ww = 0;
                        off.push_back(make_int4(a, b, c, tt));
                        w.push_back(ww);
                        hsum += ww;  // offset order: the kernel's masked sum is bitwise this
                    }
        sg.hs_full_t[st] = hsum;
    }
    sg.kstart[ntypes] = (int)off.size();
    if ((int)off.size() > kLatMaxOffs) {
        set_error("lattice radius too large (%zu offsets > %d); use tf_build_filter", off.size(), kLatMaxOffs);
        return TF_ERR_INVALID;
    }
    int Rk = 0;
    for (const int4 &q : off) Rk = std::max(Rk, std::max(abs(q.x), std::max(abs(q.y), abs(q.z))));
    const int TY = (dim == 3) ? 4 : 8, TZ = (dim == 3) ? kLatTZ : 1;
    const int HX = kTX + 2 * Rk, HY = TY + 2 * Rk;
    const size_t plane = (size_t)HX * HY * (dim == 3 ? TZ + 2 * Rk : 1);
    const size_t smem = sizeof(double) * (plane * ntypes + 1) + sizeof(LatEntry) * off.size();
    std::vector<LatEntry> tab(off.size());
    for (size_t o = 0; o < off.size(); ++o) {
        const int md = ((dim == 3) ? off[o].z * HY * HX : 0) + off[o].y * HX + off[o].x;
        tab[o].mdelta = md;
        tab[o].delta = off[o].w * (int)plane + md;
        tab[o].w = w[o];
    }
    if (smem > 200 * 1024) {
        set_error("lattice halo tile too large for shared memory (rmin/h or types); use tf_build_filter");
        return TF_ERR_INVALID;
    }
    sg.dim = dim;
    sg.nx = nx, sg.ny = ny, sg.nz = (dim == 3) ? nz : 1;
    sg.R = Rk;
    sg.K = (int)off.size();
    // tile shape of the kernel that runs: k_lattice, or k_stencil for one type per cube
    sg.ty = sg.lattice ? TY : ((dim == 3) ? 4 : 16);
    sg.tz = sg.lattice ? TZ : ((dim == 3) ? 4 : 1);
    sg.h = h;
    sg.hs_full = sg.hs_full_t[0];  // used by k_stencil when one type per cube routes there
    TF_TRY(dev_alloc(&f->lattice_table, sizeof(LatEntry) * tab.size(), s, "lattice offset table"));
    TF_CUDA_TRY(cudaMemcpyAsync(f->lattice_table, tab.data(), sizeof(LatEntry) * tab.size(), cudaMemcpyHostToDevice,
                                s));
    TF_TRY(dalloc(&f->stencil_off, off.size(), s, "lattice offsets"));
    TF_TRY(dalloc(&f->stencil_w, w.size(), s, "lattice weights"));
    TF_CUDA_TRY(cudaMemcpyAsync(f->stencil_off, off.data(), sizeof(int4) * off.size(), cudaMemcpyHostToDevice, s));
    TF_CUDA_TRY(cudaMemcpyAsync(f->stencil_w, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice, s));
    const int64_t ncell = nx * ny * sg.nz * ntypes;
    TF_TRY(dalloc(&f->hs, (size_t)ncell, s, "lattice row sums"));
    {
        DeviceInfo di;
        TF_TRY(device_info(&di));
        const unsigned blocks = (unsigned)std::min<int64_t>((ncell + 255) / 256, (int64_t)di.sms * 16);
        if (dim == 3) k_lattice_hs<3><<<blocks, 256, 0, s>>>(sg, f->stencil_off, f->stencil_w, f->hs);
        else k_lattice_hs<2><<<blocks, 256, 0, s>>>(sg, f->stencil_off, f->stencil_w, f->hs);
        TF_LAUNCH_CHECK();
    }
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    int64_t nnz = 0;  // the equivalent CSR's nonzeros
    for (const int4 &q : off)
        nnz += std::max<int64_t>(0, nx - abs(q.x)) * std::max<int64_t>(0, ny - abs(q.y)) *
               std::max<int64_t>(0, sg.nz - abs(q.z));
    f->nnz = nnz;
    return TF_OK;
}

tf_status build_stencil(int dim, int64_t nx, int64_t ny, int64_t nz, double h, double rmin, cudaStream_t s,
                        tf_filter_s *f) {
    // integer offsets with the pair test of the CSR build (d2 < rmin^2, same fp64 expression)
    const double r2 = rmin * rmin;
    const int R = (int)floor(rmin / h) + 1;
    std::vector<int4> off;
    std::vector<double> w;
    const int zr = (dim == 3) ? R : 0;
    for (int c = -zr; c <= zr; ++c)
        for (int b = -R; b <= R; ++b)
            for (int a = -R; a <= R; ++a) {
                const volatile double dx = (double)a * h, dy = (double)b * h, dz = (double)c * h;
                const volatile double dxx = dx * dx, dyy = dy * dy, dzz = dz * dz;
                const volatile double s2 = dxx + dyy;
                const double d2 = (dim == 3) ? (double)(s2 + dzz) : (double)s2;
                if (!(d2 < r2)) continue;
                const volatile double sq = sqrt(d2);
                double ww = rmin - sq;
                if (ww < 0) ww = 0;
                off.push_back(make_int4(a, b, c, 0));
                w.push_back(ww);
            }
    if ((int)off.size() > kMaxOffsets) {
        set_error("stencil radius too large (%zu offsets > %d); use tf_build_filter", off.size(), kMaxOffsets);
        return TF_ERR_INVALID;
    }
    int Rk = 0;
    for (const int4 &o : off) Rk = std::max(Rk, std::max(abs(o.x), std::max(abs(o.y), abs(o.z))));
    const size_t halo = sizeof(double) * (size_t)(32 + 2 * Rk) * ((dim == 3 ? 4 : 16) + 2 * Rk) * (dim == 3 ? 4 + 2 * Rk : 1);
    if (halo + 12 * off.size() > 200 * 1024) {
        set_error("stencil halo tile too large for shared memory (rmin/h too big); use tf_build_filter");
        return TF_ERR_INVALID;
    }
    StencilGeom &sg = f->stencil;
    sg.dim = dim;
    sg.nx = nx, sg.ny = ny, sg.nz = (dim == 3) ? nz : 1;
    sg.R = Rk;
    sg.K = (int)off.size();
    sg.ty = (dim == 3) ? 4 : 16;  // must match the kernel's TY/TZ
    sg.tz = (dim == 3) ? 4 : 1;
    sg.h = h;
    double hs_full = 0.0;
    for (double ww : w) hs_full += ww;  // full-stencil row sum in offset order (interior cells)
    sg.hs_full = hs_full;
    sg.T = 1;
    sg.kstart[0] = 0;
    sg.kstart[1] = (int)off.size();
    sg.hs_full_t[0] = hs_full;
    // handle-owned device copy of the offset table (read-only; concurrent applies are safe)
    TF_TRY(dalloc(&f->stencil_off, off.size(), s, "stencil offsets"));
    TF_TRY(dalloc(&f->stencil_w, w.size(), s, "stencil weights"));
    TF_CUDA_TRY(cudaMemcpyAsync(f->stencil_off, off.data(), sizeof(int4) * off.size(), cudaMemcpyHostToDevice, s));
    TF_CUDA_TRY(cudaMemcpyAsync(f->stencil_w, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice, s));
    // truncated row sums of the boundary cells (offset order), once per handle
    const int64_t ncell = nx * ny * sg.nz;
    TF_TRY(dalloc(&f->hs, (size_t)ncell, s, "stencil row sums"));
    {
        DeviceInfo di;
        TF_TRY(device_info(&di));
        const unsigned blocks = (unsigned)std::min<int64_t>((ncell + 255) / 256, (int64_t)di.sms * 16);
        if (dim == 3) k_lattice_hs<3><<<blocks, 256, 0, s>>>(sg, f->stencil_off, f->stencil_w, f->hs);
        else k_lattice_hs<2><<<blocks, 256, 0, s>>>(sg, f->stencil_off, f->stencil_w, f->hs);
        TF_LAUNCH_CHECK();
    }
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    // nnz of the equivalent CSR: every offset times the cells whose neighbour is in the grid
    int64_t nnz = 0;
    for (const int4 &o : off)
        nnz += std::max<int64_t>(0, nx - abs(o.x)) * std::max<int64_t>(0, ny - abs(o.y)) *
               std::max<int64_t>(0, sg.nz - abs(o.z));
    f->nnz = nnz;
    return TF_OK;
}

static tf_status launch_lattice(const tf_filter_s *f, const double *x, const double *dc, double *out, bool sens,
                                cudaStream_t s) {
    const StencilGeom &sg = f->stencil;
    const int TY = sg.ty, TZ = (sg.dim == 3) ? sg.tz : 1, R = sg.R;
    const size_t plane = (size_t)(kTX + 2 * R) * (TY + 2 * R) * ((sg.dim == 3) ? TZ + 2 * R : 1);
    const size_t smem = sizeof(double) * (plane * sg.T + 1) + sizeof(LatEntry) * (size_t)sg.K;
    const LatEntry *tab = reinterpret_cast<const LatEntry *>(f->lattice_table);
    dim3 grid((unsigned)((sg.nx + kTX - 1) / kTX), (unsigned)((sg.ny + TY - 1) / TY),
              (unsigned)((sg.dim == 3) ? (sg.nz + TZ - 1) / TZ : 1));
    auto go = [&](auto kern) -> tf_status {
        TF_TRY(allow_dynamic_smem(kern, smem));
        kern<<<grid, 256, smem, s>>>(sg, tab, f->hs, x, dc, out);
        TF_LAUNCH_CHECK();
        return TF_OK;
    };
    // specialisations: (3D, 6 types) = BoxMesh tetrahedra (reach 1 cube at rmin <= 1.5h: type
    // offsets differ by <= h/2 per axis), (2D, 2 types) = triangulated squares
    if (sg.dim == 3 && sg.T == 6) {
        switch (R) {
            case 1: return sens ? go(k_lattice<true, 3, 1, 6>) : go(k_lattice<false, 3, 1, 6>);
            case 2: return sens ? go(k_lattice<true, 3, 2, 6>) : go(k_lattice<false, 3, 2, 6>);
            default: break;
        }
    }
    if (sg.dim == 2 && sg.T == 2) {
        switch (R) {
            case 1: return sens ? go(k_lattice<true, 2, 1, 2>) : go(k_lattice<false, 2, 1, 2>);
            case 2: return sens ? go(k_lattice<true, 2, 2, 2>) : go(k_lattice<false, 2, 2, 2>);
            case 3: return sens ? go(k_lattice<true, 2, 3, 2>) : go(k_lattice<false, 2, 3, 2>);
            default: break;
        }
    }
    if (sg.dim == 3) return sens ? go(k_lattice<true, 3, 0, 0>) : go(k_lattice<false, 3, 0, 0>);
    return sens ? go(k_lattice<true, 2, 0, 0>) : go(k_lattice<false, 2, 0, 0>);
}

tf_status launch_stencil(const tf_filter_s *f, const double *x, const double *dc, double *out, bool sens,
                         cudaStream_t s) {
    const StencilGeom &sg = f->stencil;
    if (sg.lattice) return launch_lattice(f, x, dc, out, sens, s);
    const int TY = sg.ty, TZ = (sg.dim == 3) ? sg.tz : 1, R = sg.R;
    const size_t smem = sizeof(double) * (size_t)(kTX + 2 * R) * (TY + 2 * R) * ((sg.dim == 3) ? TZ + 2 * R : 1) +
                        sizeof(int) * ((sg.K + 1) & ~1) + sizeof(double) * sg.K;
    dim3 grid((unsigned)((sg.nx + kTX - 1) / kTX), (unsigned)((sg.ny + TY - 1) / TY),
              (unsigned)((sg.dim == 3) ? (sg.nz + TZ - 1) / TZ : 1));
    auto go = [&](auto kern) -> tf_status {
        TF_TRY(allow_dynamic_smem(kern, smem));
        kern<<<grid, 256, smem, s>>>(sg, f->stencil_off, f->stencil_w, f->hs, x, dc, out);
        TF_LAUNCH_CHECK();
        return TF_OK;
    };
#define TF_ST_R(D, RR)                                                                          \
    case RR:                                                                                    \
        return sens ? go(k_stencil<true, D, RR>) : go(k_stencil<false, D, RR>);
    if (sg.dim == 3) {
        switch (R) {
            TF_ST_R(3, 1) TF_ST_R(3, 2) TF_ST_R(3, 3) TF_ST_R(3, 4)
            default: return sens ? go(k_stencil<true, 3, 0>) : go(k_stencil<false, 3, 0>);
        }
    }
    switch (R) {
        TF_ST_R(2, 1) TF_ST_R(2, 2) TF_ST_R(2, 3) TF_ST_R(2, 4)
        default: return sens ? go(k_stencil<true, 2, 0>) : go(k_stencil<false, 2, 0>);
    }
#undef TF_ST_R
}

}  // namespace tf
