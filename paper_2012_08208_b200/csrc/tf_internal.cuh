// tf_internal.cuh -- internal declarations shared by the libtopofilt translation units.
// Product code only: nothing here is shared with oracle/ (see DESIGN.md "Independence").
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/topofilt.h"

namespace tf {

// ------------------------------------------------------------------ errors
void set_error(const char *fmt, ...);
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

struct Status {  // lightweight status carrier for host orchestration
    tf_status code = TF_OK;
    bool ok() const { return code == TF_OK; }
};

#define TF_CUDA_TRY(expr)                                                                 \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess) {                                                          \
            ::tf::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),       \
                            __FILE__, __LINE__);                                          \
            return TF_ERR_CUDA;                                                           \
        }                                                                                 \
    } while (0)

#define TF_LAUNCH_CHECK()                                                                 \
    do {                                                                                  \
        ::tf::count_launch();                                                             \
        cudaError_t _e = cudaGetLastError();                                              \
        if (_e != cudaSuccess) {                                                          \
            ::tf::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e),   \
                            __FILE__, __LINE__);                                          \
            return TF_ERR_CUDA;                                                           \
        }                                                                                 \
    } while (0)

#define TF_TRY(expr)                                                                      \
    do {                                                                                  \
        tf_status _s = (expr);                                                            \
        if (_s != TF_OK) return _s;                                                       \
    } while (0)

// Device-side bounds/invariant checks, compiled in only for the debug variant
// (`-DTF_DEBUG_CHECKS`, built by _build.py build_debug(); compute-sanitizer is unavailable).
#ifdef TF_DEBUG_CHECKS
#define TF_DCHECK(cond)                                                                   \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            printf("TF_DCHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);          \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define TF_DCHECK(cond) \
    do {                \
    } while (0)
#endif

// NVTX range per build/apply phase (SURVEY.md sec. 5 tracing); near-free without a tool attached.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// Opt-in phase timer of the build (TOPOFILT_TRACE=1): CUDA events at phase boundaries on the
// build stream, printed to stderr (ms per phase) when the build finishes. Off: no events.
struct PhaseTrace {
    static bool enabled();
    void begin(cudaStream_t s);
    void mark(const char *name, cudaStream_t s);
    void report(const char *what);
    bool on = false;
    int k = 0;
    cudaEvent_t ev[24] = {};
    const char *name[24] = {};
};
PhaseTrace &build_trace();

// Makes `device` current for the scope (handle teardown on the handle's own device).
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int device) {
        cudaGetDevice(&prev);
        if (device >= 0 && device != prev) cudaSetDevice(device);
    }
    ~DeviceScope() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// ------------------------------------------------------------------ memory
// Stream-ordered device allocation with the test-only allocation limit.
tf_status dev_alloc(void **p, size_t bytes, cudaStream_t s, const char *what);
// 32-byte pinned host slots for small device -> host results read after a stream sync (a pool:
// cudaMallocHost costs ~1 ms, too much per build); nullptr if pinned memory is unavailable
unsigned long long *pinned_slot_acquire();
void pinned_slot_release(unsigned long long *p);
void dev_free(void *p, cudaStream_t s);
void reset_alloc_budget();

template <class T>
inline tf_status dalloc(T **p, size_t count, cudaStream_t s, const char *what) {
    return dev_alloc(reinterpret_cast<void **>(p), count * sizeof(T), s, what);
}

// Scoped temporary device buffer (freed stream-ordered on scope exit).
template <class T>
struct DevBuf {
    T *p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { reset(); }
    tf_status alloc(size_t count, cudaStream_t st, const char *what) {
        reset();
        s = st;
        return dalloc(&p, count ? count : 1, st, what);
    }
    void reset() {
        if (p) dev_free(p, s);
        p = nullptr;
    }
    T *release() {
        T *q = p;
        p = nullptr;
        return q;
    }
};

// ------------------------------------------------------------------ device info
struct DeviceInfo {
    int device = -1;
    int sms = 148;
    size_t smem_optin = 227 * 1024;
};
tf_status device_info(DeviceInfo *di);
// Allow `bytes` of dynamic shared memory for launches of `func` on the current device. The limit is a
// per-function, process-wide attribute: it is only ever RAISED, and to one value (the device's opt-in
// maximum minus the kernel's static shared memory), once per (function, device). Setting the exact size
// before every launch -- as this library did -- lets concurrent builds on different host threads lower
// the limit under each other's launches ("invalid argument"; found by tools/soak_all.py).
tf_status allow_dynamic_smem_impl(const void *func, size_t bytes);
template <class K>
inline tf_status allow_dynamic_smem(K kern, size_t bytes) {
    return allow_dynamic_smem_impl(reinterpret_cast<const void *>(kern), bytes);
}
// TF_ERR_INVALID unless p is a non-NULL device (or managed) pointer
tf_status require_device(const void *p, const char *name);
// TF_ERR_INVALID unless the current CUDA device is `device` (a handle's build device)
tf_status require_current_device(int device, const char *who);

// ------------------------------------------------------------------ the exact pair expression
// Shared by every build path (cell list and lattice): d2 = (dx*dx + dy*dy) + dz*dz with
// __dmul_rn/__dadd_rn (never contracted to FMA), the oracle's expression (R2-R3).
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

// w = max(0, rmin - sqrt(d2)). d2 == 0 (every row's diagonal) sits outside the fast range of
// the correctly rounded sqrt sequence and would send the whole warp through its slow-path
// call once per row; sqrt(0) = 0 exactly, so feed it a safe argument and select rmin.
__device__ __forceinline__ double weight_of(double rmin, double d2) {
    const double r = __dsqrt_rn(d2 > 0.0 ? d2 : 1.0);
    double w = (d2 > 0.0) ? __dsub_rn(rmin, r) : rmin;
    return w < 0.0 ? 0.0 : w;
}

// ------------------------------------------------------------------ grid of the cell list
struct Grid {
    int dim;
    double lo[3];
    double inv_s;   // 1/s, s = bin side
    double s;
    int nb[3];      // bins per dimension (nb[2] = 1 in 2D)
    int64_t nbins;
    double rmin, r2;
    // fp32 prefilter (R4b): d2_f32 < t_in => exact test accepts; >= t_out => rejects
    int use_f32;
    float t_in, t_out;
};

// ------------------------------------------------------------------ cell-list sorted points
// Centroids in cell-list order (build.cu a4): exact fp64 SoA copies, original ids, cell starts.
struct SortedPtsView {
    const double *x, *y, *z;  // SoA, sorted by (bin key, id)
    const int32_t *id;
    const int32_t *cs;        // cell start [nbins+1]
    const double4 *a;         // AoS copy (x, y, z, id bits): one 32-byte sector per gathered point
};

// ------------------------------------------------------------------ apply plan
struct ApplyPlan {
    int64_t nblocks = 0;      // row blocks
    int32_t *rb = nullptr;    // [nblocks+1] first row of each block
    int block_nnz = 0;        // target nnz per block (window)
    int stage_cap = 0;        // staged-path capacity (nnz)
    int group = 1;            // lanes per row in the reduction phase (power of two <= 32)
    int64_t *wlo = nullptr;   // [2*nblocks+1] aligned staging window start / end per row block
    int grid = 0;             // persistent grid size
    int unroll = 4;           // loads in flight per lane in the row loop (4 or 8): density
    int unroll_sens = 4;      // the same for the sensitivity launches
    int unroll_both = 4;      // the same for the both-filters launches (16-byte gathers)
    int64_t direct_rows = 0;  // sensitivity applies on filters with n <= this skip the t pass
    int pdl = 0;              // sensitivity: t pass + programmatic dependent SpMV launch
    // row-range chunks of the host pipeline: windows [chunk_w[i], chunk_w[i+1]) cover rows
    // [chunk_r[i], chunk_r[i+1])
    int nchunks = -1;  // -1: not computed yet
    int64_t chunk_w[17] = {};
    int32_t chunk_r[17] = {};
    int32_t chunk_maxcol[16] = {};  // largest column read by chunk i (-1: none)
};
#ifndef TF_HOST_CHUNKS
#define TF_HOST_CHUNKS 8
#endif
constexpr int kMaxChunks = TF_HOST_CHUNKS;  // <= 16 (array sizes above)
static_assert(kMaxChunks >= 1 && kMaxChunks <= 16, "host pipeline chunks");

// ------------------------------------------------------------------ matrix-free stencil (a10)
constexpr int kMaxTypes = 8;  // cells per lattice cube (tf_build_lattice)
struct StencilGeom {
    int dim = 0;
    int64_t nx = 0, ny = 0, nz = 0;
    int R = 0;      // largest |offset| component
    int K = 0;      // number of offsets (0: not a stencil handle)
    int ty = 4, tz = 2;
    double h = 0;
    double hs_full = 0;  // row sum of an interior cell (all offsets in the grid)
    // periodic lattices (T > 1 types per cube, cell = T*cube + type): offsets of type s are
    // [kstart[s], kstart[s+1]) as (dx, dy, dz, target type); hs_full_t = interior row sums
    int T = 1;
    bool lattice = false;  // built by tf_build_lattice (k_lattice), else k_stencil
    int kstart[kMaxTypes + 1] = {};
    double hs_full_t[kMaxTypes] = {};
};

}  // namespace tf

// ------------------------------------------------------------------ the handle
struct tf_filter_s {
    int device = -1;  // the CUDA device current at build time; every call must use it
    cudaStream_t stream = nullptr;  // the build stream: tf_free releases the memory stream-ordered on it
    // speculative exact lattice build (lattice_build.cu): results of the verification pass, the
    // fill's agreement flag and the scanned nnz land here (pinned) by the build's final sync and
    // are checked then; lat_nnz_host is the nnz the host tables predicted
    bool lat_pending = false;
    unsigned long long *lat_check = nullptr;  // pinned: [0] dev bits, [1] flags, [2] fill flag, [3] nnz
    int64_t lat_nnz_host = 0;
    int64_t n = 0, nnz = 0;
    int dim = 0;
    double rmin = 0;
    int64_t *rowptr = nullptr;
    int32_t *cols = nullptr;
    double *vals = nullptr;
    double *hs = nullptr;
    tf::ApplyPlan plan;
    bool cols_ascending = false;  // set by the library's own build (tf_filter_from_csr: unknown)
    int64_t max_row_hint = -1;    // longest row when the build knows it (count pass, lattice exact tables)
    tf_build_info info{};
    // host-API scratch (lazily allocated, owned) + a side stream / event for copy overlap
    double *hx = nullptr, *hdc = nullptr, *hout = nullptr, *hout2 = nullptr, *ht = nullptr;
    cudaStream_t side = nullptr, side2 = nullptr;  // upload / download streams of the host pipeline
    cudaEvent_t ev = nullptr, ev2 = nullptr;
    cudaEvent_t evc[2 * tf::kMaxChunks] = {};  // per-chunk completion of the host pipeline
    cudaEvent_t evx[tf::kMaxChunks] = {}, evd[tf::kMaxChunks] = {};  // x / dc piece uploaded
    // matrix-free stencil handles (tf_build_stencil): no CSR; offset table on the device
    tf::StencilGeom stencil;
    int4 *stencil_off = nullptr;
    double *stencil_w = nullptr;
    // periodic lattice handles: the device offset table (16-byte entries for the tile shape)
    void *lattice_table = nullptr;
};

// ------------------------------------------------------------------ shard plan (NEXT-4)
struct tf_shard_s {
    int device = -1;
    int nranks = 0, rank = 0, axis = 0;
    double cut_lo = 0, cut_hi = 0;   // this rank's slab along `axis` (-inf / +inf at the ends)
    int64_t n_interior = 0, n_owned = 0, n_halo = 0;
    std::vector<int64_t> recv, send;  // per rank: halo points received from / sent to it
    int32_t *local_ids = nullptr;     // [n_owned + n_halo] global ids in local order
    int32_t *send_idx = nullptr;      // sum(send): local indices, grouped by destination rank
    cudaStream_t stream = nullptr;
};

namespace tf {

// shard.cu (NEXT-4): the device slab partition of rank `me` of W; gather of centroid rows
tf_status shard_plan(const double *c, int64_t n, int dim, double rmin, int W, int me, cudaStream_t s,
                     tf_shard_s *p);
tf_status launch_gather_rows(const double *src, int dim, const int32_t *idx, int64_t m, double *dst, cudaStream_t s);

// scan.cu
tf_status exclusive_scan_i32_i64(const int32_t *in, int64_t *out, int64_t n, cudaStream_t s);
tf_status exclusive_scan_i32_i32(const int32_t *in, int32_t *out, int64_t n, cudaStream_t s);

// radix.cu: stable LSD sort of (key, val) pairs by the low `bits` bits of key.
// Results land in (keys_out, vals_out); the inputs are used as ping-pong scratch.
tf_status radix_sort_pairs(uint32_t *keys, uint32_t *vals, uint32_t *keys_alt, uint32_t *vals_alt,
                           int64_t n, int bits, cudaStream_t s, uint32_t **keys_out,
                           uint32_t **vals_out, int *passes);

// build.cu (flags: TF_BUILD_*, optionally | kBuildNoSpeculation; the lattice path is tried first
// unless TF_BUILD_CELL_LIST)
constexpr int kBuildNoSpeculation = 1 << 16;
tf_status build_filter_device(const double *c, int64_t n, int dim, double rmin, int flags, cudaStream_t s,
                              tf_filter_s *h);
// cl_build.cu: the group kernels of the cell-list build (count -> scan -> fill) on the sorted
// points; *done = false (TF_OK, nothing allocated in h) when a union exceeds their capacity
tf_status build_cell_list_groups(const SortedPtsView &P, const uint32_t *sorted_keys, const Grid &g, int64_t n,
                                 cudaStream_t s, tf_filter_s *h, bool *done);
// dense_build.cu: the all-pairs ablation (TF_BUILD_DENSE)
tf_status build_dense_csr(const double *c, int64_t n, int dim, double rmin, cudaStream_t s, tf_filter_s *h);
// lattice_build.cu: *used = false (and TF_OK) when the centroids are not a verified lattice
tf_status build_lattice_csr(const double *c, int64_t n, int dim, double rmin, cudaStream_t s, tf_filter_s *h,
                            bool *used, bool speculate = true);
// after the build's final synchronisation: false if the speculative exact lattice build must be
// redone (verification failed, or the fill disagreed with the predicted row lengths)
bool lattice_check_ok(const tf_filter_s *h);
// the detection step alone on a host array (no CUDA calls): T = 0 if not lattice-ordered
tf_status lattice_detect_host(const double *c, int64_t n, int dim, int32_t *T, int64_t cubes[3], double spacing[3]);

// stencil.cu
tf_status build_stencil(int dim, int64_t nx, int64_t ny, int64_t nz, double h, double rmin, cudaStream_t s,
                        tf_filter_s *f);
tf_status launch_stencil(const tf_filter_s *f, const double *x, const double *dc, double *out, bool sens,
                         cudaStream_t s);
tf_status build_lattice(int dim, int64_t nx, int64_t ny, int64_t nz, double h, int ntypes, const double *type_offsets,
                        double rmin, cudaStream_t s, tf_filter_s *f);

// oc.cu (NEXT-1)
tf_status oc_update(const double *x, const double *dc, int64_t n, double volfrac, double move, double l1,
                    double l2, double tol, double *xnew, double *lmid_out, int *iters_out, cudaStream_t s);

// apply.cu
tf_status make_apply_plan(tf_filter_s *h, cudaStream_t s);
tf_status launch_sensitivity(const tf_filter_s *h, const double *x, const double *dc, double *out,
                             cudaStream_t s);
tf_status launch_density(const tf_filter_s *h, const double *x, double *out, cudaStream_t s);
tf_status launch_sensitivity_rows(const tf_filter_s *h, const double *x, const double *dc, double *out,
                                  int64_t nrows, cudaStream_t s);
tf_status launch_density_rows(const tf_filter_s *h, const double *x, double *out, int64_t nrows, cudaStream_t s);
// rows [r0, r1) (NEXT-4 interior/boundary split); rows of the first window before r0 are recomputed
tf_status launch_sensitivity_rowrange(const tf_filter_s *h, const double *x, const double *dc, double *out,
                                      int64_t r0, int64_t r1, cudaStream_t s);
tf_status launch_density_rowrange(const tf_filter_s *h, const double *x, double *out, int64_t r0, int64_t r1,
                                  cudaStream_t s);
// both filters in one pass over H (sensitivity -> sens_out, density -> dens_out)
tf_status launch_both(const tf_filter_s *h, const double *x, const double *dc, double *sens_out, double *dens_out,
                      cudaStream_t s);
// row-range chunk i of the plan (host pipeline); the sensitivity chunk 0 computes t = x*dc into
// tbuf (cooperative), later chunks reuse it
tf_status ensure_chunk_plan(tf_filter_s *h, cudaStream_t s);
tf_status launch_halo_pack(const double *src, const int32_t *idx, int64_t m, double *dst, cudaStream_t s);
tf_status launch_density_range(const tf_filter_s *h, const double *x, double *out, int chunk, cudaStream_t s);
tf_status launch_hadamard_piece(const tf_filter_s *h, const double *x, const double *dc, double *t, int piece,
                                cudaStream_t s);
tf_status launch_sensitivity_range(const tf_filter_s *h, const double *x, const double *dc, double *out, double *tbuf,
                                   int chunk, int tpass, cudaStream_t s);
tf_status launch_sensitivity_energy(const tf_filter_s *h, const double *x, const double *U, double penal,
                                    double *out, cudaStream_t s);

}  // namespace tf
