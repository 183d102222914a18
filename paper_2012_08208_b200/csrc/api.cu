// api.cu -- the C ABI of libtopofilt (include/topofilt.h): argument validation, handle
// lifetime, stream-ordered allocation, host-buffer variants and diagnostics. All compute
// is in build.cu / radix.cu / scan.cu / apply.cu; nothing here falls back to the CPU.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <unordered_map>
#include <new>
#include <vector>

#include "tf_internal.cuh"

namespace tf {

static thread_local char g_err[1024] = "";
std::atomic<uint64_t> g_launches{0};
static std::atomic<uint64_t> g_alloc_limit{0};

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

tf_status dev_alloc(void **p, size_t bytes, cudaStream_t s, const char *what) {
    *p = nullptr;
    const uint64_t lim = g_alloc_limit.load();
    if (lim && bytes > lim) {
        set_error("out of device memory: %s needs %zu bytes (test allocation limit %llu)", what, bytes,
                  (unsigned long long)lim);
        return TF_ERR_NOMEM;
    }
    cudaError_t e = cudaMallocAsync(p, bytes, s);
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear the sticky-free allocation error
        *p = nullptr;
        set_error("out of device memory: %s needs %zu bytes (%s)", what, bytes, cudaGetErrorString(e));
        return (e == cudaErrorMemoryAllocation) ? TF_ERR_NOMEM : TF_ERR_CUDA;
    }
    return TF_OK;
}

static std::mutex g_pin_mu;
static unsigned long long *g_pin_block = nullptr;
static std::vector<unsigned long long *> g_pin_free;

unsigned long long *pinned_slot_acquire() {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_block) {
        constexpr int kSlots = 256;
        if (cudaMallocHost((void **)&g_pin_block, (size_t)kSlots * 4 * sizeof(unsigned long long)) != cudaSuccess) {
            cudaGetLastError();
            g_pin_block = nullptr;
            return nullptr;
        }
        for (int i = kSlots - 1; i >= 0; --i) g_pin_free.push_back(g_pin_block + 4 * i);
    }
    if (g_pin_free.empty()) return nullptr;
    unsigned long long *p = g_pin_free.back();
    g_pin_free.pop_back();
    return p;
}

void pinned_slot_release(unsigned long long *p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(p);
}

void dev_free(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

bool PhaseTrace::enabled() {
    const char *e = getenv("TOPOFILT_TRACE");
    return e && *e && *e != '0';
}
void PhaseTrace::begin(cudaStream_t s) {
    on = enabled();
    k = 0;
    if (on) mark("start", s);
}
void PhaseTrace::mark(const char *nm, cudaStream_t s) {
    if (!on || k >= 24) return;
    if (!ev[k]) cudaEventCreate(&ev[k]);
    cudaEventRecord(ev[k], s);
    name[k++] = nm;
}
void PhaseTrace::report(const char *what) {
    if (!on || k < 2) return;
    cudaEventSynchronize(ev[k - 1]);
    float total = 0.f;
    cudaEventElapsedTime(&total, ev[0], ev[k - 1]);
    fprintf(stderr, "[topofilt trace] %s %.3f ms:", what, total);
    for (int i = 1; i < k; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
        fprintf(stderr, " %s %.3f", name[i], ms);
    }
    fprintf(stderr, "\n");
    on = false;
}
PhaseTrace &build_trace() {
    static thread_local PhaseTrace t;
    return t;
}

tf_status require_current_device(int device, const char *who) {
    int cur = -1;
    TF_CUDA_TRY(cudaGetDevice(&cur));
    if (cur != device) {
        set_error("%s: the handle was built on device %d but device %d is current", who, device, cur);
        return TF_ERR_INVALID;
    }
    return TF_OK;
}

tf_status device_info(DeviceInfo *di) {
    TF_CUDA_TRY(cudaGetDevice(&di->device));
    // Keep freed stream-ordered allocations cached in the device's default pool (like a
    // caching allocator) so rebuilding a filter does not go back to the driver each time.
    static thread_local int pool_set_for = -1;
    if (pool_set_for != di->device) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, di->device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
        pool_set_for = di->device;
    }
    TF_CUDA_TRY(cudaDeviceGetAttribute(&di->sms, cudaDevAttrMultiProcessorCount, di->device));
    int optin = 0;
    TF_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, di->device));
    di->smem_optin = (size_t)optin;
    return TF_OK;
}

tf_status allow_dynamic_smem_impl(const void *func, size_t bytes) {
    // (raised on first use whatever the size: static + dynamic shared memory above 48 KB needs the
    // opt-in even when the dynamic part alone is below it)
    int dev = 0;
    TF_CUDA_TRY(cudaGetDevice(&dev));
    static std::mutex mu;
    static std::unordered_map<const void *, uint64_t> raised;  // function -> bit mask of devices done
    int limit = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        uint64_t &m = raised[func];
        if (dev < 64 && (m >> dev) & 1) return TF_OK;  // (sizes were validated by the callers' own capacity rules)
        cudaFuncAttributes fa;
        TF_CUDA_TRY(cudaFuncGetAttributes(&fa, func));
        int optin = 0;
        TF_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        limit = optin - (int)fa.sharedSizeBytes;
        TF_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, limit));
        if (dev < 64) m |= 1ull << dev;
    }
    if ((int64_t)bytes > (int64_t)limit) {
        set_error("internal: a kernel needs %zu bytes of dynamic shared memory, the device allows %d", bytes, limit);
        return TF_ERR_INVALID;
    }
    return TF_OK;
}

// Device (or managed) memory check: host pointers are rejected with TF_ERR_INVALID.
tf_status require_device(const void *p, const char *name) {
    if (!p) {
        set_error("%s is NULL", name);
        return TF_ERR_INVALID;
    }
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("%s: cudaPointerGetAttributes failed: %s", name, cudaGetErrorString(e));
        return TF_ERR_INVALID;
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) {
        set_error("%s is not a device pointer (use the *_host variant for host buffers)", name);
        return TF_ERR_INVALID;
    }
    int cur = -1;
    if (a.type == cudaMemoryTypeDevice && cudaGetDevice(&cur) == cudaSuccess && a.device != cur) {
        set_error("%s lives on device %d but device %d is current", name, a.device, cur);
        return TF_ERR_INVALID;
    }
    return TF_OK;
}

static bool overlaps(const void *a, const void *b, size_t bytes) {
    const char *x = (const char *)a, *y = (const char *)b;
    return x < y + bytes && y < x + bytes;
}

static void destroy(tf_filter_s *h) {
    if (!h) return;
    DeviceScope on(h->device);  // free on the handle's device, whichever is current
    // Stream-ordered release on the handle's build stream (no device-wide synchronisation): work
    // the handle's own host-pipeline streams may still run is ordered before the frees by events;
    // work the caller issued on other streams must be complete or ordered before tf_free (the
    // cudaFreeAsync contract, include/topofilt.h).
    cudaStream_t fs = h->stream;
    for (cudaStream_t side : {h->side, h->side2}) {
        if (!side) continue;
        cudaEvent_t e = nullptr;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
            cudaEventRecord(e, side);
            cudaStreamWaitEvent(fs, e, 0);
            cudaEventDestroy(e);
        } else {
            cudaStreamSynchronize(side);
        }
    }
    for (void *p : {(void *)h->rowptr, (void *)h->cols, (void *)h->vals, (void *)h->hs, (void *)h->plan.rb,
                    (void *)h->plan.wlo, (void *)h->stencil_off, (void *)h->stencil_w, h->lattice_table,
                    (void *)h->hx, (void *)h->hdc, (void *)h->hout, (void *)h->hout2, (void *)h->ht})
        if (p) cudaFreeAsync(p, fs);
    if (h->side) cudaStreamDestroy(h->side);  // returns at once; pending work still completes
    if (h->side2) cudaStreamDestroy(h->side2);
    for (cudaEvent_t e : h->evc)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < tf::kMaxChunks; ++i) {
        if (h->evx[i]) cudaEventDestroy(h->evx[i]);
        if (h->evd[i]) cudaEventDestroy(h->evd[i]);
    }
    if (h->ev) cudaEventDestroy(h->ev);
    if (h->ev2) cudaEventDestroy(h->ev2);
    if (h->lat_check) pinned_slot_release(h->lat_check);
    cudaGetLastError();  // nothing to report from a void call
    delete h;
}

static tf_status check_build_args(int64_t n, int dim, double rmin, tf_filter *out) {
    if (!out) {
        set_error("out is NULL");
        return TF_ERR_INVALID;
    }
    *out = nullptr;
    if (dim != 2 && dim != 3) {
        set_error("dim must be 2 or 3 (got %d)", dim);
        return TF_ERR_INVALID;
    }
    if (n < 1 || n >= (int64_t)0x7fffffff) {
        set_error("n must satisfy 1 <= n < 2^31-1 (got %lld)", (long long)n);
        return TF_ERR_INVALID;
    }
    if (!isfinite(rmin) || !(rmin > 0.0)) {
        set_error("rmin must be finite and > 0 (got %g)", rmin);
        return TF_ERR_INVALID;
    }
    return TF_OK;
}

static tf_status build_common(const double *c, int64_t n, int dim, double rmin, int flags, cudaStream_t s,
                              tf_filter *out) {
    tf_filter_s *h = new (std::nothrow) tf_filter_s();
    if (!h) {
        set_error("host allocation failed");
        return TF_ERR_NOMEM;
    }
    if (cudaGetDevice(&h->device) != cudaSuccess) {
        delete h;
        set_error("cudaGetDevice failed");
        return TF_ERR_CUDA;
    }
    h->stream = s;
    h->n = n;
    h->dim = dim;
    h->rmin = rmin;
    build_trace().begin(s);
    tf_status st = build_filter_device(c, n, dim, rmin, flags, s, h);
    h->cols_ascending = true;  // the fill writes every row's columns ascending
    if (st == TF_OK) st = make_apply_plan(h, s);
    build_trace().mark("apply_plan", s);
    if (st == TF_OK) {
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            set_error("tf_build_filter: %s", cudaGetErrorString(e));
            st = TF_ERR_CUDA;
        }
    }
    if (st == TF_OK && h->lat_pending && !lattice_check_ok(h)) {
        // the speculative exact lattice build did not hold up (verification or fill check): redo
        // it without speculation (tested lattice mode or the cell list)
        tf_filter_s *g = new (std::nothrow) tf_filter_s();
        if (!g) {
            destroy(h);
            set_error("host allocation failed");
            return TF_ERR_NOMEM;
        }
        g->device = h->device;
        g->stream = s;
        g->n = n;
        g->dim = dim;
        g->rmin = rmin;
        destroy(h);
        h = g;
        st = build_filter_device(c, n, dim, rmin, flags | kBuildNoSpeculation, s, h);
        h->cols_ascending = true;
        if (st == TF_OK) st = make_apply_plan(h, s);
        if (st == TF_OK) {
            cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) {
                set_error("tf_build_filter: %s", cudaGetErrorString(e));
                st = TF_ERR_CUDA;
            }
        }
    }
    if (h->lat_check) {
        pinned_slot_release(h->lat_check);
        h->lat_check = nullptr;
    }
    h->lat_pending = false;
    build_trace().report(st == TF_OK ? "tf_build_filter" : "tf_build_filter (failed)");
    if (st != TF_OK) {
        destroy(h);
        return st;
    }
    *out = h;
    return TF_OK;
}

}  // namespace tf

using namespace tf;

extern "C" {

int tf_version(void) { return TOPOFILT_VERSION; }

const char *tf_last_error(void) { return g_err; }

tf_status tf_halo_pack(const double *src, const int32_t *idx, int64_t m, double *dst, void *stream) {
    if (m < 0) {
        set_error("tf_halo_pack: m must be >= 0");
        return TF_ERR_INVALID;
    }
    if (m == 0) return TF_OK;
    TF_TRY(require_device(src, "tf_halo_pack: src"));
    TF_TRY(require_device(idx, "tf_halo_pack: idx"));
    TF_TRY(require_device(dst, "tf_halo_pack: dst"));
    return launch_halo_pack(src, idx, m, dst, (cudaStream_t)stream);
}

uint64_t tf_kernel_launches(void) { return g_launches.load(); }

void tf_debug_set_alloc_limit(uint64_t bytes) { g_alloc_limit.store(bytes); }

tf_status tf_build_filter(const double *centroids, int64_t n, int dim, double rmin, void *stream,
                          tf_filter *out) {
    try {
        TF_TRY(check_build_args(n, dim, rmin, out));
        TF_TRY(require_device(centroids, "centroids"));
        return build_common(centroids, n, dim, rmin, TF_BUILD_AUTO, (cudaStream_t)stream, out);
    } catch (...) {
        set_error("tf_build_filter: unexpected host exception");
        return TF_ERR_NOMEM;
    }
}

tf_status tf_build_filter_ex(const double *centroids, int64_t n, int dim, double rmin, int flags, void *stream,
                             tf_filter *out) {
    try {
        TF_TRY(check_build_args(n, dim, rmin, out));
        if (flags != TF_BUILD_AUTO && flags != TF_BUILD_CELL_LIST && flags != TF_BUILD_LATTICE &&
            flags != TF_BUILD_CELL_LIST_BINS && flags != TF_BUILD_DENSE) {
            set_error("tf_build_filter_ex: unknown flags %d", flags);
            return TF_ERR_INVALID;
        }
        if (flags == TF_BUILD_DENSE && n > 4000000) {
            set_error("tf_build_filter_ex: TF_BUILD_DENSE is an O(n^2) ablation; n = %lld > 4,000,000", (long long)n);
            return TF_ERR_INVALID;
        }
        TF_TRY(require_device(centroids, "centroids"));
        return build_common(centroids, n, dim, rmin, flags, (cudaStream_t)stream, out);
    } catch (...) {
        set_error("tf_build_filter_ex: unexpected host exception");
        return TF_ERR_NOMEM;
    }
}

tf_status tf_lattice_detect_host(const double *centroids_host, int64_t n, int dim, int32_t *ntypes, int64_t cubes[3],
                                 double spacing[3]) {
    try {
        if (!centroids_host || !ntypes || !cubes || !spacing) {
            set_error("tf_lattice_detect_host: NULL argument");
            return TF_ERR_INVALID;
        }
        if ((dim != 2 && dim != 3) || n < 1 || n >= (int64_t)0x7fffffff) {
            set_error("tf_lattice_detect_host: dim must be 2 or 3 and 1 <= n < 2^31-1");
            return TF_ERR_INVALID;
        }
        return lattice_detect_host(centroids_host, n, dim, ntypes, cubes, spacing);
    } catch (...) {
        set_error("tf_lattice_detect_host: unexpected host exception");
        return TF_ERR_NOMEM;
    }
}

tf_status tf_build_filter_host(const double *centroids_host, int64_t n, int dim, double rmin, void *stream,
                               tf_filter *out) {
    try {
        TF_TRY(check_build_args(n, dim, rmin, out));
        if (!centroids_host) {
            set_error("centroids_host is NULL");
            return TF_ERR_INVALID;
        }
        cudaStream_t s = (cudaStream_t)stream;
        DevBuf<double> dc;
        TF_TRY(dc.alloc((size_t)n * dim, s, "centroids (device copy)"));
        TF_CUDA_TRY(cudaMemcpyAsync(dc.p, centroids_host, (size_t)n * dim * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
        return build_common(dc.p, n, dim, rmin, TF_BUILD_AUTO, s, out);
    } catch (...) {
        set_error("tf_build_filter_host: unexpected host exception");
        return TF_ERR_NOMEM;
    }
}

tf_status tf_build_stencil(int dim, int64_t nx, int64_t ny, int64_t nz, double h, double rmin, void *stream,
                           tf_filter *out) {
    try {
        if (!out) {
            set_error("out is NULL");
            return TF_ERR_INVALID;
        }
        *out = nullptr;
        if (dim != 2 && dim != 3) {
            set_error("dim must be 2 or 3 (got %d)", dim);
            return TF_ERR_INVALID;
        }
        const int64_t nzz = (dim == 3) ? nz : 1;
        if (nx < 1 || ny < 1 || nzz < 1 || nx * ny * nzz >= (int64_t)0x7fffffff) {
            set_error("grid dimensions must be >= 1 with nx*ny*nz < 2^31-1");
            return TF_ERR_INVALID;
        }
        if (!isfinite(rmin) || !(rmin > 0.0) || !isfinite(h) || !(h > 0.0)) {
            set_error("rmin and h must be finite and > 0");
            return TF_ERR_INVALID;
        }
        tf_filter_s *f = new (std::nothrow) tf_filter_s();
        if (!f) return TF_ERR_NOMEM;
        cudaGetDevice(&f->device);
        f->stream = (cudaStream_t)stream;
        f->n = nx * ny * nzz;
        f->dim = dim;
        f->rmin = rmin;
        tf_status st = build_stencil(dim, nx, ny, nzz, h, rmin, (cudaStream_t)stream, f);
        if (st != TF_OK) {
            destroy(f);
            return st;
        }
        *out = f;
        return TF_OK;
    } catch (...) {
        set_error("tf_build_stencil: unexpected host exception");
        return TF_ERR_NOMEM;
    }
}

tf_status tf_build_lattice(int dim, int64_t nx, int64_t ny, int64_t nz, double h, int ntypes,
                           const double *type_offsets_host, double rmin, void *stream, tf_filter *out) {
    try {
        if (!out) {
            set_error("out is NULL");
            return TF_ERR_INVALID;
        }
        *out = nullptr;
        if (dim != 2 && dim != 3) {
            set_error("dim must be 2 or 3 (got %d)", dim);
            return TF_ERR_INVALID;
        }
        if (ntypes < 1 || ntypes > kMaxTypes || !type_offsets_host) {
            set_error("ntypes must be in [1, %d] with a host array of ntypes*dim offsets", kMaxTypes);
            return TF_ERR_INVALID;
        }
        for (int i = 0; i < ntypes * dim; ++i)
            if (!(type_offsets_host[i] >= 0.0 && type_offsets_host[i] < 1.0)) {
                set_error("type offsets must lie in [0, 1) (entry %d)", i);
                return TF_ERR_INVALID;
            }
        const int64_t nzz = (dim == 3) ? nz : 1;
        if (nx < 1 || ny < 1 || nzz < 1 || nx * ny * nzz * ntypes >= (int64_t)0x7fffffff) {
            set_error("lattice dimensions must be >= 1 with nx*ny*nz*ntypes < 2^31-1");
            return TF_ERR_INVALID;
        }
        if (!isfinite(rmin) || !(rmin > 0.0) || !isfinite(h) || !(h > 0.0)) {
            set_error("rmin and h must be finite and > 0");
            return TF_ERR_INVALID;
        }
        tf_filter_s *f = new (std::nothrow) tf_filter_s();
        if (!f) return TF_ERR_NOMEM;
        cudaGetDevice(&f->device);
        f->stream = (cudaStream_t)stream;
        f->n = nx * ny * nzz * ntypes;
        f->dim = dim;
        f->rmin = rmin;
        tf_status st = build_lattice(dim, nx, ny, nzz, h, ntypes, type_offsets_host, rmin, (cudaStream_t)stream, f);
        if (st != TF_OK) {
            destroy(f);
            return st;
        }
        *out = f;
        return TF_OK;
    } catch (...) {
        set_error("tf_build_lattice: unexpected host exception");
        return TF_ERR_NOMEM;
    }
}

tf_status tf_filter_view(tf_filter h, tf_view *v) {
    if (!h || !v) {
        set_error("tf_filter_view: NULL argument");
        return TF_ERR_INVALID;
    }
    if (h->stencil.K > 0) {
        set_error("tf_filter_view: a stencil filter stores no CSR (build it with tf_build_filter)");
        return TF_ERR_INVALID;
    }
    v->n = h->n;
    v->nnz = h->nnz;
    v->dim = h->dim;
    v->rmin = h->rmin;
    v->rowptr = h->rowptr;
    v->cols = h->cols;
    v->vals = h->vals;
    v->hs = h->hs;
    return TF_OK;
}

tf_status tf_build_stats(tf_filter h, tf_build_info *info) {
    if (!h || !info) {
        set_error("tf_build_stats: NULL argument");
        return TF_ERR_INVALID;
    }
    *info = h->info;
    return TF_OK;
}

static tf_status check_apply(tf_filter h, const double *x, const double *dc, double *out, bool sens) {
    if (!h) {
        set_error("filter handle is NULL");
        return TF_ERR_INVALID;
    }
    TF_TRY(require_current_device(h->device, "apply"));
    TF_TRY(require_device(x, "x"));
    if (sens) TF_TRY(require_device(dc, "dc"));
    TF_TRY(require_device(out, "out"));
    const size_t bytes = (size_t)h->n * sizeof(double);
    if (overlaps(out, x, bytes) || (sens && overlaps(out, dc, bytes))) {
        set_error("out must not overlap x or dc");
        return TF_ERR_INVALID;
    }
    return TF_OK;
}

tf_status tf_sensitivity_filter(tf_filter h, const double *x, const double *dc, double *out, void *stream) {
    TF_TRY(check_apply(h, x, dc, out, true));
    return launch_sensitivity(h, x, dc, out, (cudaStream_t)stream);
}

tf_status tf_sensitivity_filter_energy(tf_filter h, const double *x, const double *U, double penal, double *out,
                                       void *stream) {
    TF_TRY(check_apply(h, x, U, out, true));
    if (!isfinite(penal)) {
        set_error("penal must be finite");
        return TF_ERR_INVALID;
    }
    if (h->stencil.K > 0) {
        set_error("tf_sensitivity_filter_energy: stencil handles are not supported (use a CSR filter)");
        return TF_ERR_INVALID;
    }
    return launch_sensitivity_energy(h, x, U, penal, out, (cudaStream_t)stream);
}

tf_status tf_density_filter(tf_filter h, const double *x, double *out, void *stream) {
    TF_TRY(check_apply(h, x, nullptr, out, false));
    return launch_density(h, x, out, (cudaStream_t)stream);
}

tf_status tf_sensitivity_filter_rows(tf_filter h, const double *x, const double *dc, double *out, int64_t nrows,
                                     void *stream) {
    TF_TRY(check_apply(h, x, dc, out, true));
    if (nrows < 0 || nrows > h->n) {
        set_error("nrows %lld outside [0, n = %lld]", (long long)nrows, (long long)h->n);
        return TF_ERR_INVALID;
    }
    if (nrows == 0) return TF_OK;
    return launch_sensitivity_rows(h, x, dc, out, nrows, (cudaStream_t)stream);
}

tf_status tf_density_filter_rows(tf_filter h, const double *x, double *out, int64_t nrows, void *stream) {
    TF_TRY(check_apply(h, x, nullptr, out, false));
    if (nrows < 0 || nrows > h->n) {
        set_error("nrows %lld outside [0, n = %lld]", (long long)nrows, (long long)h->n);
        return TF_ERR_INVALID;
    }
    if (nrows == 0) return TF_OK;
    return launch_density_rows(h, x, out, nrows, (cudaStream_t)stream);
}

static tf_status check_range(const tf_filter_s *h, int64_t r0, int64_t r1) {
    if (r0 < 0 || r1 < r0 || r1 > h->n) {
        set_error("row range [%lld, %lld) outside [0, n = %lld]", (long long)r0, (long long)r1, (long long)h->n);
        return TF_ERR_INVALID;
    }
    return TF_OK;
}

tf_status tf_sensitivity_filter_range(tf_filter h, const double *x, const double *dc, double *out, int64_t r0,
                                      int64_t r1, void *stream) {
    TF_TRY(check_apply(h, x, dc, out, true));
    TF_TRY(check_range(h, r0, r1));
    return launch_sensitivity_rowrange(h, x, dc, out, r0, r1, (cudaStream_t)stream);
}

tf_status tf_density_filter_range(tf_filter h, const double *x, double *out, int64_t r0, int64_t r1, void *stream) {
    TF_TRY(check_apply(h, x, nullptr, out, false));
    TF_TRY(check_range(h, r0, r1));
    return launch_density_rowrange(h, x, out, r0, r1, (cudaStream_t)stream);
}

tf_status tf_shard_plan(const double *centroids, int64_t n, int dim, double rmin, int32_t nranks, int32_t rank,
                        void *stream, tf_shard *out) {
    try {
        TF_TRY(check_build_args(n, dim, rmin, reinterpret_cast<tf_filter *>(out)));
        if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks) {
            set_error("tf_shard_plan: need 1 <= nranks <= 64 and 0 <= rank < nranks (got %d, %d)", nranks, rank);
            return TF_ERR_INVALID;
        }
        TF_TRY(require_device(centroids, "tf_shard_plan: centroids"));
        tf_shard_s *p = new (std::nothrow) tf_shard_s();
        if (!p) {
            set_error("host allocation failed");
            return TF_ERR_NOMEM;
        }
        cudaGetDevice(&p->device);
        p->nranks = nranks;
        p->rank = rank;
        p->stream = (cudaStream_t)stream;
        tf_status st = shard_plan(centroids, n, dim, rmin, nranks, rank, (cudaStream_t)stream, p);
        if (st != TF_OK) {
            tf_shard_free(p);
            return st;
        }
        *out = p;
        return TF_OK;
    } catch (const std::exception &e) {
        set_error("tf_shard_plan: %s", e.what());
        return TF_ERR_NOMEM;
    }
}

tf_status tf_shard_view_get(tf_shard s, tf_shard_view *v) {
    if (!s || !v) {
        set_error("tf_shard_view_get: NULL argument");
        return TF_ERR_INVALID;
    }
    v->nranks = s->nranks;
    v->rank = s->rank;
    v->axis = s->axis;
    v->cut_lo = s->cut_lo;
    v->cut_hi = s->cut_hi;
    v->n_interior = s->n_interior;
    v->n_owned = s->n_owned;
    v->n_halo = s->n_halo;
    v->local_ids = s->local_ids;
    v->send_idx = s->send_idx;
    return TF_OK;
}

tf_status tf_shard_counts(tf_shard s, int64_t *recv_host, int64_t *send_host) {
    if (!s || !recv_host || !send_host) {
        set_error("tf_shard_counts: NULL argument");
        return TF_ERR_INVALID;
    }
    for (int k = 0; k < s->nranks; ++k) recv_host[k] = s->recv[k], send_host[k] = s->send[k];
    return TF_OK;
}

void tf_shard_free(tf_shard s) {
    if (!s) return;
    DeviceScope on(s->device);
    if (s->local_ids) cudaFreeAsync(s->local_ids, s->stream);
    if (s->send_idx) cudaFreeAsync(s->send_idx, s->stream);
    cudaGetLastError();
    delete s;
}

tf_status tf_gather_rows(const double *src, int32_t dim, const int32_t *idx, int64_t m, double *dst, void *stream) {
    if (dim < 1 || dim > 3 || m < 0) {
        set_error("tf_gather_rows: need 1 <= dim <= 3 and m >= 0");
        return TF_ERR_INVALID;
    }
    if (m == 0) return TF_OK;
    TF_TRY(require_device(src, "tf_gather_rows: src"));
    TF_TRY(require_device(idx, "tf_gather_rows: idx"));
    TF_TRY(require_device(dst, "tf_gather_rows: dst"));
    return launch_gather_rows(src, dim, idx, m, dst, (cudaStream_t)stream);
}

tf_status tf_filter_both(tf_filter h, const double *x, const double *dc, double *sens_out, double *dens_out,
                         void *stream) {
    TF_TRY(check_apply(h, x, dc, sens_out, true));
    TF_TRY(check_apply(h, x, nullptr, dens_out, false));
    const size_t bytes = (size_t)h->n * sizeof(double);
    if (overlaps(dens_out, dc, bytes) || overlaps(sens_out, dens_out, bytes)) {
        set_error("tf_filter_both: outputs must not overlap each other, x or dc");
        return TF_ERR_INVALID;
    }
    return launch_both(h, x, dc, sens_out, dens_out, (cudaStream_t)stream);
}

// Device staging for the *_host calls: stream-ordered pool allocations on the caller's stream
// (every later use is on that stream or on the side stream after an event recorded on it).
static tf_status ensure_host_scratch(tf_filter h, cudaStream_t s, bool second_out) {
    const size_t bytes = (size_t)h->n * sizeof(double);
    if (!h->hx) {
        TF_TRY(dev_alloc((void **)&h->hx, bytes, s, "host-path staging x"));
        TF_TRY(dev_alloc((void **)&h->hdc, bytes, s, "host-path staging dc"));
        TF_TRY(dev_alloc((void **)&h->hout, bytes, s, "host-path staging out"));
    }
    if (second_out && !h->hout2) TF_TRY(dev_alloc((void **)&h->hout2, bytes, s, "host-path staging out2"));
    if (second_out && !h->ht) TF_TRY(dev_alloc((void **)&h->ht, bytes, s, "host-path t = x*dc"));
    return TF_OK;
}

tf_status tf_sensitivity_filter_host(tf_filter h, const double *x_host, const double *dc_host, double *out_host,
                                     void *stream) {
    if (!h || !x_host || !dc_host || !out_host) {
        set_error("tf_sensitivity_filter_host: NULL argument");
        return TF_ERR_INVALID;
    }
    TF_TRY(require_current_device(h->device, "tf_sensitivity_filter_host"));
    cudaStream_t s = (cudaStream_t)stream;
    TF_TRY(ensure_host_scratch(h, s, false));
    const size_t bytes = (size_t)h->n * sizeof(double);
    TF_CUDA_TRY(cudaMemcpyAsync(h->hx, x_host, bytes, cudaMemcpyHostToDevice, s));
    TF_CUDA_TRY(cudaMemcpyAsync(h->hdc, dc_host, bytes, cudaMemcpyHostToDevice, s));
    TF_TRY(launch_sensitivity(h, h->hx, h->hdc, h->hout, s));
    TF_CUDA_TRY(cudaMemcpyAsync(out_host, h->hout, bytes, cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    return TF_OK;
}

tf_status tf_filter_iteration_host(tf_filter h, const double *x_host, const double *dc_host, double *sens_host,
                                   double *dens_host, void *stream) {
    if (!h || !x_host || !dc_host || !sens_host || !dens_host) {
        set_error("tf_filter_iteration_host: NULL argument");
        return TF_ERR_INVALID;
    }
    TF_TRY(require_current_device(h->device, "tf_filter_iteration_host"));
    cudaStream_t s = (cudaStream_t)stream;
    TF_TRY(ensure_host_scratch(h, s, true));
    if (!h->side) TF_CUDA_TRY(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
    if (!h->side2) TF_CUDA_TRY(cudaStreamCreateWithFlags(&h->side2, cudaStreamNonBlocking));
    if (!h->ev) TF_CUDA_TRY(cudaEventCreateWithFlags(&h->ev, cudaEventDisableTiming));
    if (!h->ev2) TF_CUDA_TRY(cudaEventCreateWithFlags(&h->ev2, cudaEventDisableTiming));
    const size_t bytes = (size_t)h->n * sizeof(double);
    if (h->stencil.K == 0) TF_TRY(ensure_chunk_plan(h, s));
    const int K = (h->stencil.K > 0) ? 0 : h->plan.nchunks;
    TF_CUDA_TRY(cudaEventRecord(h->ev, s));  // orders the side streams after earlier work on s
    TF_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev, 0));
    TF_CUDA_TRY(cudaStreamWaitEvent(h->side2, h->ev, 0));
    if (K < 2) {
        // x goes up once for both filters; dc uploads (side stream) while the density filter runs
        TF_CUDA_TRY(cudaMemcpyAsync(h->hx, x_host, bytes, cudaMemcpyHostToDevice, s));
        TF_CUDA_TRY(cudaEventRecord(h->ev2, s));  // x first at full PCIe bandwidth, then dc
        TF_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev2, 0));
        TF_CUDA_TRY(cudaMemcpyAsync(h->hdc, dc_host, bytes, cudaMemcpyHostToDevice, h->side));
        TF_CUDA_TRY(cudaEventRecord(h->ev2, h->side));  // dc is on the device
        // stencil handles / tiny plans: whole-array launches; the density result drains (side2)
        // while the sensitivity filter runs
        TF_TRY(launch_density(h, h->hx, h->hout2, s));
        TF_CUDA_TRY(cudaEventRecord(h->ev, s));  // (a wait binds the record made before it)
        TF_CUDA_TRY(cudaStreamWaitEvent(h->side2, h->ev, 0));
        TF_CUDA_TRY(cudaMemcpyAsync(dens_host, h->hout2, bytes, cudaMemcpyDeviceToHost, h->side2));
        TF_CUDA_TRY(cudaStreamWaitEvent(s, h->ev2, 0));
        TF_TRY(launch_sensitivity(h, h->hx, h->hdc, h->hout, s));
        TF_CUDA_TRY(cudaMemcpyAsync(sens_host, h->hout, bytes, cudaMemcpyDeviceToHost, s));
    } else {
        // Row-range pipeline. Uploads (side stream) in K pieces = the chunks' row ranges, x first
        // then dc; chunk i of a filter starts once the pieces up to the one holding its largest
        // column (and its own rows) have landed; t = x o dc is formed piece by piece as dc
        // arrives; every chunk's result downloads on side2 while the next chunk computes
        // (PCIe is duplex). Pieces land in order on one stream, so waiting for piece P covers
        // pieces 0..P.
        for (int i = 0; i < 2 * K; ++i)
            if (!h->evc[i]) TF_CUDA_TRY(cudaEventCreateWithFlags(&h->evc[i], cudaEventDisableTiming));
        for (int i = 0; i < K; ++i) {
            if (!h->evx[i]) TF_CUDA_TRY(cudaEventCreateWithFlags(&h->evx[i], cudaEventDisableTiming));
            if (!h->evd[i]) TF_CUDA_TRY(cudaEventCreateWithFlags(&h->evd[i], cudaEventDisableTiming));
        }
        const int32_t *cr = h->plan.chunk_r;
        auto piece_bytes = [&](int p) { return (size_t)(cr[p + 1] - cr[p]) * sizeof(double); };
        auto gate = [&](int i) {  // last piece chunk i reads
            int g = i;
            const int32_t mc = h->plan.chunk_maxcol[i];
            for (int p = 0; p < K; ++p)
                if (mc >= cr[p] && mc < cr[p + 1]) g = std::max(g, p);
            return g;
        };
        // the x upload issued on s above is replaced by pieces on the side stream
        for (int p = 0; p < K; ++p) {
            TF_CUDA_TRY(cudaMemcpyAsync(h->hx + cr[p], x_host + cr[p], piece_bytes(p), cudaMemcpyHostToDevice, h->side));
            TF_CUDA_TRY(cudaEventRecord(h->evx[p], h->side));
        }
        for (int p = 0; p < K; ++p) {
            TF_CUDA_TRY(cudaMemcpyAsync(h->hdc + cr[p], dc_host + cr[p], piece_bytes(p), cudaMemcpyHostToDevice,
                                        h->side));
            TF_CUDA_TRY(cudaEventRecord(h->evd[p], h->side));
        }
        auto drain = [&](double *dst_host, const double *src, int i, cudaEvent_t e) -> tf_status {
            TF_CUDA_TRY(cudaEventRecord(e, s));
            TF_CUDA_TRY(cudaStreamWaitEvent(h->side2, e, 0));
            TF_CUDA_TRY(cudaMemcpyAsync(dst_host + cr[i], src + cr[i], piece_bytes(i), cudaMemcpyDeviceToHost,
                                        h->side2));
            return TF_OK;
        };
        for (int i = 0; i < K; ++i) {
            TF_CUDA_TRY(cudaStreamWaitEvent(s, h->evx[gate(i)], 0));
            TF_TRY(launch_density_range(h, h->hx, h->hout2, i, s));
            TF_TRY(drain(dens_host, h->hout2, i, h->evc[i]));
        }
        int tdone = -1;  // pieces of t formed so far
        for (int i = 0; i < K; ++i) {
            const int gi = gate(i);
            for (; tdone < gi; ) {
                ++tdone;
                TF_CUDA_TRY(cudaStreamWaitEvent(s, h->evd[tdone], 0));
                TF_TRY(launch_hadamard_piece(h, h->hx, h->hdc, h->ht, tdone, s));
            }
            TF_TRY(launch_sensitivity_range(h, h->hx, h->hdc, h->hout, h->ht, i, 0, s));
            TF_TRY(drain(sens_host, h->hout, i, h->evc[K + i]));
        }
    }
    TF_CUDA_TRY(cudaStreamSynchronize(h->side2));
    TF_CUDA_TRY(cudaStreamSynchronize(h->side));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    return TF_OK;
}

tf_status tf_density_filter_host(tf_filter h, const double *x_host, double *out_host, void *stream) {
    if (!h || !x_host || !out_host) {
        set_error("tf_density_filter_host: NULL argument");
        return TF_ERR_INVALID;
    }
    TF_TRY(require_current_device(h->device, "tf_density_filter_host"));
    cudaStream_t s = (cudaStream_t)stream;
    TF_TRY(ensure_host_scratch(h, s, false));
    const size_t bytes = (size_t)h->n * sizeof(double);
    TF_CUDA_TRY(cudaMemcpyAsync(h->hx, x_host, bytes, cudaMemcpyHostToDevice, s));
    TF_TRY(launch_density(h, h->hx, h->hout, s));
    TF_CUDA_TRY(cudaMemcpyAsync(out_host, h->hout, bytes, cudaMemcpyDeviceToHost, s));
    TF_CUDA_TRY(cudaStreamSynchronize(s));
    return TF_OK;
}

tf_status tf_filter_from_csr(const int64_t *rowptr_host, const int32_t *cols_host, const double *vals_host,
                             const double *hs_host, int64_t n, void *stream, tf_filter *out) {
    if (!out) {
        set_error("out is NULL");
        return TF_ERR_INVALID;
    }
    *out = nullptr;
    if (!rowptr_host || !cols_host || !vals_host || !hs_host || n < 1 || n >= (int64_t)0x7fffffff) {
        set_error("tf_filter_from_csr: NULL array or n out of range");
        return TF_ERR_INVALID;
    }
    if (rowptr_host[0] != 0) {
        set_error("tf_filter_from_csr: rowptr[0] != 0");
        return TF_ERR_INVALID;
    }
    for (int64_t i = 0; i < n; ++i)
        if (rowptr_host[i + 1] < rowptr_host[i]) {
            set_error("tf_filter_from_csr: rowptr not monotone at %lld", (long long)i);
            return TF_ERR_INVALID;
        }
    const int64_t nnz = rowptr_host[n];
    for (int64_t k = 0; k < nnz; ++k)
        if (cols_host[k] < 0 || cols_host[k] >= n) {
            set_error("tf_filter_from_csr: column out of range at %lld", (long long)k);
            return TF_ERR_INVALID;
        }
    cudaStream_t s = (cudaStream_t)stream;
    tf_filter_s *h = new (std::nothrow) tf_filter_s();
    if (!h) return TF_ERR_NOMEM;
    cudaGetDevice(&h->device);
    h->stream = s;
    h->n = n;
    h->nnz = nnz;
    tf_status st = TF_OK;
    auto fail = [&](tf_status e) {
        destroy(h);
        return e;
    };
    if ((st = dalloc(&h->rowptr, n + 3, s, "rowptr")) != TF_OK) return fail(st);
    if ((st = dalloc(&h->cols, nnz + 4, s, "cols")) != TF_OK) return fail(st);
    if ((st = dalloc(&h->vals, nnz + 4, s, "vals")) != TF_OK) return fail(st);
    if ((st = dalloc(&h->hs, n, s, "hs")) != TF_OK) return fail(st);
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMemcpyAsync(h->rowptr, rowptr_host, (n + 1) * 8, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(h->cols, cols_host, nnz * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(h->vals, vals_host, nnz * 8, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h->hs, hs_host, n * 8, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
        set_error("tf_filter_from_csr: %s", cudaGetErrorString(e));
        return fail(TF_ERR_CUDA);
    }
    if ((st = make_apply_plan(h, s)) != TF_OK) return fail(st);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        set_error("tf_filter_from_csr: %s", cudaGetErrorString(e));
        return fail(TF_ERR_CUDA);
    }
    *out = h;
    return TF_OK;
}

int64_t tf_filter_nnz(tf_filter h) { return h ? h->nnz : -1; }

tf_status tf_oc_update(const double *x, const double *dc, int64_t n, double volfrac, double move, double l1,
                       double l2, double tol, double *x_new, double *lmid_out, int32_t *iters_out, void *stream) {
    if (n < 1 || n >= (int64_t)0x7fffffff) {
        set_error("tf_oc_update: n out of range");
        return TF_ERR_INVALID;
    }
    if (!isfinite(volfrac) || !(volfrac > 0) || !isfinite(move) || !(move >= 0) || !isfinite(l1) ||
        !isfinite(l2) || !(l2 >= l1) || !(tol > 0)) {
        set_error("tf_oc_update: invalid volfrac/move/l1/l2/tol");
        return TF_ERR_INVALID;
    }
    TF_TRY(require_device(x, "x"));
    TF_TRY(require_device(dc, "dc"));
    TF_TRY(require_device(x_new, "x_new"));
    TF_TRY(require_device(lmid_out, "lmid_out"));
    if (iters_out) TF_TRY(require_device(iters_out, "iters_out"));
    return oc_update(x, dc, n, volfrac, move, l1, l2, tol, x_new, lmid_out, iters_out, (cudaStream_t)stream);
}

void tf_free(tf_filter h) { destroy(h); }

}  // extern "C"
