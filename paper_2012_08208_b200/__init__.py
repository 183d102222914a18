"""Python binding of libtopofilt (include/topofilt.h): argument marshalling only.

Every step of the filter path runs in the CUDA kernels of libtopofilt.so (built in-tree
for sm_100a by ``_build.py``); this module only passes device pointers, sizes and the
current torch CUDA stream through ctypes. There is no CPU fallback: if the shared
library is missing, importing this package raises.

Names mirror the C ABI: ``tf_build_filter``, ``tf_sensitivity_filter``,
``tf_density_filter``, ``tf_filter_view``, ``tf_free`` (+ ``*_host`` variants), and a
convenience ``Filter`` object returned by ``tf_build_filter``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TOPOFILT_LIB") or os.path.join(_HERE, "libtopofilt.so")  # override: tuning variants

TF_OK, TF_ERR_INVALID, TF_ERR_NOMEM, TF_ERR_CUDA, TF_ERR_OVERFLOW = range(5)
_STATUS = {0: "TF_OK", 1: "TF_ERR_INVALID", 2: "TF_ERR_NOMEM", 3: "TF_ERR_CUDA", 4: "TF_ERR_OVERFLOW"}

# Every symbol include/topofilt.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "tf_build_filter", "tf_build_filter_ex", "tf_lattice_detect_host", "tf_filter_view", "tf_build_stats", "tf_sensitivity_filter", "tf_density_filter",
    "tf_free", "tf_last_error", "tf_build_filter_host", "tf_sensitivity_filter_host",
    "tf_density_filter_host", "tf_filter_from_csr", "tf_kernel_launches", "tf_debug_set_alloc_limit",
    "tf_version", "tf_build_stencil", "tf_filter_nnz", "tf_oc_update", "tf_sensitivity_filter_energy",
    "tf_filter_iteration_host", "tf_filter_both", "tf_build_lattice", "tf_halo_pack",
    "tf_sensitivity_filter_range", "tf_density_filter_range", "tf_gather_rows",
    "tf_shard_plan", "tf_shard_view_get", "tf_shard_counts", "tf_shard_free",
    "tf_sensitivity_filter_rows", "tf_density_filter_rows",
    # include/topofilt_helmholtz.h (NEXT-3)
    "tf_helmholtz_build", "tf_helmholtz_filter", "tf_helmholtz_sensitivity", "tf_helmholtz_view",
    "tf_helmholtz_free",
]


# tf_build_filter_ex flags (TF_BUILD_*) and tf_build_info.path values (TF_PATH_*)
BUILD_FLAGS = {"auto": 0, "cell_list": 1, "lattice": 2, "cell_list_bins": 3, "dense": 4}
BUILD_PATHS = {0: "cell_list", 1: "lattice_tested", 2: "lattice_exact", 3: "dense"}


class TopofiltError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class tf_view(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("dim", ctypes.c_int32),
                ("rmin", ctypes.c_double), ("rowptr", ctypes.c_void_p), ("cols", ctypes.c_void_p),
                ("vals", ctypes.c_void_p), ("hs", ctypes.c_void_p)]


class tf_build_info(ctypes.Structure):
    _fields_ = [("bin_side", ctypes.c_double), ("bins", ctypes.c_int64 * 3), ("nbins", ctypes.c_int64),
                ("max_candidates", ctypes.c_int64), ("large_rows", ctypes.c_int64),
                ("radix_passes", ctypes.c_int32), ("path", ctypes.c_int32), ("groups", ctypes.c_int64)]


class tf_shard_view(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("axis", ctypes.c_int32),
                ("cut_lo", ctypes.c_double), ("cut_hi", ctypes.c_double), ("n_interior", ctypes.c_int64),
                ("n_owned", ctypes.c_int64), ("n_halo", ctypes.c_int64), ("local_ids", ctypes.c_void_p),
                ("send_idx", ctypes.c_void_p)]


class tf_helmholtz_info(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32), ("rel_residual", ctypes.c_double)]


class tf_helmholtz_system(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("n_cells", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("dim", ctypes.c_int32), ("R", ctypes.c_double), ("rowptr", ctypes.c_void_p),
                ("cols", ctypes.c_void_p), ("vals_A", ctypes.c_void_p), ("vals_M", ctypes.c_void_p),
                ("node_weight", ctypes.c_void_p), ("cell_volume", ctypes.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtopofilt.so not built at {LIB_PATH}: run `python __graft_entry__.py build` "
                          "(the CUDA path has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "tf_build_filter": ([P, I64, I32, D, P, PP], I32),
        "tf_build_filter_ex": ([P, I64, I32, D, I32, P, PP], I32),
        "tf_lattice_detect_host": ([P, I64, I32, P, P, P], I32),
        "tf_build_filter_host": ([P, I64, I32, D, P, PP], I32),
        "tf_filter_view": ([P, ctypes.POINTER(tf_view)], I32),
        "tf_build_stats": ([P, ctypes.POINTER(tf_build_info)], I32),
        "tf_sensitivity_filter": ([P, P, P, P, P], I32),
        "tf_density_filter": ([P, P, P, P], I32),
        "tf_sensitivity_filter_rows": ([P, P, P, P, I64, P], I32),
        "tf_density_filter_rows": ([P, P, P, I64, P], I32),
        "tf_sensitivity_filter_host": ([P, P, P, P, P], I32),
        "tf_density_filter_host": ([P, P, P, P], I32),
        "tf_filter_from_csr": ([P, P, P, P, I64, P, PP], I32),
        "tf_free": ([P], None),
        "tf_last_error": ([], ctypes.c_char_p),
        "tf_kernel_launches": ([], ctypes.c_uint64),
        "tf_debug_set_alloc_limit": ([ctypes.c_uint64], None),
        "tf_version": ([], I32),
        "tf_build_stencil": ([I32, I64, I64, I64, D, D, P, PP], I32),
        "tf_filter_nnz": ([P], I64),
        "tf_oc_update": ([P, P, I64, D, D, D, D, D, P, P, P, P], I32),
        "tf_sensitivity_filter_energy": ([P, P, P, D, P, P], I32),
        "tf_filter_iteration_host": ([P, P, P, P, P, P], I32),
        "tf_filter_both": ([P, P, P, P, P, P], I32),
        "tf_build_lattice": ([I32, I64, I64, I64, D, I32, P, D, P, PP], I32),
        "tf_halo_pack": ([P, P, I64, P, P], I32),
        "tf_sensitivity_filter_range": ([P, P, P, P, I64, I64, P], I32),
        "tf_density_filter_range": ([P, P, P, I64, I64, P], I32),
        "tf_shard_plan": ([P, I64, I32, D, I32, I32, P, PP], I32),
        "tf_shard_view_get": ([P, ctypes.POINTER(tf_shard_view)], I32),
        "tf_shard_counts": ([P, P, P], I32),
        "tf_shard_free": ([P], None),
        "tf_gather_rows": ([P, I32, P, I64, P, P], I32),
        "tf_helmholtz_build": ([P, I64, P, I64, I32, D, P, PP], I32),
        "tf_helmholtz_filter": ([P, P, P, D, I32, P, P], I32),
        "tf_helmholtz_sensitivity": ([P, P, P, P, D, I32, P, P], I32),
        "tf_helmholtz_view": ([P, ctypes.POINTER(tf_helmholtz_system)], I32),
        "tf_helmholtz_free": ([P], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


_lib = _load()


def lib():
    return _lib


def _check(status: int):
    if status != TF_OK:
        raise TopofiltError(status, _lib.tf_last_error().decode(errors="replace"))


def _stream_ptr(stream=None, device=None):
    """None -> torch's current CUDA stream (of `device` if given); 0 -> the legacy default stream;
    else a torch.cuda.Stream."""
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    import torch
    s = torch.cuda.current_stream(device) if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dptr(t, name, dtype=None, numel=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch.Tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {t.numel()}")
    return ctypes.c_void_p(t.data_ptr())


class _CudaArray:
    """Minimal __cuda_array_interface__ wrapper for zero-copy torch views of handle memory."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class Filter:
    """A built filter (owns a tf_filter handle). Immutable; applies are stream-ordered."""

    def __init__(self, handle: ctypes.c_void_p, keepalive=None, stencil=None):
        self._h = handle
        self._keep = keepalive
        self.is_stencil = stencil is not None
        if self.is_stencil:  # matrix-free: no CSR view
            self.dim, self.rmin, self.n = stencil
            self.nnz = int(_lib.tf_filter_nnz(self._h))
            self._v = None
            return
        v = tf_view()
        _check(_lib.tf_filter_view(self._h, ctypes.byref(v)))
        self.n, self.nnz, self.dim, self.rmin = v.n, v.nnz, v.dim, v.rmin
        self._v = v

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("filter is closed")
        return self._h

    def sensitivity(self, x, dc, out=None, stream=None, rows=None):
        """dc~ = H(x∘dc) / (Hs∘max(1e-3, x)) (Eq. filter_mat).
        rows: only rows [0, rows) are guaranteed (tf_sensitivity_filter_rows)."""
        import torch
        if out is None:
            out = torch.empty_like(x)
        if rows is None:
            tf_sensitivity_filter(self, x, dc, out, stream)
        else:
            tf_sensitivity_filter_rows(self, x, dc, out, rows, stream)
        return out

    def density(self, x, out=None, stream=None, rows=None):
        """x~ = Hx / Hs (BASELINE.json north_star). rows: as in sensitivity."""
        import torch
        if out is None:
            out = torch.empty_like(x)
        if rows is None:
            tf_density_filter(self, x, out, stream)
        else:
            tf_density_filter_rows(self, x, out, rows, stream)
        return out

    def both(self, x, dc, sens_out=None, dens_out=None, stream=None):
        """Both filters in one pass over H; returns (sensitivity, density)."""
        return tf_filter_both(self, x, dc, sens_out, dens_out, stream)

    def csr(self):
        """Zero-copy torch views (rowptr int64, cols int32, vals f64, hs f64) tied to this handle."""
        import torch
        v = self._v
        if v is None:  # matrix-free handle: the C ABI reports it (TF_ERR_INVALID)
            v = tf_view()
            _check(_lib.tf_filter_view(self.handle, ctypes.byref(v)))
        mk = lambda p, n, t: torch.as_tensor(_CudaArray(p, (n,), t), device="cuda")
        return (mk(v.rowptr, self.n + 1, "<i8"), mk(v.cols, self.nnz, "<i4"),
                mk(v.vals, self.nnz, "<f8"), mk(v.hs, self.n, "<f8"))

    def stats(self) -> dict:
        info = tf_build_info()
        _check(_lib.tf_build_stats(self.handle, ctypes.byref(info)))
        return {"bin_side": info.bin_side, "bins": list(info.bins), "nbins": info.nbins,
                "max_candidates": info.max_candidates, "large_rows": info.large_rows,
                "radix_passes": info.radix_passes, "path": BUILD_PATHS[info.path], "groups": info.groups}

    def sensitivity_host(self, x: np.ndarray, dc: np.ndarray, out: np.ndarray | None = None, stream=None):
        return tf_sensitivity_filter_host(self, x, dc, out, stream)

    def density_host(self, x: np.ndarray, out: np.ndarray | None = None, stream=None):
        return tf_density_filter_host(self, x, out, stream)

    def close(self):
        if self._h is not None:
            _lib.tf_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


# ------------------------------------------------------------------ C-ABI-named functions

def tf_build_filter(centroids, rmin: float, stream=None, path: str = "auto") -> Filter:
    """Build H (CSR) and Hs from device centroids [N, dim] float64.
    path: "auto" (tf_build_filter: lattice detection, else the cell list), "cell_list" or
    "lattice" (tf_build_filter_ex with TF_BUILD_CELL_LIST / TF_BUILD_LATTICE)."""
    import torch
    if centroids.dim() != 2:
        raise ValueError("centroids must be [N, dim]")
    n, dim = centroids.shape
    h = ctypes.c_void_p()
    ptr = _dptr(centroids, "centroids", torch.float64)
    if path == "auto":
        _check(_lib.tf_build_filter(ptr, n, dim, float(rmin), _stream_ptr(stream), ctypes.byref(h)))
    else:
        _check(_lib.tf_build_filter_ex(ptr, n, dim, float(rmin), BUILD_FLAGS[path], _stream_ptr(stream),
                                       ctypes.byref(h)))
    return Filter(h)


def tf_lattice_detect_host(centroids: np.ndarray):
    """Detection step of the lattice build on a host array (no GPU needed): returns None or
    {"T": cells per cube, "cubes": (nx, ny, nz), "spacing": (hx, hy, hz)}."""
    c = np.ascontiguousarray(centroids, dtype=np.float64)
    if c.ndim != 2:
        raise ValueError("centroids must be [N, dim]")
    T = ctypes.c_int32()
    cubes = (ctypes.c_int64 * 3)()
    sp = (ctypes.c_double * 3)()
    _check(_lib.tf_lattice_detect_host(c.ctypes.data_as(ctypes.c_void_p), c.shape[0], c.shape[1], ctypes.byref(T),
                                       cubes, sp))
    if T.value == 0:
        return None
    return {"T": T.value, "cubes": tuple(cubes), "spacing": tuple(sp)}


def tf_build_stencil(dim: int, nx: int, ny: int, nz: int, h: float, rmin: float, stream=None) -> Filter:
    """Matrix-free filter on a regular grid (row a10): cells (k*ny + j)*nx + i, spacing h."""
    hnd = ctypes.c_void_p()
    _check(_lib.tf_build_stencil(int(dim), int(nx), int(ny), int(nz), float(h), float(rmin), _stream_ptr(stream),
                                 ctypes.byref(hnd)))
    n = int(nx) * int(ny) * (int(nz) if dim == 3 else 1)
    return Filter(hnd, stencil=(int(dim), float(rmin), n))


def tf_build_lattice(dim: int, nx: int, ny: int, nz: int, h: float, type_offsets, rmin: float,
                     stream=None) -> Filter:
    """Matrix-free filter on a periodic lattice: cell T*((k*ny + j)*nx + i) + t at h*((i,j,k) + o_t)."""
    o = np.ascontiguousarray(type_offsets, dtype=np.float64)
    if o.ndim != 2 or o.shape[1] != dim:
        raise ValueError("type_offsets must be [ntypes, dim]")
    hnd = ctypes.c_void_p()
    _check(_lib.tf_build_lattice(int(dim), int(nx), int(ny), int(nz), float(h), int(o.shape[0]),
                                 o.ctypes.data_as(ctypes.c_void_p), float(rmin), _stream_ptr(stream),
                                 ctypes.byref(hnd)))
    n = int(nx) * int(ny) * (int(nz) if dim == 3 else 1) * int(o.shape[0])
    return Filter(hnd, stencil=(int(dim), float(rmin), n))


def tf_build_filter_host(centroids: np.ndarray, rmin: float, stream=None) -> Filter:
    c = np.ascontiguousarray(centroids, dtype=np.float64)
    n, dim = c.shape
    h = ctypes.c_void_p()
    _check(_lib.tf_build_filter_host(c.ctypes.data_as(ctypes.c_void_p), n, dim, float(rmin),
                                     _stream_ptr(stream), ctypes.byref(h)))
    return Filter(h)


def tf_sensitivity_filter(f: Filter, x, dc, out, stream=None):
    import torch
    _check(_lib.tf_sensitivity_filter(f.handle, _dptr(x, "x", torch.float64, f.n),
                                      _dptr(dc, "dc", torch.float64, f.n),
                                      _dptr(out, "out", torch.float64, f.n), _stream_ptr(stream)))
    return out


def tf_sensitivity_filter_energy(f: Filter, x, U, penal: float, out=None, stream=None):
    """NEXT-2: sensitivity filter of dc = -penal x^(penal-1) U, dc evaluated in-kernel."""
    import torch
    if out is None:
        out = torch.empty_like(x)
    _check(_lib.tf_sensitivity_filter_energy(f.handle, _dptr(x, "x", torch.float64, f.n),
                                             _dptr(U, "U", torch.float64, f.n), float(penal),
                                             _dptr(out, "out", torch.float64, f.n), _stream_ptr(stream)))
    return out


def tf_filter_both(f: Filter, x, dc, sens_out=None, dens_out=None, stream=None):
    """Sensitivity and density filter in one pass over H (bitwise equal to the separate calls)."""
    import torch
    if sens_out is None:
        sens_out = torch.empty_like(x)
    if dens_out is None:
        dens_out = torch.empty_like(x)
    _check(_lib.tf_filter_both(f.handle, _dptr(x, "x", torch.float64, f.n), _dptr(dc, "dc", torch.float64, f.n),
                               _dptr(sens_out, "sens_out", torch.float64, f.n),
                               _dptr(dens_out, "dens_out", torch.float64, f.n), _stream_ptr(stream)))
    return sens_out, dens_out


def tf_sensitivity_filter_rows(f: Filter, x, dc, out, nrows: int, stream=None):
    """Rows [0, nrows) of the sensitivity filter (NEXT-4: a shard's owned rows)."""
    import torch
    _check(_lib.tf_sensitivity_filter_rows(f.handle, _dptr(x, "x", torch.float64, f.n),
                                           _dptr(dc, "dc", torch.float64, f.n),
                                           _dptr(out, "out", torch.float64, f.n), int(nrows), _stream_ptr(stream)))
    return out


def tf_density_filter_rows(f: Filter, x, out, nrows: int, stream=None):
    """Rows [0, nrows) of the density filter."""
    import torch
    _check(_lib.tf_density_filter_rows(f.handle, _dptr(x, "x", torch.float64, f.n),
                                       _dptr(out, "out", torch.float64, f.n), int(nrows), _stream_ptr(stream)))
    return out


def tf_sensitivity_filter_range(f: Filter, x, dc, out, r0: int, r1: int, stream=None):
    """Rows [r0, r1) of the sensitivity filter (NEXT-4: interior rows during the halo exchange,
    then the boundary rows)."""
    import torch
    _check(_lib.tf_sensitivity_filter_range(f.handle, _dptr(x, "x", torch.float64, f.n),
                                            _dptr(dc, "dc", torch.float64, f.n),
                                            _dptr(out, "out", torch.float64, f.n), int(r0), int(r1),
                                            _stream_ptr(stream)))
    return out


def tf_density_filter_range(f: Filter, x, out, r0: int, r1: int, stream=None):
    """Rows [r0, r1) of the density filter."""
    import torch
    _check(_lib.tf_density_filter_range(f.handle, _dptr(x, "x", torch.float64, f.n),
                                        _dptr(out, "out", torch.float64, f.n), int(r0), int(r1),
                                        _stream_ptr(stream)))
    return out


def tf_gather_rows(src, idx, out, stream=None):
    """out[t] = src[idx[t]] for rows of a [*, dim] fp64 array (library kernel)."""
    import torch
    dim = 1 if src.dim() == 1 else src.shape[1]
    m = idx.numel()
    _check(_lib.tf_gather_rows(_dptr(src, "src", torch.float64), int(dim), _dptr(idx, "idx", torch.int32, m),
                               m, _dptr(out, "out", torch.float64, m * dim), _stream_ptr(stream, src.device)))
    return out


def tf_density_filter(f: Filter, x, out, stream=None):
    import torch
    _check(_lib.tf_density_filter(f.handle, _dptr(x, "x", torch.float64, f.n),
                                  _dptr(out, "out", torch.float64, f.n), _stream_ptr(stream)))
    return out


def _host(a, n, name, writable=False):
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous or a.size != n:
        raise TypeError(f"{name} must be a contiguous float64 numpy array of {n} elements")
    if writable and not a.flags.writeable:
        raise ValueError(f"{name} must be writable")
    return a.ctypes.data_as(ctypes.c_void_p)


def tf_sensitivity_filter_host(f: Filter, x, dc, out=None, stream=None):
    if out is None:
        out = np.empty(f.n, dtype=np.float64)
    _check(_lib.tf_sensitivity_filter_host(f.handle, _host(x, f.n, "x"), _host(dc, f.n, "dc"),
                                           _host(out, f.n, "out", True), _stream_ptr(stream)))
    return out


def tf_filter_iteration_host(f: Filter, x, dc, sens_out=None, dens_out=None, stream=None):
    """Both filters of one iteration on host arrays (x, dc uploaded once; D2H overlapped)."""
    if sens_out is None:
        sens_out = np.empty(f.n, dtype=np.float64)
    if dens_out is None:
        dens_out = np.empty(f.n, dtype=np.float64)
    _check(_lib.tf_filter_iteration_host(f.handle, _host(x, f.n, "x"), _host(dc, f.n, "dc"),
                                         _host(sens_out, f.n, "sens_out", True),
                                         _host(dens_out, f.n, "dens_out", True), _stream_ptr(stream)))
    return sens_out, dens_out


def tf_density_filter_host(f: Filter, x, out=None, stream=None):
    if out is None:
        out = np.empty(f.n, dtype=np.float64)
    _check(_lib.tf_density_filter_host(f.handle, _host(x, f.n, "x"), _host(out, f.n, "out", True),
                                       _stream_ptr(stream)))
    return out


def tf_filter_view(f: Filter):
    return f.csr()


def tf_free(f: Filter):
    f.close()


def tf_filter_from_csr(rowptr, cols, vals, hs, stream=None) -> Filter:
    """TEST HOOK: wrap a host CSR (e.g. the oracle's) so the apply kernels can be tested alone."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    hs = np.ascontiguousarray(hs, dtype=np.float64)
    n = rowptr.shape[0] - 1
    h = ctypes.c_void_p()
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _check(_lib.tf_filter_from_csr(p(rowptr), p(cols), p(vals), p(hs), n, _stream_ptr(stream),
                                   ctypes.byref(h)))
    return Filter(h)


def kernel_launches() -> int:
    return int(_lib.tf_kernel_launches())


def set_alloc_limit(nbytes: int):
    _lib.tf_debug_set_alloc_limit(int(nbytes))


def version() -> int:
    return int(_lib.tf_version())


def tf_oc_update(x, dc, volfrac: float, move: float = 0.2, l1: float = 0.0, l2: float = 100000.0,
                 tol: float = 1e-4, x_new=None, stream=None, flags: bool = False):
    """NEXT-1: OC update with bisection. Returns (x_new, lmid tensor[1], iters
    tensor[1]), plus the flags tensor[1] (TF_OC_* bits: 1 bracket exhausted, 2 no progress) when
    flags=True. Runs on x's device."""
    import torch
    n = x.numel()
    with torch.cuda.device(x.device):
        if x_new is None:
            x_new = torch.empty_like(x)
        lm = torch.empty(1, dtype=torch.float64, device=x.device)
        it = torch.empty(2, dtype=torch.int32, device=x.device)
        _check(_lib.tf_oc_update(_dptr(x, "x", torch.float64), _dptr(dc, "dc", torch.float64, n), n,
                                 float(volfrac), float(move), float(l1), float(l2), float(tol),
                                 _dptr(x_new, "x_new", torch.float64, n), _dptr(lm, "lmid"),
                                 ctypes.c_void_p(it.data_ptr()), _stream_ptr(stream, x.device)))
    if flags:
        return x_new, lm, it[:1], it[1:]
    return x_new, lm, it[:1]


# ------------------------------------------------------------------ NEXT-3: Helmholtz PDE filter

def helmholtz_radius(rmin: float) -> float:
    """R = rmin / (2 sqrt 3) (R17)."""
    return float(rmin) / (2.0 * 3.0 ** 0.5)


class Helmholtz:
    """A built Helmholtz filter (owns a tf_helmholtz handle; include/topofilt_helmholtz.h).
    Calls on one handle share its CG scratch: keep them on one stream."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        v = tf_helmholtz_system()
        _check(_lib.tf_helmholtz_view(self._h, ctypes.byref(v)))
        self._v = v
        self.n_nodes, self.n_cells, self.nnz, self.dim, self.R = v.n_nodes, v.n_cells, v.nnz, v.dim, v.R

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("Helmholtz filter is closed")
        return self._h

    def _info(self, device):
        import torch
        return torch.zeros(2, dtype=torch.float64, device=device)  # 16 bytes = tf_helmholtz_info

    @staticmethod
    def decode_info(t) -> dict:
        """(iterations, converged, rel_residual) from the 16-byte info tensor (synchronises)."""
        raw = t.cpu().numpy().tobytes()
        info = tf_helmholtz_info.from_buffer_copy(raw)
        return {"iterations": info.iterations, "converged": bool(info.converged), "rel_residual": info.rel_residual}

    def filter(self, sigma, out=None, rtol: float = 1e-12, maxit: int = 1000, info=None, stream=None):
        """s~ = Helmholtz(sigma) over cells. Returns (out, info tensor)."""
        import torch
        if out is None:
            out = torch.empty_like(sigma)
        if info is None:
            info = self._info(sigma.device)
        _check(_lib.tf_helmholtz_filter(self.handle, _dptr(sigma, "sigma", torch.float64, self.n_cells),
                                        _dptr(out, "out", torch.float64, self.n_cells), float(rtol), int(maxit),
                                        ctypes.c_void_p(info.data_ptr()), _stream_ptr(stream)))
        return out, info

    def sensitivity(self, x, dc, out=None, rtol: float = 1e-12, maxit: int = 1000, info=None, stream=None):
        """dc~ = Helmholtz(x∘dc) / max(1e-3, x). Returns (out, info tensor)."""
        import torch
        if out is None:
            out = torch.empty_like(x)
        if info is None:
            info = self._info(x.device)
        _check(_lib.tf_helmholtz_sensitivity(self.handle, _dptr(x, "x", torch.float64, self.n_cells),
                                             _dptr(dc, "dc", torch.float64, self.n_cells),
                                             _dptr(out, "out", torch.float64, self.n_cells), float(rtol), int(maxit),
                                             ctypes.c_void_p(info.data_ptr()), _stream_ptr(stream)))
        return out, info

    def system(self):
        """Zero-copy views (rowptr, cols, vals_A, vals_M, node_weight, cell_volume)."""
        import torch
        v = self._v
        mk = lambda p, n, t: torch.as_tensor(_CudaArray(p, (n,), t), device="cuda")  # noqa: E731
        return (mk(v.rowptr, self.n_nodes + 1, "<i8"), mk(v.cols, self.nnz, "<i4"), mk(v.vals_A, self.nnz, "<f8"),
                mk(v.vals_M, self.nnz, "<f8"), mk(v.node_weight, self.n_nodes, "<f8"),
                mk(v.cell_volume, self.n_cells, "<f8"))

    def close(self):
        if self._h is not None:
            _lib.tf_helmholtz_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tf_helmholtz_build(nodes, cells, R: float, stream=None) -> Helmholtz:
    """Assemble the Helmholtz filter: nodes [Nn, dim] float64, cells [Nc, dim+1] int32 (device)."""
    import torch
    if nodes.dim() != 2 or cells.dim() != 2 or cells.shape[1] != nodes.shape[1] + 1:
        raise ValueError("nodes must be [Nn, dim] and cells [Nc, dim+1]")
    h = ctypes.c_void_p()
    _check(_lib.tf_helmholtz_build(_dptr(nodes, "nodes", torch.float64), nodes.shape[0],
                                   _dptr(cells, "cells", torch.int32), cells.shape[0], nodes.shape[1], float(R),
                                   _stream_ptr(stream), ctypes.byref(h)))
    return Helmholtz(h)
