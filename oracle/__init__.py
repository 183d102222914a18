"""ctypes wrapper of the plain C oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py. The product package
(paper_2012_08208_b200) never imports this module.

Every function here marshals numpy arrays into oracle.c and back; the arithmetic
lives in oracle.c, whose header cites the paper passages it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.or_bf_rowptr.argtypes = [P, I64, ctypes.c_int, ctypes.c_double, P]
        L.or_bf_rowptr.restype = I64
        L.or_bf_fill.argtypes = [P, I64, ctypes.c_int, ctypes.c_double, P, P, P, P]
        L.or_bf_fill.restype = None
        L.or_bf_rows_rowptr.argtypes = [P, I64, ctypes.c_int, ctypes.c_double, P, I64, P]
        L.or_bf_rows_rowptr.restype = I64
        L.or_bf_rows_fill.argtypes = [P, I64, ctypes.c_int, ctypes.c_double, P, I64, P, P, P, P]
        L.or_bf_rows_fill.restype = None
        L.or_cl_create.argtypes = [P, I64, ctypes.c_int, ctypes.c_double, ctypes.c_double]
        L.or_cl_create.restype = P
        L.or_cl_free.argtypes = [P]
        L.or_cl_free.restype = None
        L.or_cl_binside.argtypes = [P]
        L.or_cl_binside.restype = ctypes.c_double
        L.or_cl_nbins.argtypes = [P]
        L.or_cl_nbins.restype = I64
        L.or_cl_rowptr.argtypes = [P, P, I64, P]
        L.or_cl_rowptr.restype = I64
        L.or_cl_fill.argtypes = [P, P, I64, P, P, P, P]
        L.or_cl_fill.restype = None
        L.or_apply_sensitivity.argtypes = [I64, P, P, P, P, P, P, P, P]
        L.or_apply_sensitivity.restype = None
        L.or_apply_density.argtypes = [I64, P, P, P, P, P, P, P]
        L.or_apply_density.restype = None
        L.or_oc_update.argtypes = [I64, P, P, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_double, P, P, P]
        L.or_oc_update.restype = ctypes.c_int
        L.or_compliance_sensitivity.argtypes = [I64, P, P, ctypes.c_double, P]
        L.or_compliance_sensitivity.restype = None
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


@dataclass
class CSR:
    """Oracle CSR. `rows[r]` is the global row index of CSR row r (None: all rows)."""
    rowptr: np.ndarray   # int64 [m+1]
    cols: np.ndarray     # int32 [nnz]
    vals: np.ndarray     # float64 [nnz]
    hs: np.ndarray       # float64 [m]
    rows: np.ndarray | None = None

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def dense(self, n: int) -> np.ndarray:
        m = self.rowptr.shape[0] - 1
        d = np.zeros((m, n))
        for r in range(m):
            s, e = self.rowptr[r], self.rowptr[r + 1]
            d[r, self.cols[s:e]] = self.vals[s:e]
        return d


def build_bruteforce(c: np.ndarray, rmin: float) -> CSR:
    """O1: brute force over all pairs (Eq. filter_cond; listing PAPER.md:442-445)."""
    c = _c64(c)
    n, dim = c.shape
    rowptr = np.empty(n + 1, dtype=np.int64)
    nnz = lib().or_bf_rowptr(_p(c), n, dim, float(rmin), _p(rowptr))
    cols = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64)
    hs = np.empty(n, dtype=np.float64)
    lib().or_bf_fill(_p(c), n, dim, float(rmin), _p(rowptr), _p(cols), _p(vals), _p(hs))
    return CSR(rowptr, cols, vals, hs)


def build_bruteforce_rows(c: np.ndarray, rmin: float, rows: np.ndarray) -> CSR:
    """O1 on the listed rows only, each tested against all N points."""
    c = _c64(c)
    n, dim = c.shape
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    m = rows.shape[0]
    rowptr = np.empty(m + 1, dtype=np.int64)
    nnz = lib().or_bf_rows_rowptr(_p(c), n, dim, float(rmin), _p(rows), m, _p(rowptr))
    cols = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64)
    hs = np.empty(m, dtype=np.float64)
    lib().or_bf_rows_fill(_p(c), n, dim, float(rmin), _p(rows), m, _p(rowptr), _p(cols), _p(vals), _p(hs))
    return CSR(rowptr, cols, vals, hs, rows)


class CellList:
    """O2: plain uniform cell list (bin side >= rmin*(1+1e-6)*bin_factor)."""

    def __init__(self, c: np.ndarray, rmin: float, bin_factor: float = 1.0):
        self.c = _c64(c)
        self.n, self.dim = self.c.shape
        self.rmin = float(rmin)
        self._h = lib().or_cl_create(_p(self.c), self.n, self.dim, self.rmin, float(bin_factor))
        if not self._h:
            raise ValueError("invalid cell-list arguments")

    @property
    def bin_side(self) -> float:
        return lib().or_cl_binside(self._h)

    @property
    def nbins(self) -> int:
        return lib().or_cl_nbins(self._h)

    def rows(self, rows: np.ndarray | None = None) -> CSR:
        if rows is not None:
            rows = np.ascontiguousarray(rows, dtype=np.int64)
            m = rows.shape[0]
        else:
            m = self.n
        rowptr = np.empty(m + 1, dtype=np.int64)
        nnz = lib().or_cl_rowptr(self._h, _p(rows), m, _p(rowptr))
        cols = np.empty(nnz, dtype=np.int32)
        vals = np.empty(nnz, dtype=np.float64)
        hs = np.empty(m, dtype=np.float64)
        lib().or_cl_fill(self._h, _p(rows), m, _p(rowptr), _p(cols), _p(vals), _p(hs))
        return CSR(rowptr, cols, vals, hs, rows)

    def close(self):
        if self._h:
            lib().or_cl_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_celllist(c: np.ndarray, rmin: float, bin_factor: float = 1.0) -> CSR:
    cl = CellList(c, rmin, bin_factor)
    try:
        return cl.rows()
    finally:
        cl.close()


def apply_sensitivity(H: CSR, x: np.ndarray, dc: np.ndarray) -> np.ndarray:
    """O3: out_i = sum_j H_ij (x_j dc_j) / (Hs_i max(1e-3, x_i)) (Eq. filter_mat)."""
    x = _c64(x)
    dc = _c64(dc)
    m = H.rowptr.shape[0] - 1
    out = np.empty(m, dtype=np.float64)
    rows = None if H.rows is None else np.ascontiguousarray(H.rows, dtype=np.int64)
    lib().or_apply_sensitivity(m, _p(rows), _p(H.rowptr), _p(H.cols), _p(H.vals), _p(H.hs),
                               _p(x), _p(dc), _p(out))
    return out


def apply_density(H: CSR, x: np.ndarray) -> np.ndarray:
    """O3: out_i = sum_j H_ij x_j / Hs_i (BASELINE.json north_star)."""
    x = _c64(x)
    m = H.rowptr.shape[0] - 1
    out = np.empty(m, dtype=np.float64)
    rows = None if H.rows is None else np.ascontiguousarray(H.rows, dtype=np.int64)
    lib().or_apply_density(m, _p(rows), _p(H.rowptr), _p(H.cols), _p(H.vals), _p(H.hs),
                           _p(x), _p(out))
    return out


def oc_update(d: np.ndarray, dc: np.ndarray, volfrac: float, move: float = 0.2, l1: float = 0.0,
              l2: float = 100000.0, tol: float = 1e-4, flags: bool = False):
    """NEXT-1: OC update with bisection (Eq. update; listing PAPER.md:380-385),
    exact-sum branch decisions (R15), termination rule R23. Returns (density_new,
    last l_mid, iterations), plus the flags word (bit 0 bracket exhausted, bit 1 no progress)
    when flags=True."""
    d = _c64(d)
    dc = _c64(dc)
    out = np.empty_like(d)
    lm = np.zeros(1)
    fl = np.zeros(1, dtype=np.int32)
    it = lib().or_oc_update(d.shape[0], _p(d), _p(dc), float(volfrac), float(move), float(l1), float(l2),
                            float(tol), _p(out), _p(lm), fl.ctypes.data)
    if flags:
        return out, float(lm[0]), int(it), int(fl[0])
    return out, float(lm[0]), int(it)


def compliance_sensitivity(x: np.ndarray, U: np.ndarray, penal: float) -> np.ndarray:
    """NEXT-2: dc = -penal * x**(penal-1) * U (listing PAPER.md:376)."""
    x = _c64(x)
    U = _c64(U)
    out = np.empty_like(x)
    lib().or_compliance_sensitivity(x.shape[0], _p(x), _p(U), float(penal), _p(out))
    return out
