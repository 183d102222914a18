"""The C-ABI library loads and exports every symbol include/topofilt.h declares; host-side
argument validation (no GPU needed: these paths return before any CUDA call)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2012_08208_b200 as tf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = sorted(os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))
                 if f.endswith(".h"))


def declared():
    src = "".join(open(h).read() for h in HEADERS)
    return sorted(set(re.findall(r"TF_API\s+[\w\s\*]*?\b(tf_\w+)\s*\(", src)))


def test_header_declares_expected_calls():
    names = declared()
    for must in ("tf_build_filter", "tf_sensitivity_filter", "tf_density_filter", "tf_free"):
        assert must in names
    assert sorted(tf.EXPORTS) == names


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(tf.LIB_PATH)
    for name in declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", tf.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tf_\w+)", out))
    assert set(declared()) <= exported
    # nothing else leaks out of the library (hidden visibility)
    assert exported == set(declared())


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", tf.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for other in ("sm_90", "sm_80", "sm_103"):
        assert other not in out


def test_version_and_counters():
    assert tf.version() == 1
    assert tf.kernel_launches() >= 0


def _build_status(ptr, n, dim, rmin, out=True):
    h = ctypes.c_void_p()
    st = tf.lib().tf_build_filter(ptr, n, dim, rmin, None, ctypes.byref(h) if out else None)
    return st, tf.lib().tf_last_error().decode()


@pytest.mark.parametrize("n,dim,rmin,frag", [
    (10, 4, 1.0, "dim"), (10, 1, 1.0, "dim"), (0, 2, 1.0, "n must"), (-5, 3, 1.0, "n must"),
    (2 ** 31, 3, 1.0, "n must"), (10, 2, 0.0, "rmin"), (10, 2, -1.0, "rmin"),
    (10, 3, float("nan"), "rmin"), (10, 3, float("inf"), "rmin"),
])
def test_build_rejects_bad_arguments(n, dim, rmin, frag):
    st, msg = _build_status(ctypes.c_void_p(0x1000), n, dim, rmin)
    assert st == tf.TF_ERR_INVALID and frag in msg


def test_build_rejects_null_out():
    st, msg = _build_status(ctypes.c_void_p(0x1000), 10, 2, 1.0, out=False)
    assert st == tf.TF_ERR_INVALID


def test_from_csr_validates_on_host():
    rowptr = np.array([0, 2, 1], dtype=np.int64)  # not monotone
    with pytest.raises(tf.TopofiltError, match="monotone"):
        tf.tf_filter_from_csr(rowptr, np.array([0, 1], np.int32), np.ones(2), np.ones(2), stream=0)
    with pytest.raises(tf.TopofiltError, match="out of range"):
        tf.tf_filter_from_csr(np.array([0, 1, 2]), np.array([0, 5], np.int32), np.ones(2), np.ones(2), stream=0)
    with pytest.raises(tf.TopofiltError, match=r"rowptr\[0\]"):
        tf.tf_filter_from_csr(np.array([1, 1, 2]), np.array([0, 1], np.int32), np.ones(2), np.ones(2), stream=0)


def test_apply_null_handle_rejected():
    st = tf.lib().tf_density_filter(None, None, None, None)
    assert st == tf.TF_ERR_INVALID
    st = tf.lib().tf_sensitivity_filter_host(None, None, None, None, None)
    assert st == tf.TF_ERR_INVALID


def test_free_null_is_noop():
    tf.lib().tf_free(None)


def test_no_oracle_in_product():
    """The product package neither imports nor links the oracle (independence rule)."""
    pkg = os.path.join(ROOT, "paper_2012_08208_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "oracle.h" not in src
    ldd = subprocess.run(["ldd", tf.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in ldd


@pytest.mark.parametrize("nn,nc,dim,R,frag", [
    (10, 5, 4, 1.0, "dim"), (0, 5, 2, 1.0, "n_nodes"), (2 ** 31, 5, 3, 1.0, "n_nodes"), (10, 0, 2, 1.0, "n_nodes"),
    (10, 5, 2, -1.0, "R must"), (10, 5, 3, float("nan"), "R must"), (10, 5, 2, float("inf"), "R must"),
    (10, 2 ** 27, 3, 1.0, "2^31"),
])
def test_helmholtz_build_rejects_bad_args(nn, nc, dim, R, frag):
    """NEXT-3 argument validation happens before any CUDA call."""
    h = ctypes.c_void_p()
    st = tf.lib().tf_helmholtz_build(None, nn, None, nc, dim, R, None, ctypes.byref(h))
    assert st in (tf.TF_ERR_INVALID, tf.TF_ERR_OVERFLOW)
    assert frag in tf.lib().tf_last_error().decode()
    assert not h.value
