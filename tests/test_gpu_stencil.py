"""Matrix-free stencil filter against the oracle's CSR of the same
lattice centroids: both filters within 1e-10 relative; equivalent-CSR nnz exact."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL_OUT = 1e-10


@pytest.fixture(scope="module")
def tf():
    assert torch.cuda.is_available()
    import paper_2012_08208_b200 as m
    return m


def assert_rel(g, r, rtol, what):
    scale = np.where(r != 0, np.abs(r), np.abs(r).max())
    bad = np.abs(g - r) > rtol * scale
    assert not bad.any(), f"{what}: {bad.sum()} of {r.size} outside {rtol}"


def lattice(dim, nx, ny, nz, h):
    c = synth.hex_grid(nx, ny, nz) if dim == 3 else synth.quad_grid(nx, ny)
    return c * h


CASES = [
    # (dim, nx, ny, nz, h, rmin)
    (2, 60, 20, 1, 1.0, 1.5),       # config 1
    (3, 160, 80, 80, 1.0, 2.0),     # config 3
    (2, 37, 11, 1, 1.0, 2.5),
    (2, 33, 9, 1, 0.5, 1.6),
    (3, 37, 11, 5, 1.0, 1.5),
    (3, 19, 7, 6, 1.0, 3.2),
    (3, 21, 13, 9, 0.5, 1.0),
    (3, 8, 8, 8, 1.0, 0.9),         # diagonal only: filtered = input
    (3, 1, 1, 1, 1.0, 2.0),         # single cell
]


@pytest.mark.parametrize("dim,nx,ny,nz,h,rmin", CASES)
def test_stencil_matches_oracle(tf, dim, nx, ny, nz, h, rmin):
    c = lattice(dim, nx, ny, nz, h)
    n = c.shape[0]
    ref = oracle.build_celllist(c, rmin)
    f = tf.tf_build_stencil(dim, nx, ny, nz, h, rmin)
    assert f.nnz == ref.nnz
    x = synth.uniform(31, 0, n, 0.001, 1.0)
    dc = (-3.0 * (x * x)) * synth.uniform(32, 0, n, 0.5, 1.5)
    xs, dcs = torch.from_numpy(x).cuda(), torch.from_numpy(dc).cuda()
    assert_rel(f.sensitivity(xs, dcs).cpu().numpy(), oracle.apply_sensitivity(ref, x, dc), RTOL_OUT, "stencil sens")
    assert_rel(f.density(xs).cpu().numpy(), oracle.apply_density(ref, x), RTOL_OUT, "stencil dens")
    f.close()


def test_stencil_equals_csr_path(tf):
    """Same outputs as the stored-CSR path on config 3 (both GPU)."""
    c, x, dc, rmin = synth.workload(3)
    fc = tf.tf_build_filter(torch.from_numpy(c).cuda(), rmin)
    fs = tf.tf_build_stencil(3, 160, 80, 80, 1.0, rmin)
    assert fs.nnz == fc.nnz
    xs, dcs = torch.from_numpy(x).cuda(), torch.from_numpy(dc).cuda()
    a, b = fc.sensitivity(xs, dcs).cpu().numpy(), fs.sensitivity(xs, dcs).cpu().numpy()
    assert_rel(b, a, 1e-12, "stencil vs csr")


def test_stencil_host_variant_and_errors(tf):
    f = tf.tf_build_stencil(2, 30, 10, 1, 1.0, 1.5)
    x = synth.uniform(33, 0, 300, 0.001, 1.0)
    d_host = f.density_host(x)
    np.testing.assert_array_equal(d_host, f.density(torch.from_numpy(x).cuda()).cpu().numpy())
    assert f.is_stencil
    import ctypes
    v = tf.tf_view()
    assert tf.lib().tf_filter_view(f.handle, ctypes.byref(v)) == tf.TF_ERR_INVALID
    with pytest.raises(tf.TopofiltError):
        tf.tf_build_stencil(4, 3, 3, 3, 1.0, 1.5)
    with pytest.raises(tf.TopofiltError):
        tf.tf_build_stencil(3, 3, 3, 3, 1.0, 50.0)  # too many offsets
    with pytest.raises(tf.TopofiltError):
        tf.tf_build_stencil(3, 3, 3, 3, 0.0, 1.5)
