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


# ------------------------------------------------------------------ periodic lattices (tf_build_lattice)

def lattice_cells(kind, nx, ny, nz):
    if kind == "kuhn":
        return synth.kuhn_tets(nx, ny, nz), synth.kuhn_lattice_offsets(), 3
    return synth.tri_grid(nx, ny, kind), synth.tri_lattice_offsets(kind), 2


LATTICE_CASES = [
    # (kind, nx, ny, nz, rmin)
    ("right", 300, 100, 1, 2.5),    # config 2
    ("left", 41, 13, 1, 1.7),
    ("right", 3, 2, 1, 4.0),         # every cell near the boundary, reach > grid
    ("kuhn", 20, 12, 10, 1.5),       # config 5's lattice, scaled down
    ("kuhn", 9, 7, 5, 2.2),
    ("kuhn", 2, 2, 1, 1.5),          # boundary-only tiles
    ("kuhn", 4, 3, 3, 0.3),          # diagonal only
]


@pytest.mark.parametrize("kind,nx,ny,nz,rmin", LATTICE_CASES)
def test_lattice_matches_oracle(tf, kind, nx, ny, nz, rmin):
    """Both filters of the matrix-free lattice vs the oracle's CSR of the same centroids (1e-10);
    equivalent nnz exact; the device CSR path on the same centroids agrees too."""
    c, offs, dim = lattice_cells(kind, nx, ny, nz)
    n = c.shape[0]
    ref = oracle.build_celllist(c, rmin)
    f = tf.tf_build_lattice(dim, nx, ny, nz, 1.0, offs, rmin)
    assert f.n == n and f.nnz == ref.nnz
    x = synth.uniform(41, 0, n, 0.001, 1.0)
    dc = (-3.0 * (x * x)) * synth.uniform(42, 0, n, 0.5, 1.5)
    xs, dcs = torch.from_numpy(x).cuda(), torch.from_numpy(dc).cuda()
    s = f.sensitivity(xs, dcs).cpu().numpy()
    d = f.density(xs).cpu().numpy()
    assert_rel(s, oracle.apply_sensitivity(ref, x, dc), RTOL_OUT, "lattice sens")
    assert_rel(d, oracle.apply_density(ref, x), RTOL_OUT, "lattice dens")
    sb, db = f.both(xs, dcs)
    assert np.array_equal(sb.cpu().numpy(), s) and np.array_equal(db.cpu().numpy(), d)
    s2, d2 = tf.tf_filter_iteration_host(f, x, dc)
    assert np.array_equal(s2, s) and np.array_equal(d2, d)
    f.close()


def test_lattice_config5_vs_csr(tf):
    """Config 5 (12M Kuhn tets): the lattice filters agree with the stored-CSR path on every
    cell (1e-10 relative) and the equivalent nnz is the lattice count 1,030,251,952."""
    c, x, dc, rmin = synth.workload(5)
    xs, dcs = torch.from_numpy(x).cuda(), torch.from_numpy(dc).cuda()
    f = tf.tf_build_lattice(3, 200, 100, 100, 1.0, synth.kuhn_lattice_offsets(), rmin)
    assert f.nnz == 1_030_251_952
    s_l, d_l = f.sensitivity(xs, dcs).cpu().numpy(), f.density(xs).cpu().numpy()
    f.close()
    g = tf.tf_build_filter(torch.from_numpy(c).cuda(), rmin)
    s_c, d_c = g.sensitivity(xs, dcs).cpu().numpy(), g.density(xs).cpu().numpy()
    g.close()
    assert_rel(s_l, s_c, RTOL_OUT, "c5 lattice vs CSR sens")
    assert_rel(d_l, d_c, RTOL_OUT, "c5 lattice vs CSR dens")


def test_lattice_rejects_bad_args(tf):
    o = synth.kuhn_lattice_offsets()
    for args in [(3, 4, 4, 4, 1.0, np.zeros((0, 3)), 1.5), (3, 4, 4, 4, 1.0, np.zeros((9, 3)), 1.5),
                 (3, 4, 4, 4, 1.0, o + 0.5, 1.5), (3, 4, 4, 4, 1.0, -o, 1.5), (3, 4, 4, 4, 0.0, o, 1.5),
                 (3, 4, 4, 4, 1.0, o, 40.0), (3, 0, 4, 4, 1.0, o, 1.5)]:
        with pytest.raises(tf.TopofiltError):
            tf.tf_build_lattice(*args)
    f = tf.tf_build_lattice(3, 4, 4, 4, 1.0, o, 1.5)
    with pytest.raises(tf.TopofiltError):
        tf.tf_filter_view(f)
    f.close()
