"""GPU parity of the lattice build path (tf_build_filter_ex / auto detection).

The lattice path must produce the same CSR as the cell-list path and the oracle: rowptr, cols and
vals bit-exact, Hs within 1e-12 relative, filters within 1e-10. Covered: the paper's lattice
meshes (quads, "right" triangles with fp-decided ties, hexes, Kuhn tetrahedra), anisotropic
spacings, shifted origins, single rows/layers, large and tiny reach, T = 3 random offsets,
near-lattices (tested mode with a deviation margin), and inputs that must NOT take the path
(permuted ids, alternating triangles, large displacements, nx = 1), which fall back to the cell
list (auto) or are rejected (path="lattice").
"""
import numpy as np
import pytest

import oracle
import synth
from test_gpu_parity import RTOL_OUT, assert_rel, compare_applies, compare_full, dev, inputs_for

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tf():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2012_08208_b200 as m
    return m


def _t3_lattice(nx, ny, stream):
    """2D lattice with three cells per square at seeded offsets (not dyadic)."""
    off = synth.uniform(stream, 0, 6, 0.0, 1.0).reshape(3, 2)
    j, i = np.meshgrid(np.arange(ny, dtype=np.float64), np.arange(nx, dtype=np.float64), indexing="ij")
    base = np.stack([i.ravel(), j.ravel()], 1)
    return (base[:, None, :] + off[None, :, :]).reshape(-1, 2)


def _displace_tail(c, frac, amount, stream):
    """Displace the last `frac` of the points by up to `amount` per component (prefix intact)."""
    c = c.copy()
    n = c.shape[0]
    k = int(n * frac)
    c[n - k:] += synth.uniform(stream, 0, k * c.shape[1], -amount, amount).reshape(k, c.shape[1])
    return c


def _lattice_cases():
    # name, centroids, rmin, expected path
    yield "c1_quads", synth.quad_grid(60, 20), 1.5, "lattice_exact"
    yield "c2_tri_right", synth.tri_grid(300, 100, "right"), 2.5, "lattice_tested"
    yield "spec_8x4_right_rmin2", synth.tri_grid(8, 4, "right"), 2.0, "lattice_tested"
    yield "e01_180x60_rmin2", synth.tri_grid(180, 60, "right"), 2.0, "lattice_tested"
    yield "e03_180x60_rmin3", synth.tri_grid(180, 60, "right"), 3.0, "lattice_tested"
    yield "tri_left", synth.tri_grid(70, 40, "left"), 2.2, "lattice_tested"
    yield "hex_40x20x20_ties", synth.hex_grid(40, 20, 20), 2.0, "lattice_exact"
    yield "kuhn_spec_6x4x2", synth.kuhn_tets(6, 4, 2), 1.5, "lattice_exact"
    yield "kuhn_e02_60x20x4", synth.kuhn_tets(60, 20, 4), 1.5, "lattice_exact"
    yield "kuhn_rmin2.7_downgraded", synth.kuhn_tets(14, 11, 9), 2.7, "lattice_tested"  # classes beyond smem
    # tables large enough that the cycle table + class masks fit shared memory only without the weight
    # replica of the bulk stores (found by tools/lattice_soak.py: the launch asked for > 227 KB)
    yield "kuhn_13x3x2_rmin2.6_large_tables", synth.kuhn_tets(13, 3, 2), 2.6, "lattice_exact"
    yield "kuhn_13x2x2_rmin2.6_large_tables", synth.kuhn_tets(13, 2, 2), 2.6, "lattice_exact"
    yield "hex_aniso", synth.hex_grid(30, 24, 18) * np.array([1.0, 0.75, 1.25]), 1.6, "lattice_exact"
    yield "kuhn_shift_dyadic", synth.kuhn_tets(12, 10, 8) - 37.5, 1.5, "lattice_exact"
    yield "kuhn_shift_thirds", synth.kuhn_tets(12, 10, 8) + (1.0e3 + 1.0 / 3.0), 1.5, "lattice_tested"
    yield "quads_one_row", synth.quad_grid(500, 1), 2.5, "lattice_exact"
    yield "hex_ny1", synth.hex_grid(20, 1, 15), 1.8, "lattice_exact"
    yield "hex_nz1", synth.hex_grid(20, 15, 1), 1.8, "lattice_exact"
    yield "quads_reach4", synth.quad_grid(50, 40), 4.5, "lattice_exact"
    yield "hex_reach3", synth.hex_grid(20, 20, 20), 3.1, "lattice_exact"
    yield "hex_diag_only", synth.hex_grid(20, 20, 20), 0.5, "lattice_exact"
    yield "t3_random_offsets", _t3_lattice(40, 30, 4401), 1.7, "lattice_tested"
    yield "duplicate_types", np.repeat(synth.quad_grid(30, 20), 2, axis=0), 1.5, "lattice_exact"
    yield "tail_displaced_1pct", _displace_tail(synth.kuhn_tets(16, 12, 10), 0.5, 0.01, 4402), 1.5, "lattice_tested"
    yield "tail_displaced_tri", _displace_tail(synth.tri_grid(120, 80, "right"), 0.7, 0.04, 4403), 2.5, \
        "lattice_tested"


@pytest.mark.parametrize("name,c,rmin,path", list(_lattice_cases()))
def test_lattice_path_matches_oracle(tf, name, c, rmin, path):
    c = np.ascontiguousarray(c, dtype=np.float64)
    ref = oracle.build_bruteforce(c, rmin) if c.shape[0] <= 30000 else oracle.build_celllist(c, rmin)
    f = tf.tf_build_filter(dev(c), rmin)  # auto: must detect the lattice
    assert f.stats()["path"] == path, name
    compare_full(f, ref, name)
    x, dc = inputs_for(c.shape[0], 4500)
    compare_applies(f, ref, x, dc, name)
    g = tf.tf_build_filter(dev(c), rmin, path="lattice")
    assert g.stats()["path"] == path
    compare_full(g, ref, name + " (forced)")


def _not_lattice_cases():
    rng = np.random.default_rng(4404)  # permutation only (the points are the generator's)
    yield "hex_permuted", synth.hex_grid(20, 16, 12)[rng.permutation(20 * 16 * 12)], 1.6
    yield "tri_alternating", synth.tri_grid(60, 40, "right/left"), 2.0
    yield "tail_displaced_30pct", _displace_tail(synth.quad_grid(80, 60), 0.5, 0.3, 4405), 1.5
    yield "hex_nx1", synth.hex_grid(1, 30, 30), 1.5
    yield "random_cloud", synth.random_points(4406, 5000, 3, 0, 10), 1.2
    yield "lattice_plus_one", np.concatenate([synth.hex_grid(10, 10, 10), [[3.3, 3.3, 3.3]]]), 1.5


@pytest.mark.parametrize("name,c,rmin", list(_not_lattice_cases()))
def test_non_lattices_take_the_cell_list(tf, name, c, rmin):
    c = np.ascontiguousarray(c, dtype=np.float64)
    ref = oracle.build_bruteforce(c, rmin)
    f = tf.tf_build_filter(dev(c), rmin)
    assert f.stats()["path"] == "cell_list", name
    compare_full(f, ref, name)
    with pytest.raises(tf.TopofiltError, match="TF_ERR_INVALID"):
        tf.tf_build_filter(dev(c), rmin, path="lattice")


def test_lattice_nonfinite_rejected(tf):
    c = synth.hex_grid(12, 10, 8)
    c[-1, 2] = np.nan
    for path in ("auto", "lattice", "cell_list"):
        with pytest.raises(tf.TopofiltError, match="TF_ERR_INVALID"):
            tf.tf_build_filter(dev(c), 1.5, path=path)


def test_unknown_flags_rejected(tf):
    import ctypes
    c = dev(synth.hex_grid(4, 4, 4))
    h = ctypes.c_void_p()
    st = tf.lib().tf_build_filter_ex(ctypes.c_void_p(c.data_ptr()), 64, 3, 1.5, 7, None, ctypes.byref(h))
    assert st == tf.TF_ERR_INVALID


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_paths_agree_configs(tf, cfg):
    """Lattice path vs cell-list path on the same device input: identical CSR bytes."""
    c, x, dc, rmin = synth.workload(cfg)
    a = tf.tf_build_filter(dev(c), rmin, path="lattice")
    b = tf.tf_build_filter(dev(c), rmin, path="cell_list")
    assert b.stats()["path"] == "cell_list"
    ra, ca, va, ha = a.csr()
    rb, cb, vb, hb = b.csr()
    assert torch.equal(ra, rb) and torch.equal(ca, cb) and torch.equal(va, vb)
    assert_rel(ha.cpu().numpy(), hb.cpu().numpy(), 1e-12, f"c{cfg} Hs")
    assert_rel(a.sensitivity(dev(x), dev(dc)).cpu().numpy(), b.sensitivity(dev(x), dev(dc)).cpu().numpy(),
               RTOL_OUT, "sensitivity")


def test_config5_paths_agree_bitwise(tf):
    """Config 5 (12M Kuhn tets, nnz 1,030,251,952): the exact-lattice CSR equals the cell-list CSR
    byte for byte (whole arrays, compared on the device); Hs within 1e-12."""
    c, x, dc, rmin = synth.workload(5)
    cd = dev(c)
    a = tf.tf_build_filter(cd, rmin)
    assert a.stats()["path"] == "lattice_exact" and a.nnz == 1_030_251_952
    b = tf.tf_build_filter(cd, rmin, path="cell_list")
    ra, ca, va, ha = a.csr()
    rb, cb, vb, hb = b.csr()
    assert torch.equal(ra, rb)
    step = 1 << 27
    for s0 in range(0, a.nnz, step):
        assert torch.equal(ca[s0:s0 + step], cb[s0:s0 + step]), s0
        assert torch.equal(va[s0:s0 + step], vb[s0:s0 + step]), s0
    rel = ((ha - hb).abs() / hb.abs()).max().item()
    assert rel <= 1e-12, rel
    b.close()
    a.close()
