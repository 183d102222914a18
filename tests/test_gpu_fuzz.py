"""Seeded randomized parity: varied point-cloud shapes and densities (uniform, clustered blobs
whose dense neighbourhoods take the large-neighbourhood path, thin anisotropic slabs, integer
lattices full of exact ties, heavy duplication, mixed scales), each compared with the oracle:
the whole CSR bit-exact and both filters within 1e-10."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tf():
    assert torch.cuda.is_available()
    import paper_2012_08208_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def cloud(seed: int):
    """A seeded case: (points, rmin) drawn from one of six shapes."""
    u = lambda k, n, a=0.0, b=1.0: synth.uniform(10_000 + 97 * seed + k, 0, n, a, b)  # noqa: E731
    kind = seed % 6
    dim = 2 + (seed // 6) % 2
    n = int(200 + u(0, 1)[0] * 20_000)
    if kind == 0:  # uniform box
        c = u(1, n * dim, 0.0, 30.0).reshape(n, dim)
        rmin = 0.5 + 2.0 * u(2, 1)[0]
    elif kind == 1:  # clustered blobs: dense cores -> large neighbourhoods
        centres = u(1, 5 * dim, 0.0, 40.0).reshape(5, dim)
        which = np.floor(u(2, n) * 5).astype(int)
        c = centres[which] + (u(3, n * dim) - 0.5).reshape(n, dim) * (0.2 + 3.0 * u(4, n)[:, None])
        rmin = 0.8 + u(5, 1)[0]
    elif kind == 2:  # thin anisotropic slab
        ext = np.array([1000.0, 5.0, 0.05][:dim])
        c = u(1, n * dim).reshape(n, dim) * ext
        rmin = 1.0 + 2.0 * u(2, 1)[0]
    elif kind == 3:  # integer lattice subset: exact ties at integer rmin
        m = int(np.ceil(n ** (1.0 / dim))) + 2
        g = np.stack(np.meshgrid(*[np.arange(m)] * dim, indexing="ij"), -1).reshape(-1, dim).astype(np.float64)
        keep = u(1, g.shape[0]) < 0.7
        c = g[keep][:n]
        rmin = float(1 + int(u(2, 1)[0] * 3))  # 1, 2 or 3: ties at d = rmin
    elif kind == 4:  # heavy duplication
        base = u(1, (n // 8 + 1) * dim, 0.0, 20.0).reshape(-1, dim)
        c = base[np.floor(u(2, n) * base.shape[0]).astype(int)]
        rmin = 0.7 + u(3, 1)[0]
    else:  # mixed scales: a fine cluster inside a coarse cloud, offset far from the origin
        coarse = u(1, (n // 2) * dim, 0.0, 100.0).reshape(-1, dim)
        fine = 50.0 + u(2, (n - n // 2) * dim, 0.0, 2.0).reshape(-1, dim)
        c = np.concatenate([coarse, fine]) + 1.0e5
        rmin = 0.3 + u(3, 1)[0]
    return np.ascontiguousarray(c, dtype=np.float64), float(rmin)


@pytest.mark.parametrize("seed", range(24))
def test_random_clouds(tf, seed):
    c, rmin = cloud(seed)
    n = c.shape[0]
    ref = oracle.build_celllist(c, rmin)
    f = tf.tf_build_filter(dev(c), rmin)
    rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
    np.testing.assert_array_equal(rowptr, ref.rowptr)
    np.testing.assert_array_equal(cols, ref.cols)
    np.testing.assert_array_equal(vals, ref.vals)
    np.testing.assert_allclose(hs, ref.hs, rtol=1e-12)
    x = synth.uniform(20_000 + seed, 0, n, 0.001, 1.0)
    dc = -synth.uniform(30_000 + seed, 0, n, 0.0, 1.0)
    s = f.sensitivity(dev(x), dev(dc)).cpu().numpy()
    d = f.density(dev(x)).cpu().numpy()
    for got, want, what in ((s, oracle.apply_sensitivity(ref, x, dc), "sens"), (d, oracle.apply_density(ref, x), "dens")):
        scale = np.where(want != 0, np.abs(want), np.abs(want).max())
        assert np.all(np.abs(got - want) <= 1e-10 * scale), f"seed {seed} {what}"
    f.close()


@pytest.mark.parametrize("kind", ["block", "warp"])
@pytest.mark.parametrize("seed", range(24))
def test_fill_kernels(tf, seed, kind, monkeypatch):
    """Both a7 fill kernels, forced (TOPOFILT_FILL): the block-per-bin fill (staging + id sort) and
    the warp-per-query fill (exact tests + id ranks; serves rows up to 128 entries, KS = 1..4, and
    falls back to the block fill above that). Whole CSR bit-exact vs the oracle, Hs 1e-12."""
    monkeypatch.setenv("TOPOFILT_FILL", kind)
    c, rmin = cloud(seed)
    ref = oracle.build_celllist(c, rmin)
    f = tf.tf_build_filter(dev(c), rmin, path="cell_list")
    rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
    np.testing.assert_array_equal(rowptr, ref.rowptr)
    np.testing.assert_array_equal(cols, ref.cols)
    np.testing.assert_array_equal(vals, ref.vals)
    np.testing.assert_allclose(hs, ref.hs, rtol=1e-12)
    f.close()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_fill_kernels_agree_configs(tf, cfg, monkeypatch):
    """Configs 1-4 on the cell-list path: the warp fill's CSR equals the block fill's byte for byte,
    Hs within 1e-12 (different summation order)."""
    c, _, _, rmin = synth.workload(cfg)
    cd = dev(c)
    out = {}
    for kind in ("block", "warp"):
        monkeypatch.setenv("TOPOFILT_FILL", kind)
        f = tf.tf_build_filter(cd, rmin, path="cell_list")
        out[kind] = [t.clone() for t in f.csr()]
        f.close()
    (ra, ca, va, ha), (rb, cb, vb, hb) = out["block"], out["warp"]
    assert torch.equal(ra, rb) and torch.equal(ca, cb) and torch.equal(va, vb)
    assert ((ha - hb).abs() / hb.abs()).max().item() <= 1e-12


@pytest.mark.parametrize("rmin", [2.6, 2.8])
def test_fill_warp_long_rows(tf, rmin, monkeypatch):
    """Rows of 97-128 entries (longest 104 / 126): the forced warp fill's four-slot ranks (KS = 4)
    against the oracle; ragged row lengths from a uniform random cloud."""
    monkeypatch.setenv("TOPOFILT_FILL", "warp")
    c = np.ascontiguousarray(synth.uniform(777, 0, 3 * 6000, 0.0, 18.0).reshape(-1, 3))
    ref = oracle.build_celllist(c, rmin)
    assert 96 < np.diff(ref.rowptr).max() <= 128
    f = tf.tf_build_filter(dev(c), rmin, path="cell_list")
    rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
    np.testing.assert_array_equal(rowptr, ref.rowptr)
    np.testing.assert_array_equal(cols, ref.cols)
    np.testing.assert_array_equal(vals, ref.vals)
    np.testing.assert_allclose(hs, ref.hs, rtol=1e-12)
    f.close()


@pytest.mark.parametrize("scale", [1.5, 3.0])
@pytest.mark.parametrize("seed", [0, 2, 3, 6, 9, 14, 20])
def test_bin_scale_invariance(tf, seed, scale, monkeypatch):
    """The GPU cell list with bins of scale*rmin (TOPOFILT_BIN_SCALE) gives the same CSR as the
    oracle: the 3^dim rule holds for any bin side >= rmin*(1+1e-6) (SURVEY 8(c) O2 invariance)."""
    monkeypatch.setenv("TOPOFILT_BIN_SCALE", str(scale))
    c, rmin = cloud(seed)
    ref = oracle.build_celllist(c, rmin)
    f = tf.tf_build_filter(dev(c), rmin, path="cell_list")
    rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
    np.testing.assert_array_equal(rowptr, ref.rowptr)
    np.testing.assert_array_equal(cols, ref.cols)
    np.testing.assert_array_equal(vals, ref.vals)
    np.testing.assert_allclose(hs, ref.hs, rtol=1e-12)
    f.close()
