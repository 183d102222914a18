"""The group kernels of the cell-list build (cl_build.cu: k_cl_count / k_cl_fill3 / k_cl_fill4)
against the oracle and against the per-bin kernels (TF_BUILD_CELL_LIST_BINS): the whole CSR
bit-exact, Hs within 1e-12. Cases aimed at the group design's own edges: the fp32 band (pairs at
and within a few ulps of rmin), rows longer than the fill's per-lane lists, unions beyond the group
kernels' capacity (fallback to the per-bin kernels), groups cut at unit and bin-row boundaries,
sparse rows whose groups span many bins, and 2D/3D configs."""
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


def check_against_oracle(tf, c, rmin, expect_groups=True):
    ref = oracle.build_celllist(c, rmin)
    f = tf.tf_build_filter(dev(c), rmin, path="cell_list")
    st = f.stats()
    assert st["path"] == "cell_list"
    if expect_groups:
        assert st["groups"] > 0
    rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
    np.testing.assert_array_equal(rowptr, ref.rowptr)
    np.testing.assert_array_equal(cols, ref.cols)
    np.testing.assert_array_equal(vals, ref.vals)
    np.testing.assert_allclose(hs, ref.hs, rtol=1e-12)
    f.close()
    return st


def check_paths_agree(tf, c, rmin):
    fg = tf.tf_build_filter(dev(c), rmin, path="cell_list")
    fb = tf.tf_build_filter(dev(c), rmin, path="cell_list_bins")
    assert fg.stats()["groups"] > 0 and fb.stats()["groups"] == 0
    for a, b in zip(fg.csr()[:3], fb.csr()[:3]):
        assert torch.equal(a, b)
    hg, hb = fg.csr()[3], fb.csr()[3]
    assert float(((hg - hb).abs() / hb.abs()).max()) <= 1e-12
    fg.close()
    fb.close()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_configs_group_vs_bins(tf, cfg):
    c, _, _, rmin = synth.workload(cfg)
    check_paths_agree(tf, c, rmin)


def test_config4_vs_oracle(tf):
    c, _, _, rmin = synth.workload(4)
    check_against_oracle(tf, c, rmin)


def test_band_pairs_at_rmin(tf):
    """Pairs at exactly rmin and within a few ulps of it on both sides: every decision falls in
    the fp32 band and takes the exact fp64 test."""
    rng = np.random.default_rng(7)
    rmin = 1.25
    base = rng.uniform(0, 40, size=(3000, 3))
    d = rng.normal(size=(3000, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    scale = rmin * (1.0 + rng.integers(-4, 5, size=3000) * 2.0 ** -52)
    partner = base + d * scale[:, None]
    c = np.concatenate([base, partner])
    check_against_oracle(tf, c, rmin)


def test_long_rows_word_path(tf):
    """A dense cluster: rows far longer than the fill's per-lane lists (256 entries)."""
    rng = np.random.default_rng(11)
    c = np.concatenate([rng.uniform(0, 1.0, size=(1500, 3)), rng.uniform(0, 30, size=(2000, 3))])
    st = check_against_oracle(tf, c, 1.2)
    assert st["groups"] > 0


def test_union_beyond_capacity_falls_back(tf):
    """One bin neighbourhood with more points than the group kernels take (6144): the per-bin
    kernels run (groups == 0) and the CSR is still the oracle's."""
    rng = np.random.default_rng(3)
    c = np.concatenate([rng.uniform(0, 0.5, size=(7000, 2)), rng.uniform(0, 50, size=(500, 2))])
    ref = oracle.build_celllist(c, 0.6)
    f = tf.tf_build_filter(dev(c), 0.6, path="cell_list")
    assert f.stats()["groups"] == 0
    rowptr, cols, vals, _ = (t.cpu().numpy() for t in f.csr())
    np.testing.assert_array_equal(rowptr, ref.rowptr)
    np.testing.assert_array_equal(cols, ref.cols)
    np.testing.assert_array_equal(vals, ref.vals)
    f.close()


@pytest.mark.parametrize("npts,groups_run", [(4000, True), (4400, False)])
def test_union_run_code_limit(tf, npts, groups_run):
    """The sorted union travels from the count to the fill as 16-bit codes (run << 12 | offset), so a
    union run may hold at most 4,095 points. One bin with 4,000 points (unions of ~4,050 <= 6,144,
    runs < 4,096): the group kernels run, offsets up to ~4,000 are exercised and every row takes the
    long-row path; with 4,400 points the run no longer fits the code and the per-bin kernels take
    the build. Either way the CSR is the oracle's."""
    rng = np.random.default_rng(17)
    c = np.concatenate([rng.uniform(0.05, 0.45, size=(npts, 2)), rng.uniform(2.0, 60.0, size=(50, 2))])
    ref = oracle.build_celllist(c, 0.6)
    f = tf.tf_build_filter(dev(c), 0.6, path="cell_list")
    assert (f.stats()["groups"] > 0) == groups_run
    rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
    np.testing.assert_array_equal(rowptr, ref.rowptr)
    np.testing.assert_array_equal(cols, ref.cols)
    np.testing.assert_array_equal(vals, ref.vals)
    np.testing.assert_allclose(hs, ref.hs, rtol=1e-12)
    f.close()


def test_sparse_rows_wide_groups(tf):
    """Long sparse x-rows: a group's 32 points span many bins (wide union box, wide fp32 band),
    groups are cut at 32-bin unit boundaries and at bin-row ends."""
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 4000, size=6000)
    y = rng.integers(0, 3, size=6000) * 1.7 + rng.uniform(0, 0.2, size=6000)
    c = np.stack([x, y], 1)
    check_against_oracle(tf, c, 2.0)


def test_random_ids_3d(tf):
    """Ids in random order (no spatial coherence): the union sort does all the work."""
    rng = np.random.default_rng(9)
    c = rng.uniform(0, 25, size=(20000, 3))
    check_against_oracle(tf, c, 1.6)


def test_paper_right_left_triangles(tf):
    """The paper's RectangleMesh "right/left" triangles through the cell list."""
    nx, ny = 90, 30
    pts = []
    for j in range(ny):
        for i in range(nx):
            v = [(i, j), (i + 1, j), (i + 1, j + 1), (i, j + 1)]
            if (i + j) % 2 == 0:
                tris = [(v[0], v[1], v[2]), (v[0], v[2], v[3])]
            else:
                tris = [(v[0], v[1], v[3]), (v[1], v[2], v[3])]
            for a, b, d in tris:
                pts.append((((a[0] + b[0]) + d[0]) / 3.0, ((a[1] + b[1]) + d[1]) / 3.0))
    c = np.array(pts)
    check_against_oracle(tf, c, 2.0)
    check_paths_agree(tf, c, 2.0)


@pytest.mark.parametrize("kernel", ["walk3", "split"])
def test_fill_kernel_variants(tf, monkeypatch, kernel):
    """Both fill kernels of the group path build the oracle's CSR whichever one the size rule would pick:
    k_cl_fill3 (walk3: warp per group, the default for 3D-sized unions) and k_cl_fill4 (split: block per
    group with the union staged in shared memory, the default for small unions) -- on a 2D ground
    structure, a jittered Kuhn mesh and a dense cluster whose rows exceed the per-lane lists
    (word-parallel long-row path)."""
    monkeypatch.setenv("TOPOFILT_CL_FILL", kernel)
    for c, rmin in ((synth.ground_structure(4, 400, 300)[0], 3.0), (synth.kuhn_mesh(10, 8, 6, jitter=0.1, stream=5)[0], 1.5),
                    (np.concatenate([np.random.default_rng(2).uniform(0, 1.0, size=(900, 3)),
                                     np.random.default_rng(3).uniform(0, 20, size=(3000, 3))]), 1.1)):
        check_against_oracle(tf, c, rmin)
