"""GPU parity: libtopofilt (through the C ABI) against the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star):
  * rowptr and cols bit-exact; vals bit-exact (same fp64 expression, no FMA) -- the
    contract's 1e-12 relative is checked too; Hs within 1e-12 relative;
  * filtered outputs within 1e-10 relative (elementwise |g - r| <= 1e-10 |r|).
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL_HS = 1e-12
RTOL_OUT = 1e-10


@pytest.fixture(scope="module")
def tf():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2012_08208_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def assert_rel(g, r, rtol, what):
    g = np.asarray(g)
    r = np.asarray(r)
    assert g.shape == r.shape, what
    scale = np.where(r != 0, np.abs(r), np.abs(r).max() if r.size else 1.0)
    bad = np.abs(g - r) > rtol * scale
    assert not bad.any(), f"{what}: {bad.sum()} of {r.size} outside rtol {rtol}; first at {np.argmax(bad)}: " \
                          f"gpu {g[bad][0]!r} oracle {r[bad][0]!r}"


def csr_host(f):
    return tuple(t.cpu().numpy() for t in f.csr())


def compare_full(f, ref, tag=""):
    rowptr, cols, vals, hs = csr_host(f)
    np.testing.assert_array_equal(rowptr, ref.rowptr, err_msg=f"{tag} rowptr")
    np.testing.assert_array_equal(cols, ref.cols, err_msg=f"{tag} cols")
    assert_rel(vals, ref.vals, RTOL_HS, f"{tag} vals")
    np.testing.assert_array_equal(vals, ref.vals, err_msg=f"{tag} vals bitwise")
    assert_rel(hs, ref.hs, RTOL_HS, f"{tag} Hs")


def compare_applies(f, ref, x, dc, tag=""):
    s = f.sensitivity(dev(x), dev(dc)).cpu().numpy()
    d = f.density(dev(x)).cpu().numpy()
    assert_rel(s, oracle.apply_sensitivity(ref, x, dc), RTOL_OUT, f"{tag} sensitivity")
    assert_rel(d, oracle.apply_density(ref, x), RTOL_OUT, f"{tag} density")


def inputs_for(n, seed):
    x = synth.uniform(seed, 0, n, 0.001, 1.0)
    dc = (-3.0 * (x * x)) * synth.uniform(seed + 1, 0, n, 0.5, 1.5)
    return x, dc


# ------------------------------------------------------------------ apply kernels on oracle CSRs

@pytest.mark.parametrize("cfg", [1, 2])
def test_apply_on_oracle_csr(tf, cfg):
    """a8/a9 alone: the apply kernels on the oracle's CSR, imported via tf_filter_from_csr."""
    c, x, dc, rmin = synth.workload(cfg)
    ref = oracle.build_celllist(c, rmin)
    f = tf.tf_filter_from_csr(ref.rowptr, ref.cols, ref.vals, ref.hs)
    compare_applies(f, ref, x, dc, f"c{cfg}")


def test_apply_long_rows_and_ragged(tf):
    """Rows longer than the shared-memory staging (block-per-row path), ragged lengths,
    a window boundary inside a long row, and empty-ish short rows."""
    rng = np.random.default_rng(5)
    n = 9000
    lens = rng.integers(1, 40, size=n)
    lens[100] = 20000
    lens[4000:4003] = [5000, 6000, 9000]
    rowptr = np.zeros(n + 1, np.int64)
    rowptr[1:] = np.cumsum(lens)
    nnz = rowptr[-1]
    cols = np.concatenate([np.sort(rng.choice(n, size=l, replace=l > n)) for l in lens]).astype(np.int32)
    vals = rng.uniform(0, 2, size=nnz)
    hs = np.add.reduceat(vals, rowptr[:-1])
    ref = oracle.CSR(rowptr, cols, vals, hs)
    f = tf.tf_filter_from_csr(rowptr, cols, vals, hs)
    x, dc = inputs_for(n, 501)
    compare_applies(f, ref, x, dc, "ragged")


@pytest.mark.parametrize("lo,hi,longest", [(20, 120, None), (16, 90, 1000), (60, 100, 2900), (1, 15, 300)])
def test_apply_window_sizing(tf, lo, hi, longest):
    """The apply plan sizes its windows from the longest row (stage capacity minus it when rows
    average >= 16; the fixed window otherwise): enlarged windows, a longest row that keeps the
    fixed window, a row that barely fits a stage, and short rows -- all against the oracle."""
    rng = np.random.default_rng(lo * 1000 + hi)
    n = 20000
    lens = rng.integers(lo, hi + 1, size=n)
    if longest is not None:
        lens[n // 3] = longest
    rowptr = np.zeros(n + 1, np.int64)
    rowptr[1:] = np.cumsum(lens)
    nnz = rowptr[-1]
    cols = np.concatenate([np.sort(rng.choice(n, size=l, replace=False)) for l in lens]).astype(np.int32)
    vals = rng.uniform(0, 2, size=nnz)
    hs = np.add.reduceat(vals, rowptr[:-1])
    ref = oracle.CSR(rowptr, cols, vals, hs)
    f = tf.tf_filter_from_csr(rowptr, cols, vals, hs)
    x, dc = inputs_for(n, 502)
    compare_applies(f, ref, x, dc, f"windows {lo}-{hi}/{longest}")


# ------------------------------------------------------------------ full build parity

@pytest.mark.parametrize("path", ["auto", "cell_list"])
@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_build_and_apply_configs_full(tf, cfg, path):
    """Configs 1-4 in full: the whole CSR and Hs against the oracle's cell list (which is
    pinned to the brute force and the closed forms), then both filters. "auto" takes the
    lattice path on configs 1-3 (exact, tested, exact) and the cell list on config 4."""
    c, x, dc, rmin = synth.workload(cfg)
    ref = oracle.build_celllist(c, rmin)
    f = tf.tf_build_filter(dev(c), rmin, path=path)
    expect = {"cell_list": "cell_list"}.get(path, {1: "lattice_exact", 2: "lattice_tested", 3: "lattice_exact",
                                                    4: "cell_list"}[cfg])
    assert f.stats()["path"] == expect
    assert f.nnz == ref.nnz
    compare_full(f, ref, f"c{cfg}")
    compare_applies(f, ref, x, dc, f"c{cfg}")
    if cfg == 2:  # 50 iterations with fresh dc: spot-check a later one
        dc7 = synth.sensitivity(2, x, 7)
        assert_rel(f.sensitivity(dev(x), dev(dc7)).cpu().numpy(), oracle.apply_sensitivity(ref, x, dc7),
                   RTOL_OUT, "c2 t=7")


def _sampled(f, rows_np):
    rowptr, cols, vals, hs = f.csr()
    rows = torch.from_numpy(rows_np).cuda()
    starts = rowptr[rows]
    lens = rowptr[rows + 1] - starts
    total = int(lens.sum())
    seg0 = torch.repeat_interleave(torch.cumsum(lens, 0) - lens, lens)
    idx = torch.repeat_interleave(starts, lens) + (torch.arange(total, device="cuda") - seg0)
    rp = np.zeros(len(rows_np) + 1, np.int64)
    rp[1:] = np.cumsum(lens.cpu().numpy())
    return rp, cols[idx].cpu().numpy(), vals[idx].cpu().numpy(), hs[rows].cpu().numpy()


@pytest.mark.parametrize("path", ["auto", "cell_list"])
def test_config5_sampled_rows(tf, path):
    """Config 5 (12M Kuhn tets): nnz equals the exact lattice count; 10,000 seeded rows
    (stream S(5,5,0)) match the oracle bit-exactly; both filters at those rows; global
    structural properties of the whole GPU CSR checked on the device. Both build paths
    (auto = the exact lattice path)."""
    c, x, dc, rmin = synth.workload(5)
    n = c.shape[0]
    f = tf.tf_build_filter(dev(c), rmin, path=path)
    assert f.stats()["path"] == ("lattice_exact" if path == "auto" else "cell_list")
    assert f.nnz == 1_030_251_952
    rows = np.sort(synth.sample_rows(5, n, 10_000))
    cl = oracle.CellList(c, rmin)
    ref = cl.rows(rows)
    rp, cols, vals, hs = _sampled(f, rows)
    np.testing.assert_array_equal(rp, ref.rowptr)
    np.testing.assert_array_equal(cols, ref.cols)
    np.testing.assert_array_equal(vals, ref.vals)
    assert_rel(hs, ref.hs, RTOL_HS, "c5 Hs")
    s = f.sensitivity(dev(x), dev(dc))
    d = f.density(dev(x))
    rt = torch.from_numpy(rows).cuda()
    assert_rel(s[rt].cpu().numpy(), oracle.apply_sensitivity(ref, x, dc), RTOL_OUT, "c5 sensitivity")
    assert_rel(d[rt].cpu().numpy(), oracle.apply_density(ref, x), RTOL_OUT, "c5 density")
    # whole-CSR properties on the device: ascending columns, diagonal = rmin, row lengths <= 87
    rowptr, colsd, valsd, hsd = f.csr()
    lens = rowptr[1:] - rowptr[:-1]
    assert int(lens.max()) == 87 and int(lens.min()) >= 1
    rid = torch.repeat_interleave(torch.arange(n, device="cuda"), lens)
    first = torch.zeros(f.nnz, dtype=torch.bool, device="cuda")
    first[rowptr[:-1]] = True
    asc = (colsd[1:] > colsd[:-1]) | first[1:]
    assert bool(asc.all())
    diag = colsd.long() == rid
    assert int(diag.sum()) == n and bool((valsd[diag] == rmin).all())
    assert bool((hsd >= rmin).all())
    del rid, first, asc, diag


@pytest.mark.parametrize("path", ["auto", "cell_list"])
def test_nnz_beyond_int32(tf, path):
    """Maximum-size case: 28.8M Kuhn tets (300x160x100 cubes) give nnz = 2,479,728,752 > 2^31
    (exact lattice count), so every element offset past 2^31 goes through the int64 paths of
    the fill, the apply plan and the TMA window addresses. Checked: nnz against the closed
    form; 3,000 seeded rows plus the rows straddling element 2^31 and the last rows bit-exact
    against the oracle; both filters at those rows; ascending columns over the whole CSR."""
    c = synth.kuhn_tets(300, 160, 100)
    n, rmin = c.shape[0], 1.5
    f = tf.tf_build_filter(dev(c), rmin, path=path)
    assert f.nnz == 2_479_728_752 > 2**31
    rowptr, colsd, _, _ = f.csr()
    r31 = int(torch.searchsorted(rowptr, torch.tensor([2**31], device="cuda"), right=True).item()) - 1
    assert rowptr[r31] <= 2**31 < rowptr[r31 + 1]
    extra = np.concatenate([np.arange(r31 - 2, r31 + 3), np.arange(n - 50, n)])
    rows = np.unique(np.concatenate([synth.sample_rows(6, n, 3000), extra]))
    cl = oracle.CellList(c, rmin)
    ref = cl.rows(rows)
    cl.close()
    rp, cols, vals, hs = _sampled(f, rows)
    np.testing.assert_array_equal(rp, ref.rowptr)
    np.testing.assert_array_equal(cols, ref.cols)
    np.testing.assert_array_equal(vals, ref.vals)
    assert_rel(hs, ref.hs, RTOL_HS, "Hs")
    x, dc = inputs_for(n, 611)
    rt = torch.from_numpy(rows).cuda()
    s = f.sensitivity(dev(x), dev(dc))[rt].cpu().numpy()
    d = f.density(dev(x))[rt].cpu().numpy()
    assert_rel(s, oracle.apply_sensitivity(ref, x, dc), RTOL_OUT, "sensitivity")
    assert_rel(d, oracle.apply_density(ref, x), RTOL_OUT, "density")
    first = torch.zeros(f.nnz, dtype=torch.bool, device="cuda")
    first[rowptr[:-1]] = True
    assert bool(((colsd[1:] > colsd[:-1]) | first[1:]).all())
    del first, rowptr, colsd
    f.close()


# ------------------------------------------------------------------ fp-decided and paper workloads

@pytest.mark.parametrize("name,c,rmin", [
    ("spec_8x4_right_rmin2", synth.tri_grid(8, 4, "right"), 2.0),
    ("spec_kuhn_6x4x2", synth.kuhn_tets(6, 4, 2), 1.5),
    ("e01_180x60_rmin2", synth.tri_grid(180, 60, "right"), 2.0),
    ("e01_alt_180x60_rmin2", synth.tri_grid(180, 60, "right/left"), 2.0),
    ("e03_180x60_rmin3", synth.tri_grid(180, 60, "right"), 3.0),
    ("e02_kuhn_60x20x4", synth.kuhn_tets(60, 20, 4), 1.5),
])
def test_paper_and_tie_workloads(tf, name, c, rmin):
    """Thirds lattices at integer rmin: fp64 rounding decides ties (SURVEY.md 8(c) point 5);
    only the identical no-FMA expression reproduces the oracle's structure."""
    ref = oracle.build_bruteforce(c, rmin) if c.shape[0] <= 30000 else oracle.build_celllist(c, rmin)
    f = tf.tf_build_filter(dev(c), rmin)
    compare_full(f, ref, name)
    x, dc = inputs_for(c.shape[0], 700)
    compare_applies(f, ref, x, dc, name)


# ------------------------------------------------------------------ edge cases

def _edge_cases():
    yield "n1_2d", np.array([[0.5, 0.5]]), 1.0
    yield "n1_3d", np.array([[0.5, 0.5, -3.0]]), 1.0
    yield "n2_far", np.array([[0.0, 0.0], [3.0, 0.0]]), 2.0
    yield "n31", synth.random_points(801, 31, 3, 0, 4), 1.5
    yield "n33", synth.random_points(802, 33, 2, 0, 4), 1.5
    yield "n1000", synth.random_points(803, 1000, 3, -2, 2), 0.7
    yield "duplicates", np.repeat(synth.random_points(804, 200, 3, 0, 5), 4, axis=0), 1.0
    yield "collinear_3d", np.stack([np.arange(500) * 0.37, np.zeros(500), np.zeros(500)], 1), 1.0
    yield "huge_offset", synth.random_points(805, 3000, 2, 0, 30) + 1.0e6, 1.1
    yield "negative", synth.random_points(806, 3000, 3, -40, -10), 2.0
    yield "sparse_wide", synth.random_points(807, 500, 2, 0, 1.0e6), 1.0  # bin cap enlarges s
    yield "one_bin_dense_2d", synth.random_points(808, 2000, 2, 0, 1), 5.0
    yield "one_bin_large_2d", synth.random_points(809, 7000, 2, 0, 1), 5.0   # > smem cap: row sort (smem)
    yield "one_bin_large_3d", synth.random_points(810, 4500, 3, 0, 1), 5.0   # > 3D cap
    yield "mixed_large_and_small", np.concatenate([synth.random_points(811, 6000, 2, 0, 0.5),
                                                   synth.random_points(812, 3000, 2, 2, 60)]), 1.0
    yield "row_longer_than_sort_smem", synth.random_points(813, 9000, 2, 0, 1), 5.0  # global bitonic


@pytest.mark.parametrize("name,c,rmin", list(_edge_cases()))
def test_edge_cases(tf, name, c, rmin):
    c = np.ascontiguousarray(c, dtype=np.float64)
    ref = oracle.build_bruteforce(c, rmin)
    f = tf.tf_build_filter(dev(c), rmin)
    compare_full(f, ref, name)
    x, dc = inputs_for(c.shape[0], 900)
    compare_applies(f, ref, x, dc, name)


# ------------------------------------------------------------------ properties, errors, API

def test_determinism(tf):
    c, x, dc, rmin = synth.workload(2)
    f1 = tf.tf_build_filter(dev(c), rmin)
    f2 = tf.tf_build_filter(dev(c), rmin)
    for a, b in zip(csr_host(f1), csr_host(f2)):
        np.testing.assert_array_equal(a, b)
    xs, dcs = dev(x), dev(dc)
    np.testing.assert_array_equal(f1.sensitivity(xs, dcs).cpu().numpy(), f1.sensitivity(xs, dcs).cpu().numpy())
    np.testing.assert_array_equal(f1.density(xs).cpu().numpy(), f2.density(xs).cpu().numpy())


def test_config1_exact_identity_gpu(tf):
    """x = 0.5: sensitivity(x, dc) == density(dc) bitwise (same summation order on the GPU)."""
    c, x, dc, rmin = synth.workload(1)
    f = tf.tf_build_filter(dev(c), rmin)
    np.testing.assert_array_equal(f.sensitivity(dev(x), dev(dc)).cpu().numpy(), f.density(dev(dc)).cpu().numpy())


def test_host_variants_match_device(tf):
    c, x, dc, rmin = synth.workload(2)
    fh = tf.tf_build_filter_host(c, rmin)
    fd = tf.tf_build_filter(dev(c), rmin)
    for a, b in zip(csr_host(fh), csr_host(fd)):
        np.testing.assert_array_equal(a, b)
    xp = torch.from_numpy(x).pin_memory().numpy()
    np.testing.assert_array_equal(fh.sensitivity_host(xp, dc), fd.sensitivity(dev(x), dev(dc)).cpu().numpy())
    np.testing.assert_array_equal(fh.density_host(x), fd.density(dev(x)).cpu().numpy())
    s2, d2 = tf.tf_filter_iteration_host(fh, x, dc)
    np.testing.assert_array_equal(s2, fd.sensitivity(dev(x), dev(dc)).cpu().numpy())
    np.testing.assert_array_equal(d2, fd.density(dev(x)).cpu().numpy())


@pytest.mark.parametrize("case", ["one_window", "c1", "c3", "stencil_c3", "random_ids"])
def test_iteration_host_pipeline(tf, case):
    """tf_filter_iteration_host: the row-range chunk pipeline (plans with >= 2 windows: up to 8
    chunks; chunk i starts once the input pieces up to its largest column have landed, and
    downloads while the next computes) and the whole-array path (one window, stencil handles)
    give the device calls' results bitwise; repeated calls stay correct. random_ids: ids carry no
    spatial order, so every chunk reads columns up to ~N and waits for every piece."""
    if case == "random_ids":
        c, rmin = synth.random_points(613, 200_000, 3, 0.0, 40.0), 1.2
        n = c.shape[0]
        x, dc = inputs_for(n, 614)
        f = tf.tf_build_filter(dev(c), rmin)
    elif case == "one_window":
        c, rmin = synth.random_points(611, 40, 2, 0.0, 3.0), 1.0
        n = c.shape[0]
        x, dc = inputs_for(n, 612)
        f = tf.tf_build_filter(dev(c), rmin)
    elif case == "stencil_c3":
        c, x, dc, rmin = synth.workload(3)
        f = tf.tf_build_stencil(3, 160, 80, 80, 1.0, rmin)
    else:
        c, x, dc, rmin = synth.workload(int(case[1]))
        f = tf.tf_build_filter(dev(c), rmin)
    want_s = f.sensitivity(dev(x), dev(dc)).cpu().numpy()
    want_d = f.density(dev(x)).cpu().numpy()
    for _ in range(2):
        s2, d2 = tf.tf_filter_iteration_host(f, x, dc)
        np.testing.assert_array_equal(s2, want_s)
        np.testing.assert_array_equal(d2, want_d)


@pytest.mark.parametrize("case", ["c1", "c2", "c4", "ragged_long_rows", "stencil_c3"])
def test_filter_both_bitwise(tf, case):
    """tf_filter_both (one pass over H, two gathers per entry) equals the separate sensitivity and
    density calls bitwise, incl. the unstaged long-row path; and the oracle at 1e-10."""
    if case == "ragged_long_rows":
        rng = np.random.default_rng(9)
        n = 6000
        lens = rng.integers(1, 40, size=n)
        lens[[10, 3000]] = [12000, 7000]
        rowptr = np.zeros(n + 1, np.int64)
        rowptr[1:] = np.cumsum(lens)
        cols = np.concatenate([np.sort(rng.choice(n, size=l, replace=l > n)) for l in lens]).astype(np.int32)
        vals = rng.uniform(0, 2, size=rowptr[-1])
        hs = np.add.reduceat(vals, rowptr[:-1])
        ref = oracle.CSR(rowptr, cols, vals, hs)
        f = tf.tf_filter_from_csr(rowptr, cols, vals, hs)
        x, dc = inputs_for(n, 615)
    elif case == "stencil_c3":
        c, x, dc, rmin = synth.workload(3)
        f = tf.tf_build_stencil(3, 160, 80, 80, 1.0, rmin)
        ref = None
    else:
        c, x, dc, rmin = synth.workload(int(case[1]))
        f = tf.tf_build_filter(dev(c), rmin)
        ref = oracle.build_celllist(c, rmin)
    xd, dcd = dev(x), dev(dc)
    s, d = f.both(xd, dcd)
    assert torch.equal(s, f.sensitivity(xd, dcd))
    assert torch.equal(d, f.density(xd))
    if ref is not None:
        assert_rel(s.cpu().numpy(), oracle.apply_sensitivity(ref, x, dc), RTOL_OUT, "both: sensitivity")
        assert_rel(d.cpu().numpy(), oracle.apply_density(ref, x), RTOL_OUT, "both: density")
    with pytest.raises(tf.TopofiltError):
        f.both(xd, dcd, sens_out=dcd)
    o = torch.empty_like(xd)
    with pytest.raises(tf.TopofiltError):
        f.both(xd, dcd, sens_out=o, dens_out=o)


@pytest.mark.parametrize("case", ["c4", "ragged_long_rows", "stencil_c3"])
def test_filter_rows_prefix(tf, case):
    """tf_*_filter_rows: rows [0, nrows) bitwise equal to the full call for nrows at 0, 1, a window
    boundary neighbourhood, mid and n (incl. the unstaged long-row windows); out-of-range nrows
    is TF_ERR_INVALID."""
    if case == "ragged_long_rows":
        rng = np.random.default_rng(19)
        n = 6000
        lens = rng.integers(1, 40, size=n)
        lens[[10, 3000]] = [12000, 7000]
        rowptr = np.zeros(n + 1, np.int64)
        rowptr[1:] = np.cumsum(lens)
        cols = np.concatenate([np.sort(rng.choice(n, size=l, replace=l > n)) for l in lens]).astype(np.int32)
        vals = rng.uniform(0, 2, size=rowptr[-1])
        hs = np.add.reduceat(vals, rowptr[:-1])
        f = tf.tf_filter_from_csr(rowptr, cols, vals, hs)
        x, dc = inputs_for(n, 616)
    elif case == "stencil_c3":
        c, x, dc, rmin = synth.workload(3)
        f = tf.tf_build_stencil(3, 160, 80, 80, 1.0, rmin)
    else:
        c, x, dc, rmin = synth.workload(4)
        f = tf.tf_build_filter(dev(c), rmin)
    n = f.n
    xd, dcd = dev(x), dev(dc)
    full_s, full_d = f.sensitivity(xd, dcd), f.density(xd)
    for nrows in sorted({0, 1, 2047, 2048, 2049, 3001, n // 2 + 7, n - 1, n}):
        s = torch.full_like(xd, float("nan"))
        d = torch.full_like(xd, float("nan"))
        f.sensitivity(xd, dcd, out=s, rows=nrows)
        f.density(xd, out=d, rows=nrows)
        assert torch.equal(s[:nrows], full_s[:nrows]), (case, nrows)
        assert torch.equal(d[:nrows], full_d[:nrows]), (case, nrows)
    o = torch.empty_like(xd)
    for bad in (-1, n + 1):
        with pytest.raises(tf.TopofiltError):
            f.sensitivity(xd, dcd, out=o, rows=bad)
        with pytest.raises(tf.TopofiltError):
            f.density(xd, out=o, rows=bad)


def test_streams_concurrent_applies(tf):
    c, x, dc, rmin = synth.workload(3)
    f = tf.tf_build_filter(dev(c), rmin)
    xs, dcs = dev(x), dev(dc)
    ref = f.sensitivity(xs, dcs).clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1, o2 = torch.empty_like(xs), torch.empty_like(xs)
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        f.sensitivity(xs, dcs, out=o1)
    with torch.cuda.stream(s2):
        f.density(xs, out=o2)
    torch.cuda.synchronize()
    assert torch.equal(o1, ref)
    assert torch.equal(o2, f.density(xs))


def test_errors(tf):
    c = synth.quad_grid(10, 10)
    with pytest.raises(tf.TopofiltError, match="not a device pointer") as e:
        h = tf.ctypes.c_void_p()
        tf._check(tf.lib().tf_build_filter(c.ctypes.data_as(tf.ctypes.c_void_p), 100, 2, 1.5,
                                           tf._stream_ptr(), tf.ctypes.byref(h)))
    assert e.value.status == tf.TF_ERR_INVALID
    bad = c.copy()
    bad[7, 1] = np.nan
    with pytest.raises(tf.TopofiltError, match="non-finite"):
        tf.tf_build_filter(dev(bad), 1.5)
    bad[7, 1] = np.inf
    with pytest.raises(tf.TopofiltError, match="non-finite"):
        tf.tf_build_filter(dev(bad), 1.5)
    f = tf.tf_build_filter(dev(c), 1.5)
    xs = dev(np.full(100, 0.5))
    with pytest.raises(tf.TopofiltError, match="overlap"):
        f.sensitivity(xs, dev(np.ones(100)), out=xs)
    with pytest.raises(tf.TopofiltError, match="overlap"):
        f.density(xs, out=xs)
    tf.set_alloc_limit(1024)
    try:
        with pytest.raises(tf.TopofiltError) as e:
            tf.tf_build_filter(dev(synth.quad_grid(100, 100)), 1.5)
        assert e.value.status == tf.TF_ERR_NOMEM
    finally:
        tf.set_alloc_limit(0)
    f2 = tf.tf_build_filter(dev(c), 1.5)  # library still healthy after the failure
    assert f2.nnz == f.nnz


def test_launch_counter_and_stats(tf):
    c, x, dc, rmin = synth.workload(3)
    k0 = tf.kernel_launches()
    f = tf.tf_build_filter(dev(c), rmin, path="cell_list")
    k1 = tf.kernel_launches()
    assert k1 - k0 >= 8
    f.sensitivity(dev(x), dev(dc))
    assert tf.kernel_launches() - k1 == 2  # t pass + the programmatic dependent SpMV launch
    st = f.stats()
    assert st["path"] == "cell_list"
    assert st["bin_side"] >= rmin * (1 + 1e-6)
    assert st["max_candidates"] >= 27 and st["large_rows"] == 0
    g = tf.tf_build_filter(dev(c), rmin)  # lattice path: cubes per axis, the table size
    sg = g.stats()
    assert sg["path"] == "lattice_exact" and sg["bin_side"] == 0.0
    assert sg["bins"] == [160, 80, 80] and sg["max_candidates"] == 27
