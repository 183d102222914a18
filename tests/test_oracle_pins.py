"""Pins for the CPU oracle (oracle/) against what the paper and the mathematics fix.

Each test names the mistake it is there to catch. None of the expected values
comes from the oracle or from the CUDA path: golden fixtures are hand-derived
(tests/golden/*.json, each with a citation and derivation), lattice counts come
from exact integer enumeration (tests/lattice.py), the rest are invariants.
"""
import glob
import json
import math
import os

import numpy as np
import pytest

import lattice
import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden():
    for f in sorted(glob.glob(os.path.join(GOLDEN, "*.json"))):
        yield os.path.basename(f), json.load(open(f))


# ---------------------------------------------------------------- golden (hand-derived)

@pytest.mark.parametrize("name,g", list(_golden()))
def test_golden_weights(name, g):
    """W and Hs of hand-derived cases (SPEC.md:213-214, 224 corrected; 3-4-5 and 3D cases).
    Catches: wrong weight formula, dropped dz term, wrong cut-off, non-strict test."""
    c = np.array(g["centroids"], dtype=np.float64)
    for H in (oracle.build_bruteforce(c, g["rmin"]), oracle.build_celllist(c, g["rmin"])):
        W = H.dense(c.shape[0])
        np.testing.assert_allclose(W, np.array(g["W"], dtype=np.float64), rtol=0, atol=4e-16 * g["rmin"])
        if "Hs" in g:
            np.testing.assert_allclose(H.hs, g["Hs"], rtol=4 * 2.0 ** -52)
        # only pairs strictly inside rmin are stored (zeros of W are absent)
        assert H.nnz == int(np.count_nonzero(np.array(g["W"], dtype=np.float64)))


@pytest.mark.parametrize("name,g", [(n, g) for n, g in _golden() if "sensitivity" in g])
def test_golden_filters(name, g):
    """Sensitivity (Eq. filter / filter_mat) and density filters on hand-derived cases.
    Catches: x_i vs x_j swap, missing x_i in the denominator, missing max(1e-3, x) floor."""
    c = np.array(g["centroids"], dtype=np.float64)
    H = oracle.build_bruteforce(c, g["rmin"])
    s = oracle.apply_sensitivity(H, np.array(g["x"]), np.array(g["dc"]))
    d = oracle.apply_density(H, np.array(g["x"]))
    np.testing.assert_allclose(s, g["sensitivity"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(d, g["density"], rtol=1e-14, atol=1e-15)


# ---------------------------------------------------------------- closed forms (exact integers)

CLOSED = [
    # (name, centroids, rmin, lattice, interior nnz, interior Hs closed form)
    ("c1_quads_60x20", lambda: synth.quad_grid(60, 20), 1.5, lattice.quads(60, 20), 9, 9.5 - 4 * math.sqrt(2)),
    ("quads_17x11", lambda: synth.quad_grid(17, 11), 1.5, lattice.quads(17, 11), 9, 9.5 - 4 * math.sqrt(2)),
    ("c2_like_tris_40x30", lambda: synth.tri_grid(40, 30, "right"), 2.5, lattice.tris_right(40, 30), 41, 33.251217136068),
    ("c3_like_hex_20x14x12", lambda: synth.hex_grid(20, 14, 12), 2.0, lattice.hexes(20, 14, 12), 27,
     48 - 12 * math.sqrt(2) - 8 * math.sqrt(3)),
    ("c5_like_kuhn_12x9x7", lambda: synth.kuhn_tets(12, 9, 7), 1.5, lattice.kuhn(12, 9, 7), 87, 32.133071926883),
]


def test_closed_form_full_configs():
    """SURVEY.md App. A nnz at full size, from exact integer enumeration (no fp64)."""
    assert lattice.quads(60, 20).nnz() == 10_324
    assert lattice.tris_right(300, 100).nnz() == 2_425_680
    assert lattice.hexes(160, 80, 80).nnz() == 27_075_832
    assert lattice.kuhn(200, 100, 100).nnz() == 1_030_251_952
    # BASELINE.json's "~33 neighbours" for config 3 is the non-strict count (reading R1)
    assert lattice.hexes(3, 3, 3).interior(0)[0] == 27
    le = lattice.Lattice((3, 3, 3), ((1, 1, 1),), 2, 4)
    cnt_le = sum(1 for dl in le._deltas() if sum((2 * v) ** 2 for v in dl) <= 16)
    assert cnt_le == 33


@pytest.mark.parametrize("name,cfn,rmin,lat,icount,ihs", CLOSED)
def test_closed_form_lattices(name, cfn, rmin, lat, icount, ihs):
    """Oracle nnz equals the exact lattice count; interior rows have the closed-form
    count and row sum. Catches: wrong bin-neighbour enumeration, <= vs <, d^2 errors."""
    c = cfn()
    H = oracle.build_celllist(c, rmin)
    assert H.nnz == lat.nnz()
    lens = np.diff(H.rowptr)
    assert lens.max() == icount
    # exact interior Hs, from the lattice enumeration and the App. A closed form
    for s in range(len(lat.offsets)):
        assert lat.interior(s)[0] == icount
        assert abs(lat.interior_hs(s) - ihs) < 1e-11
    full = lens == icount
    assert full.sum() > 0
    np.testing.assert_allclose(H.hs[full], ihs, rtol=1e-12)


# ---------------------------------------------------------------- O1 == O2 and invariants

def _workloads_small():
    yield "c1", synth.centroids(1), 1.5
    yield "spec_8x4_right_rmin2", synth.tri_grid(8, 4, "right"), 2.0
    yield "spec_kuhn_6x4x2", synth.kuhn_tets(6, 4, 2), 1.5
    yield "tri_alt_30x12_rmin3", synth.tri_grid(30, 12, "right/left"), 3.0
    yield "rand2d_777", synth.random_points(9001, 777, 2, 0.0, 20.0), 1.7
    yield "rand3d_1013", synth.random_points(9002, 1013, 3, -5.0, 5.0), 1.3
    yield "dup_points", np.repeat(synth.random_points(9003, 40, 3, 0, 3), 3, axis=0), 0.9
    yield "single_point", np.array([[1.0, 2.0, 3.0]]), 0.5
    yield "all_in_one_bin", synth.random_points(9004, 300, 2, 0.0, 1.0), 10.0


@pytest.mark.parametrize("name,c,rmin", list(_workloads_small()))
def test_bruteforce_equals_celllist(name, c, rmin):
    """O2 == O1 bit for bit (structure, weights, Hs) on small and fp-decided workloads."""
    A = oracle.build_bruteforce(c, rmin)
    B = oracle.build_celllist(c, rmin)
    np.testing.assert_array_equal(A.rowptr, B.rowptr)
    np.testing.assert_array_equal(A.cols, B.cols)
    np.testing.assert_array_equal(A.vals, B.vals)
    np.testing.assert_array_equal(A.hs, B.hs)


def test_fp_decided_ties_spec_8x4():
    """SURVEY.md 8(c) point 5: thirds-lattice at integer rmin; fp64 includes tied pairs
    (1,064 entries vs 1,024 in exact arithmetic with ((v0+v1)+v2)/3)."""
    c = synth.tri_grid(8, 4, "right")
    H = oracle.build_bruteforce(c, 2.0)
    assert lattice.tris_right(8, 4, R=12).nnz() == 1024
    assert H.nnz == 1064


def test_bruteforce_equals_celllist_e01():
    """Paper E01 filter sub-workload (180x60 triangles, rmin 2)."""
    c = synth.tri_grid(180, 60, "right")
    A = oracle.build_bruteforce(c, 2.0)
    B = oracle.build_celllist(c, 2.0)
    assert A.nnz == 471_864  # SURVEY.md App. A, fp64 with ((v0+v1)+v2)/3
    np.testing.assert_array_equal(A.cols, B.cols)
    np.testing.assert_array_equal(A.vals, B.vals)
    np.testing.assert_array_equal(A.hs, B.hs)


@pytest.mark.slow
def test_bruteforce_equals_celllist_c2():
    c = synth.centroids(2)
    A = oracle.build_bruteforce(c, 2.5)
    B = oracle.build_celllist(c, 2.5)
    assert A.nnz == 2_425_680
    np.testing.assert_array_equal(A.rowptr, B.rowptr)
    np.testing.assert_array_equal(A.cols, B.cols)
    np.testing.assert_array_equal(A.vals, B.vals)
    np.testing.assert_array_equal(A.hs, B.hs)


@pytest.mark.parametrize("factor", [1.5, 3.0, 7.0])
def test_bin_size_invariance(factor):
    """Chunk/bin-size invariance (SPEC.md:238 analogue): identical CSR for s in {1, 1.5, 3, 7} x rmin."""
    c = synth.random_points(9101, 3000, 3, 0.0, 15.0)
    A = oracle.build_celllist(c, 1.2)
    B = oracle.build_celllist(c, 1.2, bin_factor=factor)
    np.testing.assert_array_equal(A.rowptr, B.rowptr)
    np.testing.assert_array_equal(A.cols, B.cols)
    np.testing.assert_array_equal(A.vals, B.vals)
    np.testing.assert_array_equal(A.hs, B.hs)


@pytest.mark.parametrize("name,c,rmin", list(_workloads_small()))
def test_structural_invariants(name, c, rmin):
    """W symmetric bitwise, W_ii = rmin, 0 <= W <= rmin, Hs >= rmin, columns strictly
    ascending."""
    H = oracle.build_celllist(c, rmin)
    n = c.shape[0]
    rows = np.repeat(np.arange(n), np.diff(H.rowptr))
    assert np.all(H.vals >= 0) and np.all(H.vals <= rmin)
    diag = H.cols == rows
    assert diag.sum() == n and np.all(H.vals[diag] == rmin)
    assert np.all(H.hs >= rmin)
    for r in range(n):
        seg = H.cols[H.rowptr[r]:H.rowptr[r + 1]]
        assert np.all(np.diff(seg) > 0)
    # symmetry: (i,j,w) set equals (j,i,w) set, bitwise on w
    key = rows.astype(np.int64) * n + H.cols
    keyT = H.cols.astype(np.int64) * n + rows
    o1 = np.argsort(key)
    o2 = np.argsort(keyT)
    np.testing.assert_array_equal(key[o1], keyT[o2])
    np.testing.assert_array_equal(H.vals[o1], H.vals[o2])


def test_duplicate_points_columns_ascending():
    c = np.repeat(synth.random_points(9003, 40, 3, 0, 3), 3, axis=0)
    H = oracle.build_celllist(c, 0.9)
    for r in range(c.shape[0]):
        seg = H.cols[H.rowptr[r]:H.rowptr[r + 1]]
        assert np.all(np.diff(seg) > 0)
    # duplicated centroids are at distance 0: weight rmin
    assert H.dense(c.shape[0])[0, 1] == 0.9


# ---------------------------------------------------------------- filter invariants (P5, P6)

def _rand_filter_case():
    c = synth.random_points(9201, 2500, 2, 0.0, 30.0)
    H = oracle.build_celllist(c, 2.2)
    x = synth.uniform(9202, 0, 2500, 0.001, 1.0)
    dc = -3.0 * x * x * synth.uniform(9203, 0, 2500, 0.5, 1.5)
    return c, H, x, dc


def test_density_preserves_constants():
    """Density filter of a constant field is the constant (weighted average), within (k+2) ulp."""
    _, H, x, _ = _rand_filter_case()
    for v in (1.0, 0.37, 1e-3):
        out = oracle.apply_density(H, np.full(x.shape, v))
        k = np.diff(H.rowptr).max()
        np.testing.assert_allclose(out, v, rtol=(k + 2) * 2.0 ** -53)


def test_sensitivity_uniform_returns_dc():
    """uniform density and uniform s -> s."""
    _, H, x, _ = _rand_filter_case()
    out = oracle.apply_sensitivity(H, np.full(x.shape, 0.6), np.full(x.shape, -2.5))
    np.testing.assert_allclose(out, -2.5, rtol=1e-14)


def test_diagonal_identity():
    """rmin below the minimum spacing -> W diagonal -> filtered = input."""
    c = synth.quad_grid(30, 20)
    H = oracle.build_celllist(c, 0.99)
    assert H.nnz == c.shape[0]
    x = synth.uniform(9301, 0, 600, 0.001, 1.0)
    dc = -synth.uniform(9302, 0, 600, 0.0, 1.0)
    np.testing.assert_allclose(oracle.apply_sensitivity(H, x, dc), dc, rtol=4 * 2.0 ** -53)
    np.testing.assert_allclose(oracle.apply_density(H, x), x, rtol=4 * 2.0 ** -53)


def test_sign_preservation():
    """dc <= 0 and x > 0 -> filtered <= 0."""
    _, H, x, dc = _rand_filter_case()
    assert np.all(oracle.apply_sensitivity(H, x, dc) <= 0)


def test_linearity():
    """f(a u + b v) = a f(u) + b f(v) in dc (sensitivity) and x (density)."""
    _, H, x, dc = _rand_filter_case()
    dc2 = -synth.uniform(9401, 0, x.shape[0], 0.0, 2.0)
    a, b = 0.75, -1.25
    lhs = oracle.apply_sensitivity(H, x, a * dc + b * dc2)
    rhs = a * oracle.apply_sensitivity(H, x, dc) + b * oracle.apply_sensitivity(H, x, dc2)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-12 * np.abs(rhs).max())
    x2 = synth.uniform(9402, 0, x.shape[0], 0.001, 1.0)
    lhs = oracle.apply_density(H, a * x + b * x2)
    rhs = a * oracle.apply_density(H, x) + b * oracle.apply_density(H, x2)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-12 * np.abs(rhs).max())


def test_config1_exact_identity():
    """x = 0.5 (a power of two) -> sensitivity(x, dc) equals the density
    formula applied to dc bit for bit. Pins that the numerator uses x_j*dc_j and the
    denominator Hs_i*x_i."""
    c, x, dc, rmin = synth.workload(1)
    H = oracle.build_celllist(c, rmin)
    np.testing.assert_array_equal(oracle.apply_sensitivity(H, x, dc), oracle.apply_density(H, dc))


def test_sampled_rows_match_full():
    """The sampled-row path (used for config 5 parity) equals the full build on those rows."""
    c = synth.kuhn_tets(10, 8, 6)
    cl = oracle.CellList(c, 1.5)
    full = cl.rows()
    rows = synth.sample_rows(5, c.shape[0], 200)
    sub = cl.rows(rows)
    x = synth.density(5, c.shape[0])
    dc = synth.sensitivity(5, x)
    fs = oracle.apply_sensitivity(full, x, dc)
    ss = oracle.apply_sensitivity(sub, x, dc)
    np.testing.assert_array_equal(fs[rows], ss)
    np.testing.assert_array_equal(oracle.apply_density(full, x)[rows], oracle.apply_density(sub, x))
    for k, r in enumerate(rows):
        np.testing.assert_array_equal(full.cols[full.rowptr[r]:full.rowptr[r + 1]],
                                      sub.cols[sub.rowptr[k]:sub.rowptr[k + 1]])


@pytest.mark.parametrize("cfg,count", [(3, 1000), (4, 1000), (5, 400)])  # c5: 400 x 12M tests ~ 45 s
def test_bruteforce_rows_large_configs(cfg, count):
    """seeded rows of configs 3-5, each tested by brute force against ALL N
    points, equal the cell list's rows bit for bit (structure, weights, Hs)."""
    c = synth.centroids(cfg)
    rmin = synth.CONFIGS[cfg]["rmin"]
    rows = np.sort(synth.sample_rows(cfg, c.shape[0], count))
    bf = oracle.build_bruteforce_rows(c, rmin, rows)
    cl = oracle.CellList(c, rmin)
    ref = cl.rows(rows)
    cl.close()
    np.testing.assert_array_equal(bf.rowptr, ref.rowptr)
    np.testing.assert_array_equal(bf.cols, ref.cols)
    np.testing.assert_array_equal(bf.vals, ref.vals)
    np.testing.assert_array_equal(bf.hs, ref.hs)
