"""Host logic of the lattice build path: tf_lattice_detect_host (no GPU).

Detection proposes (T cells per cube, cubes per axis, spacings) from a prefix and a few probe rows;
the device then verifies every point before the model is used (GPU tests). Pinned here: the
paper's lattice meshes and their variants are recognised with the generator's own parameters,
and non-lattice orders are not.
"""
import numpy as np
import pytest

import synth

tf = pytest.importorskip("paper_2012_08208_b200")


def detect(c):
    return tf.tf_lattice_detect_host(np.ascontiguousarray(c, dtype=np.float64))


def _t3(nx, ny):
    off = synth.uniform(4401, 0, 6, 0.0, 1.0).reshape(3, 2)
    j, i = np.meshgrid(np.arange(ny, dtype=np.float64), np.arange(nx, dtype=np.float64), indexing="ij")
    base = np.stack([i.ravel(), j.ravel()], 1)
    return (base[:, None, :] + off[None, :, :]).reshape(-1, 2)


@pytest.mark.parametrize("name,c,T,cubes,spacing", [
    ("c1_quads", synth.quad_grid(60, 20), 1, (60, 20, 1), (1.0, 1.0)),
    ("c2_tri_right", synth.tri_grid(300, 100, "right"), 2, (300, 100, 1), (1.0, 1.0)),
    ("tri_left", synth.tri_grid(70, 40, "left"), 2, (70, 40, 1), (1.0, 1.0)),
    ("hex", synth.hex_grid(40, 20, 20), 1, (40, 20, 20), (1.0, 1.0, 1.0)),
    ("kuhn", synth.kuhn_tets(20, 10, 8), 6, (20, 10, 8), (1.0, 1.0, 1.0)),
    ("hex_aniso", synth.hex_grid(30, 24, 18) * np.array([1.0, 0.75, 1.25]), 1, (30, 24, 18), (1.0, 0.75, 1.25)),
    ("hex_ny1", synth.hex_grid(20, 1, 15), 1, (20, 1, 15), (1.0, None, 1.0)),
    ("hex_nz1", synth.hex_grid(20, 15, 1), 1, (20, 15, 1), (1.0, 1.0, None)),
    ("quads_one_row", synth.quad_grid(500, 1), 1, (500, 1, 1), (1.0, None)),
    ("t3_random_offsets", _t3(40, 30), 3, (40, 30, 1), (1.0, 1.0)),
    ("duplicate_types", np.repeat(synth.quad_grid(30, 20), 2, axis=0), 2, (30, 20, 1), (1.0, 1.0)),
    ("wide_rows_second_prefix", synth.quad_grid(3000, 5), 1, (3000, 5, 1), (1.0, 1.0)),
    ("kuhn_wide_second_prefix", synth.kuhn_tets(400, 3, 2), 6, (400, 3, 2), (1.0, 1.0, 1.0)),
    ("kuhn_shifted", synth.kuhn_tets(12, 10, 8) + (1.0e3 + 1.0 / 3.0), 6, (12, 10, 8), (1.0, 1.0, 1.0)),
    ("hex_square_layers", synth.hex_grid(6, 6, 6), 1, (6, 6, 6), (1.0, 1.0, 1.0)),
    ("hex_prime_dims", synth.hex_grid(7, 13, 11), 1, (7, 13, 11), (1.0, 1.0, 1.0)),
])
def test_detects_lattices(name, c, T, cubes, spacing):
    m = detect(c)
    assert m is not None, name
    assert m["T"] == T and m["cubes"] == cubes, (name, m)
    for got, want in zip(m["spacing"], spacing):
        if want is not None:
            assert abs(got - want) <= 1e-12 * max(1.0, abs(want)), (name, m)


def _not_lattices():
    rng = np.random.default_rng(4404)
    yield "hex_permuted", synth.hex_grid(20, 16, 12)[rng.permutation(20 * 16 * 12)]
    yield "tri_alternating", synth.tri_grid(60, 40, "right/left")
    yield "hex_nx1", synth.hex_grid(1, 30, 30)
    yield "random_cloud", synth.random_points(4406, 5000, 3, 0, 10)
    yield "lattice_plus_one", np.concatenate([synth.hex_grid(10, 10, 10), [[3.3, 3.3, 3.3]]])
    yield "row_too_wide_for_prefix", synth.quad_grid(40000, 2)  # 2 rows > 65,536 points: declined
    yield "y_major_order", synth.quad_grid(30, 20)[np.arange(600).reshape(20, 30).T.ravel()]
    yield "ground_structure_like", synth.random_points(4407, 3000, 2, 0, 50)
    yield "tiny", synth.quad_grid(1, 3)


@pytest.mark.parametrize("name,c", list(_not_lattices()))
def test_rejects_non_lattices(name, c):
    assert detect(c) is None, name


def test_prefix_only_detection_leaves_verification_to_the_device():
    # points after the prefix displaced: detection (prefix + probes) still proposes the model;
    # tf_build_filter's device pass measures the deviation (GPU test_lattice_path_matches_oracle)
    c = synth.kuhn_tets(16, 12, 10).copy()
    c[-500:] += 0.01
    m = detect(c)
    assert m is not None and m["T"] == 6 and m["cubes"] == (16, 12, 10)


def test_bad_arguments():
    c = np.zeros((10, 4))
    with pytest.raises(tf.TopofiltError, match="TF_ERR_INVALID"):
        detect(c)
