"""The all-pairs ablation build (TF_BUILD_DENSE, dense_build.cu): the paper's own method -- every
pair of midpoints visited (listing PAPER.md:442-445) -- must produce the oracle's
CSR bit for bit, and Hs bitwise (both sum in ascending column order)."""
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


def _cases():
    yield "c1_quads", synth.quad_grid(60, 20), 1.5
    yield "tri_right_left", synth.tri_grid(40, 30, "right/left"), 2.0          # fp-decided ties (R5b)
    yield "kuhn_7x5x4", synth.kuhn_tets(7, 5, 4), 1.5
    yield "jittered_2d", synth.ground_structure(4, 400, 200)[0], 3.0  # 11,410 jittered points, holes
    yield "random_3d", synth.random_points(5501, 3000, 3, 0.0, 12.0), 1.3
    yield "ragged_tail", synth.random_points(5502, 128 * 3 + 17, 2, 0.0, 9.0), 1.1  # rows and tiles with a tail
    yield "single_point", np.array([[0.25, 0.5, 0.75]]), 1.0
    yield "duplicates", np.repeat(synth.random_points(5503, 200, 2, 0.0, 4.0), 2, axis=0), 0.9


@pytest.mark.parametrize("name,c,rmin", list(_cases()))
def test_dense_matches_oracle(tf, name, c, rmin):
    ref = oracle.build_bruteforce(c, rmin) if c.shape[0] <= 4000 else oracle.build_celllist(c, rmin)
    f = tf.tf_build_filter(dev(c), rmin, path="dense")
    assert f.stats()["path"] == "dense"
    rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
    np.testing.assert_array_equal(rowptr, ref.rowptr)
    np.testing.assert_array_equal(cols, ref.cols)
    np.testing.assert_array_equal(vals, ref.vals)
    np.testing.assert_array_equal(hs, ref.hs)  # same ascending-column order of summation
    # and the applies run on a dense-built handle like on any other
    n = c.shape[0]
    x = synth.uniform(91, 0, n, 0.001, 1.0)
    dc = -synth.uniform(92, 0, n, 0.0, 1.0)
    s = f.sensitivity(dev(x), dev(dc)).cpu().numpy()
    np.testing.assert_allclose(s, oracle.apply_sensitivity(ref, x, dc), rtol=1e-10)
    f.close()


def test_dense_config2_equals_cell_list(tf):
    c, _, _, rmin = synth.workload(2)
    fd = tf.tf_build_filter(dev(c), rmin, path="dense")
    fc = tf.tf_build_filter(dev(c), rmin, path="cell_list")
    for a, b in zip(fd.csr()[:3], fc.csr()[:3]):
        assert torch.equal(a, b)
    fd.close()
    fc.close()


def test_dense_rejects_bad_input(tf):
    c = synth.random_points(5504, 500, 3, 0.0, 5.0).copy()
    c[77, 1] = np.nan
    with pytest.raises(tf.TopofiltError, match="TF_ERR_INVALID"):
        tf.tf_build_filter(dev(c), 1.0, path="dense")
