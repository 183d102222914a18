"""NEXT-3 on the GPU: tf_helmholtz_* (include/topofilt_helmholtz.h) against the oracle
(oracle/helmholtz.py, pinned in tests/test_helmholtz_oracle.py).

Bars: CSR pattern exact; A, M, node weights, volumes within 1e-13 relative (element formulas
and summation order differ from numpy's LU-based inverse and scipy's duplicate summation);
filtered fields within 1e-9 of max|s~| (CG stopped at ||r|| <= 1e-12 ||b||; the system's
condition number is O(1 + R^2/h^2), so the solution error is a few times the residual)."""
import ctypes
import math

import numpy as np
import pytest

from oracle import helmholtz as hz
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL_SYS = 1e-13
TOL_OUT = 1e-9


@pytest.fixture(scope="module")
def tf():
    assert torch.cuda.is_available()
    import paper_2012_08208_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def meshes():
    return {
        "tri_c2_right_300x100": synth.tri_mesh(300, 100, "right"),
        "tri_alt_jitter_60x40": synth.tri_mesh(60, 40, "right/left", jitter=0.25, stream=91),
        "kuhn_jitter_20x12x10": synth.kuhn_mesh(20, 12, 10, jitter=0.2, stream=92),
        "kuhn_40x24x20": synth.kuhn_mesh(40, 24, 20),
    }


MESHES = meshes()


def assert_close(g, r, tol, what):
    scale = max(1.0, float(np.abs(r).max()))
    err = float(np.abs(np.asarray(g) - np.asarray(r)).max())
    assert err <= tol * scale, f"{what}: max err {err} > {tol} * {scale}"


@pytest.mark.parametrize("name", ["tri_alt_jitter_60x40", "kuhn_jitter_20x12x10"])
def test_assembly_matches_oracle(tf, name):
    nodes, cells = MESHES[name]
    R = 0.9
    A, M, W, vol = hz.system(nodes, cells, R)
    h = tf.tf_helmholtz_build(dev(nodes), dev(cells), R)
    rowptr, cols, vA, vM, Wg, volg = (t.cpu().numpy() for t in h.system())
    np.testing.assert_array_equal(rowptr, A.indptr)
    np.testing.assert_array_equal(cols, A.indices)
    np.testing.assert_array_equal(M.indptr, A.indptr)  # same pattern (M > 0 on every adjacent pair)
    np.testing.assert_allclose(vA, A.data, rtol=RTOL_SYS, atol=RTOL_SYS * np.abs(A.data).max())
    np.testing.assert_allclose(vM, M.data, rtol=RTOL_SYS, atol=RTOL_SYS * np.abs(M.data).max())
    np.testing.assert_allclose(Wg, W, rtol=RTOL_SYS)
    np.testing.assert_allclose(volg, vol, rtol=RTOL_SYS)
    h.close()


@pytest.mark.parametrize("name", list(MESHES))
def test_filter_matches_oracle(tf, name):
    nodes, cells = MESHES[name]
    R = hz.helmholtz_radius(2.5 if name.startswith("tri") else 1.5)
    sigma = synth.uniform(93, 0, cells.shape[0], -1.0, 1.0)
    ref, _ = hz.helmholtz_filter(nodes, cells, R, sigma)
    h = tf.tf_helmholtz_build(dev(nodes), dev(cells), R)
    out, info = h.filter(dev(sigma), rtol=1e-12)
    inf = h.decode_info(info)
    assert inf["converged"] and 0 < inf["iterations"] < 200 and inf["rel_residual"] <= 1e-12
    assert_close(out.cpu().numpy(), ref, TOL_OUT, name)
    h.close()


@pytest.mark.parametrize("name", ["tri_c2_right_300x100", "kuhn_jitter_20x12x10"])
def test_sensitivity_matches_oracle(tf, name):
    nodes, cells = MESHES[name]
    n = cells.shape[0]
    R = hz.helmholtz_radius(2.5 if name.startswith("tri") else 1.5)
    x = synth.uniform(94, 0, n, 0.001, 1.0)
    dc = (-3.0 * (x * x)) * synth.uniform(95, 0, n, 0.5, 1.5)
    ref = hz.helmholtz_sensitivity(nodes, cells, R, x, dc)
    h = tf.tf_helmholtz_build(dev(nodes), dev(cells), R)
    out, info = h.sensitivity(dev(x), dev(dc))
    assert h.decode_info(info)["converged"]
    assert_close(out.cpu().numpy(), ref, TOL_OUT, name)
    # in place over dc is allowed
    dcd = dev(dc)
    h.sensitivity(dev(x), dcd, out=dcd)
    assert_close(dcd.cpu().numpy(), ref, TOL_OUT, name + " in place")
    h.close()


def test_constant_preserved_and_zero_field(tf):
    nodes, cells = MESHES["kuhn_jitter_20x12x10"]
    h = tf.tf_helmholtz_build(dev(nodes), dev(cells), 1.1)
    out, info = h.filter(dev(np.full(cells.shape[0], 3.25)))
    np.testing.assert_allclose(out.cpu().numpy(), 3.25, rtol=1e-12)
    assert h.decode_info(info)["iterations"] <= 2  # the start u = s_n is already the solution
    out, info = h.filter(dev(np.zeros(cells.shape[0])))
    assert not out.cpu().numpy().any()
    inf = h.decode_info(info)
    assert inf["converged"] and inf["iterations"] == 0 and inf["rel_residual"] == 0.0
    h.close()


def test_neumann_cosine_mode_gpu(tf):
    """The closed-form damping of cos(pi x / L) (pinned on the oracle) holds for the GPU path."""
    L, R = 40.0, 3.0
    nodes, cells = synth.kuhn_mesh(40, 2, 2)
    damp = 1.0 / (1.0 + R * R * math.pi ** 2 / (L * L))
    xc = nodes[cells][:, :, 0].mean(axis=1)
    h = tf.tf_helmholtz_build(dev(nodes), dev(cells), R)
    out, _ = h.filter(dev(np.cos(math.pi * xc / L)))
    assert np.abs(out.cpu().numpy() - damp * np.cos(math.pi * xc / L)).max() <= 4e-3
    h.close()


def test_orphan_node_and_determinism(tf):
    nodes, cells = synth.kuhn_mesh(7, 6, 5, jitter=0.2, stream=96)
    nodes = np.vstack([nodes[:10], [[50.0, 50.0, 50.0]], nodes[10:]])
    cells = np.where(cells >= 10, cells + 1, cells).astype(np.int32)  # node 10 is unused
    sigma = synth.uniform(97, 0, cells.shape[0], -1.0, 1.0)
    ref, _ = hz.helmholtz_filter(nodes, cells, 0.8, sigma)
    h = tf.tf_helmholtz_build(dev(nodes), dev(cells), 0.8)
    rowptr = h.system()[0].cpu().numpy()
    assert rowptr[11] == rowptr[10]  # empty row
    a, _ = h.filter(dev(sigma))
    b, _ = h.filter(dev(sigma))
    assert_close(a.cpu().numpy(), ref, TOL_OUT, "orphan")
    assert torch.equal(a, b)
    h.close()


def test_errors(tf):
    nodes, cells = synth.tri_mesh(3, 2)
    with pytest.raises(tf.TopofiltError, match="outside"):
        bad = cells.copy()
        bad[2, 1] = nodes.shape[0]
        tf.tf_helmholtz_build(dev(nodes), dev(bad), 1.0)
    with pytest.raises(tf.TopofiltError, match="volume"):
        bad = cells.copy()
        bad[0, 2] = bad[0, 1]
        tf.tf_helmholtz_build(dev(nodes), dev(bad), 1.0)
    with pytest.raises(tf.TopofiltError, match="R must"):
        tf.tf_helmholtz_build(dev(nodes), dev(cells), -1.0)
    h = tf.tf_helmholtz_build(dev(nodes), dev(cells), 1.0)
    host = np.zeros(cells.shape[0])
    with pytest.raises(tf.TopofiltError, match="device pointer"):
        tf._check(tf.lib().tf_helmholtz_filter(h.handle, ctypes.c_void_p(host.ctypes.data),
                                               ctypes.c_void_p(dev(host).data_ptr()), 1e-10, 10, None, None))
    h.close()
    h = tf.tf_helmholtz_build(dev(nodes), dev(cells), 1.0)
    with pytest.raises(tf.TopofiltError, match="rtol"):
        h.filter(dev(np.zeros(cells.shape[0])), rtol=0.0)
    x = dev(np.full(cells.shape[0], 0.5))
    with pytest.raises(tf.TopofiltError, match="alias"):
        h.sensitivity(x, dev(np.zeros(cells.shape[0])), out=x)
    h.close()


def test_maxit_reports_not_converged(tf):
    nodes, cells = MESHES["kuhn_jitter_20x12x10"]
    h = tf.tf_helmholtz_build(dev(nodes), dev(cells), 2.0)
    _, info = h.filter(dev(synth.uniform(98, 0, cells.shape[0], -1.0, 1.0)), rtol=1e-14, maxit=2)
    inf = h.decode_info(info)
    assert inf["iterations"] == 2 and not inf["converged"] and inf["rel_residual"] > 1e-14
    h.close()


def test_config5_mesh_full_size(tf):
    """The config-5 mesh (200x100x100 cubes, 12M Kuhn tets, 2.04M nodes): the assembled
    pattern has the lattice's 15 entries per interior row; constant fields are preserved;
    the integral identity sum |c| s~_c = sum |c| mean_c(s_n) of the natural-BC solve holds;
    the sensitivity use converges."""
    nodes, cells = synth.kuhn_mesh(200, 100, 100)
    n = cells.shape[0]
    R = hz.helmholtz_radius(1.5)
    h = tf.tf_helmholtz_build(dev(nodes), dev(cells), R)
    rowptr = h.system()[0]
    lens = (rowptr[1:] - rowptr[:-1]).cpu().numpy()
    assert lens.max() == 15 and lens.min() >= 4  # every node is in >= 1 tet
    interior = (nodes[:, 0] > 0) & (nodes[:, 0] < 200) & (nodes[:, 1] > 0) & (nodes[:, 1] < 100) & \
               (nodes[:, 2] > 0) & (nodes[:, 2] < 100)
    assert (lens[interior] == 15).all()
    out, info = h.filter(dev(np.full(n, -0.75)))
    np.testing.assert_allclose(out.cpu().numpy(), -0.75, rtol=1e-11)
    sigma = synth.uniform(99, 0, n, -1.0, 1.0)
    out, info = h.filter(dev(sigma))
    inf = h.decode_info(info)
    assert inf["converged"]
    vol = h.system()[5].cpu().numpy()
    W = h.system()[4].cpu().numpy()
    sn = hz.project(cells, vol, W, sigma)
    lhs = float(np.sum(vol * out.cpu().numpy()))
    rhs = float(np.sum(vol * sn[cells].mean(axis=1)))
    assert abs(lhs - rhs) <= 1e-9 * float(np.sum(vol * np.abs(sigma)))
    x = synth.density(5, n)
    dc = synth.sensitivity(5, x)
    _, info = h.sensitivity(dev(x), dev(dc))
    assert h.decode_info(info)["converged"]
    h.close()
