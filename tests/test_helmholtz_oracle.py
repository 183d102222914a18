"""Pins of the Helmholtz-filter oracle (NEXT-3, oracle/helmholtz.py) against things other than
itself: hand-derived element/assembly fixtures, exact identities of the P1 Galerkin system,
the closed-form Neumann eigenmode of the continuous operator, and a pure-Python evaluation of
the R = 0 limit."""
import json
import math
import os

import numpy as np
import pytest

from oracle import helmholtz as hz
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "helmholtz")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_unit_square_two_triangles_fixture():
    g = load("p1_unit_square_two_triangles.json")
    nodes, cells = np.array(g["nodes"]), np.array(g["cells"])
    A0, M, W, vol = hz.system(nodes, cells, 0.0)   # R = 0: A = M
    A1, _, _, _ = hz.system(nodes, cells, 1.0)     # R = 1: A = K + M
    np.testing.assert_allclose(vol, g["volumes"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(M.toarray() * 24.0, g["M24"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(A0.toarray(), M.toarray(), rtol=0, atol=0)
    np.testing.assert_allclose((A1 - A0).toarray(), g["K"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(W, g["node_weights"], rtol=0, atol=1e-15)


def test_unit_tet_fixture():
    g = load("p1_unit_tet.json")
    vol, K, M = hz.p1_elements(np.array(g["nodes"]), np.array(g["cells"]))
    np.testing.assert_allclose(vol, g["volumes"], rtol=1e-15)
    np.testing.assert_allclose(K[0] * 6.0, g["K6"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(M[0] * 120.0, g["M120"], rtol=0, atol=1e-13)


def test_element_invariance_under_vertex_order():
    """Reordering a cell's vertices (either orientation) permutes K and M and keeps |c|."""
    nodes, cells = synth.kuhn_mesh(2, 2, 2, jitter=0.2, stream=71)
    v1, K1, M1 = hz.p1_elements(nodes, cells)
    perm = [2, 0, 3, 1]
    v2, K2, M2 = hz.p1_elements(nodes, cells[:, perm])
    np.testing.assert_allclose(v2, v1, rtol=1e-14)
    np.testing.assert_allclose(K2, K1[:, perm][:, :, perm], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(M2, M1[:, perm][:, :, perm], rtol=1e-14)


@pytest.mark.parametrize("mesh", ["tri_right", "tri_alt_jitter", "kuhn", "kuhn_jitter"])
def test_system_identities(mesh):
    """K 1 = 0 (row sums), A symmetric, M row sums = W/(d+1) (integral of a hat function),
    total volume = box volume."""
    if mesh.startswith("tri"):
        nodes, cells = synth.tri_mesh(9, 6, "right" if mesh == "tri_right" else "right/left",
                                      jitter=0.25 if "jitter" in mesh else 0.0, stream=72)
        box, d = 9 * 6, 2
    else:
        nodes, cells = synth.kuhn_mesh(5, 4, 3, jitter=0.2 if "jitter" in mesh else 0.0, stream=73)
        box, d = 5 * 4 * 3, 3
    R = 0.7
    A, M, W, vol = hz.system(nodes, cells, R)
    K = (A - M) / (R * R)
    assert abs(vol.sum() - box) <= 1e-11 * box
    assert np.abs(K @ np.ones(K.shape[0])).max() <= 1e-12
    assert abs(A - A.T).max() <= 1e-15
    np.testing.assert_allclose(M @ np.ones(M.shape[0]), W / (d + 1), rtol=1e-13)


@pytest.mark.parametrize("dim", [2, 3])
def test_constant_field_preserved(dim):
    """A constant field is a solution (K 1 = 0, projection and nodal mean keep constants)."""
    if dim == 2:
        nodes, cells = synth.tri_mesh(12, 7, "right/left", jitter=0.2, stream=74)
    else:
        nodes, cells = synth.kuhn_mesh(6, 5, 4, jitter=0.15, stream=75)
    st, _ = hz.helmholtz_filter(nodes, cells, 1.3, np.full(cells.shape[0], -2.5))
    np.testing.assert_allclose(st, -2.5, rtol=1e-12)


@pytest.mark.parametrize("dim", [2, 3])
def test_conservation(dim):
    """With natural BCs, 1^T A u = 1^T M u = 1^T M s_n, so the integral of the solution equals
    that of the projected field; P1 integrates exactly as |c| times the vertex mean."""
    if dim == 2:
        nodes, cells = synth.tri_mesh(10, 8, "left", jitter=0.25, stream=76)
    else:
        nodes, cells = synth.kuhn_mesh(5, 5, 4, jitter=0.2, stream=77)
    sigma = synth.uniform(78, 0, cells.shape[0], -1.0, 1.0)
    A, M, W, vol = hz.system(nodes, cells, 0.9)
    sn = hz.project(cells, vol, W, sigma)
    st, _ = hz.helmholtz_filter(nodes, cells, 0.9, sigma)
    lhs = float(np.sum(vol * st))
    rhs = float(np.sum(vol * sn[cells].mean(axis=1)))
    assert abs(lhs - rhs) <= 1e-12 * float(np.sum(vol * np.abs(sigma)))
    # smoothing: the filtered field stays inside the range of the projected one (max principle
    # does not hold exactly for P1 + consistent mass, so only the extremes' order is checked)
    assert st.max() < sigma.max() and st.min() > sigma.min()


@pytest.mark.parametrize("dim", [2, 3])
def test_neumann_cosine_mode(dim):
    """cos(pi x / L) is an eigenfunction of -Laplace with natural BCs on [0, L] x ...: the
    continuous filter maps it to cos(pi x / L) / (1 + R^2 pi^2 / L^2). The P1 solution of
    A u = M f (nodal f) matches at O(h^2); so does the whole cell pipeline on cell midpoints."""
    L, R = 40.0, 3.0
    if dim == 2:
        nodes, cells = synth.tri_mesh(40, 3, "right/left")
    else:
        nodes, cells = synth.kuhn_mesh(40, 2, 2)
    damp = 1.0 / (1.0 + R * R * math.pi ** 2 / (L * L))
    A, M, W, vol = hz.system(nodes, cells, R)
    f = np.cos(math.pi * nodes[:, 0] / L)
    import scipy.sparse.linalg as spla
    u = spla.spsolve(A.tocsc(), M @ f)
    assert np.abs(u - damp * f).max() <= 2e-3
    # a wrong R^2 scale (R instead of R^2, or K doubled) moves the damping by > 1.5%
    assert abs(1.0 / (1.0 + R * math.pi ** 2 / L ** 2) - damp) > 0.015
    xc = nodes[cells][:, :, 0].mean(axis=1)
    st, _ = hz.helmholtz_filter(nodes, cells, R, np.cos(math.pi * xc / L))
    assert np.abs(st - damp * np.cos(math.pi * xc / L)).max() <= 4e-3


def test_zero_radius_is_project_then_average():
    """R = 0: A = M and u = s_n; s~_c = vertex mean of the volume-weighted projection, evaluated
    here with plain Python loops (independent of the vectorised oracle)."""
    nodes, cells = synth.tri_mesh(4, 3, "right/left", jitter=0.2, stream=79)
    sigma = synth.uniform(80, 0, cells.shape[0], -1.0, 1.0)
    st, _ = hz.helmholtz_filter(nodes, cells, 0.0, sigma)
    nn = nodes.shape[0]
    num = [0.0] * nn
    den = [0.0] * nn
    for c, tri in enumerate(cells.tolist()):
        (x0, y0), (x1, y1), (x2, y2) = (nodes[v].tolist() for v in tri)
        area = abs((x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0)) / 2.0
        for v in tri:
            num[v] += area * sigma[c]
            den[v] += area
    sn = [num[v] / den[v] for v in range(nn)]
    want = [sum(sn[v] for v in tri) / 3.0 for tri in cells.tolist()]
    np.testing.assert_allclose(st, want, rtol=1e-11, atol=1e-13)


def test_orphan_node_and_direct_vs_cg():
    """A node no cell uses is left out (R20); scipy's direct and CG solves agree."""
    nodes, cells = synth.kuhn_mesh(4, 3, 3, jitter=0.2, stream=81)
    nodes = np.vstack([nodes, [[100.0, 100.0, 100.0]]])
    sigma = synth.uniform(82, 0, cells.shape[0], -1.0, 0.0)
    s1, u1 = hz.helmholtz_filter(nodes, cells, 0.8, sigma)
    s2, u2 = hz.helmholtz_filter(nodes, cells, 0.8, sigma, solver="cg", rtol=1e-14)
    assert u1[-1] == 0.0 and u2[-1] == 0.0
    np.testing.assert_allclose(s2, s1, rtol=1e-11, atol=1e-13)


def test_radius_mapping():
    assert hz.helmholtz_radius(2.0 * math.sqrt(3.0)) == pytest.approx(1.0, rel=1e-15)
