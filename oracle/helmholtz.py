"""NEXT-3 oracle: the Helmholtz PDE filter (plain numpy / scipy, fp64).

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): imported by tests/ and bench.py's
reference leg, never by the product package.

What it computes (PAPER.md:634 replaces the distance filter by "the Helmholtz filter as
described in [Lazarov and Sigmund 2011]" for the parallel code; the paper gives no formula,
so the operator follows SPEC.md:225-233 and 243 -- DESIGN.md readings R17-R20):

  (-R^2 Laplace + 1) s~ = s  on the P1 (linear simplex) space, natural boundary conditions,
  R = rmin / (2 sqrt 3)                                   (R17)

  1. cell -> node projection by volume-weighted averaging (R18):
         s_n = sum_{c owns n} |c| s_c / sum_{c owns n} |c|
  2. Galerkin system with the standard P1 element matrices (R19): for a simplex with
     vertex coordinates X_0..X_d, J = [X_1 - X_0, ..., X_d - X_0], |c| = |det J| / d!,
     grad lambda_{1..d} = rows of J^{-1}, grad lambda_0 = -sum of them,
         K_c[a,b] = |c| grad lambda_a . grad lambda_b
         M_c[a,b] = |c| (1 + delta_ab) / ((d+1)(d+2))
     assembled A = R^2 K + M,  right-hand side b = M s_n (the projected field, consistent mass)
  3. solve A u = b (a library sparse solve: scipy.sparse.linalg.spsolve, or cg at a stated
     tolerance for large meshes)
  4. node -> cell evaluation as the nodal mean (R18): s~_c = mean_{n in c} u_n
Nodes no cell touches (|c|-weight 0) get s_n = 0 and are left out of the solve (R20).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def helmholtz_radius(rmin: float) -> float:
    """R17: R = rmin / (2 sqrt 3)."""
    return rmin / (2.0 * math.sqrt(3.0))


def p1_elements(nodes: np.ndarray, cells: np.ndarray):
    """Per-cell volume, P1 stiffness and mass matrices (step 2), vectorised over cells."""
    nodes = np.asarray(nodes, dtype=np.float64)
    cells = np.asarray(cells, dtype=np.int64)
    d = nodes.shape[1]
    X = nodes[cells]                                  # (nc, d+1, d)
    J = np.transpose(X[:, 1:, :] - X[:, :1, :], (0, 2, 1))   # columns = edges X_k - X_0
    vol = np.abs(np.linalg.det(J)) / math.factorial(d)
    Jinv = np.linalg.inv(J)                            # row k = grad lambda_{k+1}
    G = np.concatenate([-Jinv.sum(axis=1, keepdims=True), Jinv], axis=1)  # (nc, d+1, d)
    K = vol[:, None, None] * np.einsum("cak,cbk->cab", G, G)
    M = (vol / ((d + 1) * (d + 2)))[:, None, None] * (np.ones((d + 1, d + 1)) + np.eye(d + 1))
    return vol, K, M


def system(nodes: np.ndarray, cells: np.ndarray, R: float):
    """Assembled (A = R^2 K + M, M, node weights W = sum of owning cell volumes, volumes)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    cells = np.asarray(cells, dtype=np.int64)
    nn = nodes.shape[0]
    vol, K, M = p1_elements(nodes, cells)
    d1 = cells.shape[1]
    rows = np.repeat(cells, d1, axis=1).ravel()        # a-major: (c, a, b) -> row cells[c, a]
    cols = np.tile(cells, (1, d1)).ravel()             #          col cells[c, b]
    Ks = sp.coo_matrix((K.ravel(), (rows, cols)), shape=(nn, nn)).tocsr()
    Ms = sp.coo_matrix((M.ravel(), (rows, cols)), shape=(nn, nn)).tocsr()
    Ks.sum_duplicates()
    Ms.sum_duplicates()
    A = (R * R) * Ks + Ms
    A.sort_indices()
    Ms.sort_indices()
    W = np.bincount(cells.ravel(), weights=np.repeat(vol, d1), minlength=nn)
    return A, Ms, W, vol


def project(cells: np.ndarray, vol: np.ndarray, W: np.ndarray, sigma: np.ndarray) -> np.ndarray:
    """Step 1: volume-weighted cell -> node averaging (0 on untouched nodes)."""
    cells = np.asarray(cells, dtype=np.int64)
    num = np.bincount(cells.ravel(), weights=np.repeat(vol * sigma, cells.shape[1]), minlength=W.shape[0])
    out = np.zeros_like(W)
    used = W > 0
    out[used] = num[used] / W[used]
    return out


def helmholtz_filter(nodes, cells, R: float, sigma, solver: str = "direct", rtol: float = 1e-13):
    """Steps 1-4: the filtered cell field s~ (and the nodal solution u)."""
    cells = np.asarray(cells, dtype=np.int64)
    sigma = np.asarray(sigma, dtype=np.float64)
    A, M, W, vol = system(nodes, cells, R)
    sn = project(cells, vol, W, sigma)
    b = M @ sn
    used = np.flatnonzero(W > 0)
    Au = A[used][:, used].tocsc()
    u = np.zeros_like(sn)
    if solver == "direct":
        u[used] = spla.spsolve(Au, b[used])
    else:
        x, info = spla.cg(Au, b[used], x0=sn[used], rtol=rtol, atol=0.0, maxiter=10000)
        if info != 0:
            raise RuntimeError(f"oracle cg did not converge ({info})")
        u[used] = x
    return u[cells].mean(axis=1), u


def helmholtz_sensitivity(nodes, cells, R: float, x, dc, **kw):
    """Sensitivity use ("the caller divides by d_a afterward exactly as in Eq. 21's
    left factor"; floor as in the listing PAPER.md:447): s = x * dc, dc~ = s~ / max(1e-3, x)."""
    x = np.asarray(x, dtype=np.float64)
    st, _ = helmholtz_filter(nodes, cells, R, x * np.asarray(dc, dtype=np.float64), **kw)
    return st / np.maximum(1e-3, x)
