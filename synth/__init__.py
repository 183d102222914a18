"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the filter method (no distances, no weights, no
row sums, no filter formula). It only produces the *input bytes* both sides read:
cell centroids, densities x and sensitivities dc, and sampled row indices.

Recipe (BASELINE.json configs):

* RNG: counter-based SplitMix64. Draw k (k = 0, 1, ...) of stream S is
  ``mix(S + (k+1)*GAMMA) mod 2**64`` with the standard SplitMix64 finaliser;
  ``u01 = (mix >> 11) * 2**-53``; ``U(a,b) = a + (b-a)*u01``.
* Streams: ``S(c, p, t) = 1_000_000*c + 1_000*p + t`` for config c, purpose p
  (1 holes, 2 jitter, 3 x, 4 dc, 5 sampled rows) and iteration t.
* Centroids stand in for the paper's meshes (PAPER.md:330-337 RectangleMesh,
  PAPER.md:461-467 BoxMesh, PAPER.md:588-608 complex ground structure); cell
  midpoint = vertex mean (``cell.midpoint()``), h = 1 everywhere.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def stream_id(c: int, p: int, t: int = 0) -> int:
    return 1_000_000 * c + 1_000 * p + t


def mix(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on a uint64 array (wrap-around arithmetic)."""
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def raw(stream: int, k0: int, count: int) -> np.ndarray:
    """Raw 64-bit draws k0 .. k0+count-1 of a stream."""
    k = np.arange(k0 + 1, k0 + 1 + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(stream) + k * GAMMA
    return mix(z)


def u01(stream: int, k0: int, count: int) -> np.ndarray:
    return (raw(stream, k0, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(stream: int, k0: int, count: int, a: float, b: float) -> np.ndarray:
    return a + (b - a) * u01(stream, k0, count)


# --------------------------------------------------------------------------- centroids

def quad_grid(nx: int, ny: int) -> np.ndarray:
    """Config 1 style quads: index j*nx + i, centroid (i+0.5, j+0.5)."""
    j, i = np.meshgrid(np.arange(ny, dtype=np.float64), np.arange(nx, dtype=np.float64), indexing="ij")
    return np.stack([(i + 0.5).ravel(), (j + 0.5).ravel()], axis=1)


def tri_grid(nx: int, ny: int, pattern: str = "right") -> np.ndarray:
    """2D triangulated rectangle (PAPER.md:332 RectangleMesh): index 2*(j*nx+i)+t.

    "right": every square split along the lower-left -> upper-right diagonal,
      t=0: (i,j),(i+1,j),(i+1,j+1);  t=1: (i,j),(i+1,j+1),(i,j+1).
    "left": split along the lower-right -> upper-left diagonal,
      t=0: (i,j),(i+1,j),(i,j+1);    t=1: (i+1,j),(i+1,j+1),(i,j+1).
    "right/left": alternate per square ((i+j) even -> right).
    Centroid per component = ((v0+v1)+v2)/3 in fp64 (vertex mean).
    """
    j, i = np.meshgrid(np.arange(ny, dtype=np.float64), np.arange(nx, dtype=np.float64), indexing="ij")
    i = i.ravel()
    j = j.ravel()

    def cen(a, b, c):
        return ((a + b) + c) / 3.0

    r0 = (cen(i, i + 1, i + 1), cen(j, j, j + 1))
    r1 = (cen(i, i + 1, i), cen(j, j + 1, j + 1))
    l0 = (cen(i, i + 1, i), cen(j, j, j + 1))
    l1 = (cen(i + 1, i + 1, i), cen(j, j + 1, j + 1))
    if pattern == "right":
        t0, t1 = r0, r1
    elif pattern == "left":
        t0, t1 = l0, l1
    elif pattern in ("right/left", "alternate"):
        even = ((i + j) % 2) == 0
        t0 = (np.where(even, r0[0], l0[0]), np.where(even, r0[1], l0[1]))
        t1 = (np.where(even, r1[0], l1[0]), np.where(even, r1[1], l1[1]))
    else:
        raise ValueError(pattern)
    out = np.empty((i.size * 2, 2), dtype=np.float64)
    out[0::2, 0], out[0::2, 1] = t0
    out[1::2, 0], out[1::2, 1] = t1
    return out


def hex_grid(nx: int, ny: int, nz: int) -> np.ndarray:
    """Config 3: index (k*ny + j)*nx + i, centroid (i+1/2, j+1/2, k+1/2)."""
    k, j, i = np.meshgrid(np.arange(nz, dtype=np.float64), np.arange(ny, dtype=np.float64),
                          np.arange(nx, dtype=np.float64), indexing="ij")
    return np.stack([(i + 0.5).ravel(), (j + 0.5).ravel(), (k + 0.5).ravel()], axis=1)


_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def kuhn_tets(nx: int, ny: int, nz: int) -> np.ndarray:
    """Config 5 / BoxMesh-style: each cube split into 6 Kuhn tetrahedra.

    Index 6*((k*ny + j)*nx + i) + t, t enumerates the permutations sigma of (x,y,z)
    in lexicographic order; v0=(i,j,k), v1=v0+e_s1, v2=v1+e_s2, v3=v0+(1,1,1);
    centroid (((v0+v1)+v2)+v3)/4 (exact in fp64: quarters).
    """
    k, j, i = np.meshgrid(np.arange(nz, dtype=np.float64), np.arange(ny, dtype=np.float64),
                          np.arange(nx, dtype=np.float64), indexing="ij")
    base = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1)
    ncube = base.shape[0]
    out = np.empty((ncube, 6, 3), dtype=np.float64)
    for t, s in enumerate(_PERMS):
        v0 = base
        e1 = np.zeros(3)
        e1[s[0]] = 1.0
        e2 = np.zeros(3)
        e2[s[1]] = 1.0
        v1 = v0 + e1
        v2 = v1 + e2
        v3 = v0 + 1.0
        out[:, t, :] = (((v0 + v1) + v2) + v3) / 4.0
    return out.reshape(ncube * 6, 3)


def tri_lattice_offsets(pattern: str = "right") -> np.ndarray:
    """Type offsets (fractions of h) of tri_grid's two triangles per square, in its t order
    (vertex means: "right" t0 = (2/3, 1/3), t1 = (1/3, 2/3); "left" t0 = (1/3, 1/3), t1 = (2/3, 2/3))."""
    if pattern == "right":
        return np.array([[2.0 / 3.0, 1.0 / 3.0], [1.0 / 3.0, 2.0 / 3.0]])
    if pattern == "left":
        return np.array([[1.0 / 3.0, 1.0 / 3.0], [2.0 / 3.0, 2.0 / 3.0]])
    raise ValueError("periodic with two types per square: 'right' or 'left'")


def kuhn_lattice_offsets() -> np.ndarray:
    """Type offsets of kuhn_tets' six tetrahedra per cube, in its t order: (2 e_s1 + e_s2 + 1)/4."""
    out = []
    for s in _PERMS:
        o = np.ones(3)
        o[s[0]] += 2.0
        o[s[1]] += 1.0
        out.append(o / 4.0)
    return np.array(out)


def tri_mesh(nx: int, ny: int, pattern: str = "right", jitter: float = 0.0, stream: int = 0):
    """Nodes and cells of the tri_grid triangulation (same cell order and vertex order, so the
    vertex means are tri_grid's centroids when jitter = 0). Node index j*(nx+1) + i at (i, j);
    `jitter` > 0 moves every interior node by U(-jitter, jitter) per component (stream)."""
    J, I = np.meshgrid(np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    nodes = np.stack([I.ravel(), J.ravel()], axis=1).astype(np.float64)
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    i = i.ravel()
    j = j.ravel()
    v = lambda a, b: b * (nx + 1) + a  # noqa: E731
    r0 = (v(i, j), v(i + 1, j), v(i + 1, j + 1))
    r1 = (v(i, j), v(i + 1, j + 1), v(i, j + 1))
    l0 = (v(i, j), v(i + 1, j), v(i, j + 1))
    l1 = (v(i + 1, j), v(i + 1, j + 1), v(i, j + 1))
    if pattern == "right":
        t0, t1 = r0, r1
    elif pattern == "left":
        t0, t1 = l0, l1
    elif pattern in ("right/left", "alternate"):
        even = ((i + j) % 2) == 0
        t0 = tuple(np.where(even, a, b) for a, b in zip(r0, l0))
        t1 = tuple(np.where(even, a, b) for a, b in zip(r1, l1))
    else:
        raise ValueError(pattern)
    cells = np.empty((i.size * 2, 3), dtype=np.int32)
    cells[0::2] = np.stack(t0, axis=1)
    cells[1::2] = np.stack(t1, axis=1)
    if jitter > 0:
        _jitter_interior(nodes, [nx, ny], jitter, stream)
    return nodes, cells


def kuhn_mesh(nx: int, ny: int, nz: int, jitter: float = 0.0, stream: int = 0):
    """Nodes and cells of kuhn_tets (same cell and vertex order: v0, v1 = v0+e_s1,
    v2 = v1+e_s2, v3 = v0+(1,1,1)). Node index (k*(ny+1) + j)*(nx+1) + i at (i, j, k)."""
    K, J, I = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    nodes = np.stack([I.ravel(), J.ravel(), K.ravel()], axis=1).astype(np.float64)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    base = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1)
    node = lambda p: (p[:, 2] * (ny + 1) + p[:, 1]) * (nx + 1) + p[:, 0]  # noqa: E731
    cells = np.empty((base.shape[0], 6, 4), dtype=np.int32)
    for t, s in enumerate(_PERMS):
        e1 = np.zeros(3, dtype=np.int64)
        e1[s[0]] = 1
        e2 = np.zeros(3, dtype=np.int64)
        e2[s[1]] = 1
        cells[:, t, 0] = node(base)
        cells[:, t, 1] = node(base + e1)
        cells[:, t, 2] = node(base + e1 + e2)
        cells[:, t, 3] = node(base + 1)
    if jitter > 0:
        _jitter_interior(nodes, [nx, ny, nz], jitter, stream)
    return nodes, cells.reshape(-1, 4)


def _jitter_interior(nodes, n, jitter, stream):
    inner = np.ones(nodes.shape[0], dtype=bool)
    for d, nd in enumerate(n):
        inner &= (nodes[:, d] > 0) & (nodes[:, d] < nd)
    m = int(inner.sum())
    nodes[inner] += uniform(stream, 0, m * len(n), -jitter, jitter).reshape(m, len(n))


def ground_structure(config: int = 4, nx: int = 2000, ny: int = 1000):
    """Config 4: jittered 2D grid with 5 seeded circular holes and an L-bracket cut-out.

    Holes: triples (cx=nx*u, cy=ny*u, r=50+100u) from stream p=1, rejected while the
    centre lies in the removed upper-right quadrant; 5 accepted.
    Points: q = j*nx + i -> ((i+0.5) + (-0.3+0.6*u(2q)), (j+0.5) + (-0.3+0.6*u(2q+1)))
    with stream p=2 (draws consumed for every q). Removal: upper-right quadrant
    (px >= nx/2 and py >= ny/2) or strictly inside a hole.
    Returns (centroids [N,2], holes [5,3]).
    """
    s_holes = stream_id(config, 1, 0)
    holes = []
    k = 0
    while len(holes) < 5:
        u = u01(s_holes, k, 3)
        k += 3
        cx = nx * u[0]
        cy = ny * u[1]
        r = 50.0 + 100.0 * u[2]
        if cx >= nx / 2 and cy >= ny / 2:
            continue
        holes.append((cx, cy, r))
    holes = np.array(holes, dtype=np.float64)
    s_jit = stream_id(config, 2, 0)
    npts = nx * ny
    uj = u01(s_jit, 0, 2 * npts)
    j, i = np.meshgrid(np.arange(ny, dtype=np.float64), np.arange(nx, dtype=np.float64), indexing="ij")
    px = (i.ravel() + 0.5) + (-0.3 + 0.6 * uj[0::2])
    py = (j.ravel() + 0.5) + (-0.3 + 0.6 * uj[1::2])
    keep = ~((px >= nx / 2) & (py >= ny / 2))
    for cx, cy, r in holes:
        keep &= ~(((px - cx) ** 2 + (py - cy) ** 2) < r * r)
    return np.stack([px[keep], py[keep]], axis=1), holes


# --------------------------------------------------------------------------- configs

CONFIGS = {
    1: dict(name="c1_mbb_quads_60x20", dim=2, rmin=1.5, applies=1),
    2: dict(name="c2_tri_300x100", dim=2, rmin=2.5, applies=50),
    3: dict(name="c3_hex_160x80x80", dim=3, rmin=2.0, applies=100),
    4: dict(name="c4_ground_structure_2000x1000", dim=2, rmin=3.0, applies=50),
    5: dict(name="c5_kuhn_200x100x100", dim=3, rmin=1.5, applies=20),
}


def centroids(config: int) -> np.ndarray:
    if config == 1:
        return quad_grid(60, 20)
    if config == 2:
        return tri_grid(300, 100, "right")
    if config == 3:
        return hex_grid(160, 80, 80)
    if config == 4:
        return ground_structure(4)[0]
    if config == 5:
        return kuhn_tets(200, 100, 100)
    raise ValueError(config)


def density(config: int, n: int) -> np.ndarray:
    """x: 0.5 everywhere for config 1, else U(0.001, 1) from stream S(c,3,0)."""
    if config == 1:
        return np.full(n, 0.5, dtype=np.float64)
    return uniform(stream_id(config, 3, 0), 0, n, 0.001, 1.0)


def sensitivity(config: int, x: np.ndarray, t: int = 0) -> np.ndarray:
    """dc: -U(0,1) for configs 1 and 4, else -3*(x*x)*U(0.5,1.5); stream S(c,4,t)."""
    n = x.shape[0]
    u = uniform(stream_id(config, 4, t), 0, n, 0.5, 1.5) if config not in (1, 4) else None
    if u is None:
        return -uniform(stream_id(config, 4, t), 0, n, 0.0, 1.0)
    return (-3.0 * (x * x)) * u


def sample_rows(config: int, n: int, count: int) -> np.ndarray:
    """First `count` distinct rows floor(u*N) from successive draws of S(c,5,0)."""
    s = stream_id(config, 5, 0)
    seen = set()
    out = []
    k = 0
    while len(out) < min(count, n):
        u = u01(s, k, 4 * count)
        k += 4 * count
        for r in np.floor(u * n).astype(np.int64):
            r = int(min(r, n - 1))
            if r not in seen:
                seen.add(r)
                out.append(r)
                if len(out) == count:
                    break
    return np.array(out, dtype=np.int64)


def random_points(seed_stream: int, n: int, dim: int, lo: float, hi: float) -> np.ndarray:
    """Uniform random cloud (edge-case and ragged-size tests)."""
    return uniform(seed_stream, 0, n * dim, lo, hi).reshape(n, dim)


def workload(config: int):
    """Centroids, x, dc(t=0) and rmin for a config."""
    c = centroids(config)
    x = density(config, c.shape[0])
    dc = sensitivity(config, x, 0)
    return c, x, dc, CONFIGS[config]["rmin"]
