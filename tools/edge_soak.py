"""Soak run on degenerate geometries, each through every build path that accepts it (auto, cell_list,
cell_list_bins, dense) against the oracle's brute force, whole CSR bit-exact: huge coordinate offsets,
rmin tiny or huge against the extent, points on a line / in a plane, heavy duplication, single rows of
bins, two-point and one-point sets, mixed-magnitude coordinates. python tools/edge_soak.py [cases]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402


def make(case, rng):
    kind = case % 10
    dim = 2 + (case // 10) % 2
    n = int(rng.integers(1, 3500))
    if kind == 0:    # huge offsets (fp32 offsets from the group origin must still resolve the pairs)
        c = rng.uniform(0, 30, (n, dim)) + float(rng.choice([1e6, 1e8, -3e7, 1e9]))
        rmin = float(rng.uniform(0.8, 2.5))
    elif kind == 1:  # rmin tiny against the extent: the bin grid hits its caps
        c = rng.uniform(0, 1e6, (n, dim))
        rmin = float(rng.uniform(1e-3, 5.0))
    elif kind == 2:  # rmin huge: every pair is a neighbour (one bin)
        n = min(n, 1500)
        c = rng.uniform(0, 1, (n, dim))
        rmin = float(rng.uniform(2.0, 50.0))
    elif kind == 3:  # on a line / in a plane
        c = rng.uniform(0, 200, (n, dim))
        c[:, 1:] = c[0, 1:] if case % 20 < 10 else np.round(c[:, 1:])
        rmin = float(rng.uniform(0.5, 3.0))
    elif kind == 4:  # heavy duplication
        base = rng.uniform(0, 10, (max(1, n // 50), dim))
        c = base[rng.integers(0, base.shape[0], n)]
        rmin = float(rng.uniform(0.3, 2.0))
    elif kind == 5:  # integer lattice points in random order with gaps (exact ties at integer rmin)
        m = int(np.ceil(n ** (1.0 / dim))) + 1
        g = np.stack(np.meshgrid(*[np.arange(m)] * dim, indexing="ij"), -1).reshape(-1, dim).astype(np.float64)
        c = g[rng.permutation(g.shape[0])[:n]]
        rmin = float(rng.integers(1, 4))
    elif kind == 6:  # one or two points, or all identical
        n = int(rng.integers(1, 4))
        c = np.repeat(rng.uniform(-5, 5, (1, dim)), n, axis=0) if case % 20 < 10 else rng.uniform(-5, 5, (n, dim))
        rmin = float(rng.uniform(0.1, 20.0))
    elif kind == 7:  # mixed magnitudes per axis
        c = rng.uniform(0, 1, (n, dim)) * np.array([1e4, 1.0, 1e-3][:dim])
        rmin = float(rng.uniform(0.2, 2.0))
    elif kind == 8:  # negative coordinates, denormal-scale spread in one axis
        c = rng.uniform(-50, 0, (n, dim))
        c[:, -1] *= 1e-300
        rmin = float(rng.uniform(0.5, 2.0))
    else:            # clustered + far outliers
        c = np.concatenate([rng.normal(0, 0.3, (n, dim)), rng.uniform(-1e5, 1e5, (max(1, n // 20), dim))])
        rmin = float(rng.uniform(0.2, 1.0))
    return np.ascontiguousarray(c, dtype=np.float64), rmin


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(4242)
    bad = 0
    for case in range(cases):
        c, rmin = make(case, rng)
        ref = oracle.build_bruteforce(c, rmin)
        cd = torch.from_numpy(c).cuda()
        for path in ("auto", "cell_list", "cell_list_bins", "dense"):
            try:
                f = tf.tf_build_filter(cd, rmin, path=path)
            except tf.TopofiltError as e:
                bad += 1
                print(f"ERROR case {case} kind {case % 10} path {path} n {c.shape[0]} rmin {rmin}: {e}", flush=True)
                continue
            rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
            ok = (np.array_equal(rowptr, ref.rowptr) and np.array_equal(cols, ref.cols) and
                  np.array_equal(vals, ref.vals) and np.allclose(hs, ref.hs, rtol=1e-12, atol=0))
            if not ok:
                bad += 1
                print(f"MISMATCH case {case} kind {case % 10} path {path} ({f.stats()['path']}) n {c.shape[0]} "
                      f"dim {c.shape[1]} rmin {rmin}", flush=True)
            f.close()
    print(f"edge soak: {cases} cases x 4 paths, {bad} problems")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
