"""Soak run of the lattice build (exact mode with closed-form row pointers, and tested mode) on random
small lattices: random cube counts (including axes shorter than the reach), 1-6 cells per cube at
random dyadic offsets (exact mode) or perturbed ones (tested mode), random rmin, 2D and 3D -- whole CSR
bit-exact against the oracle's brute force. python tools/lattice_soak.py [cases]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    rng = np.random.default_rng(20261021)
    bad = 0
    paths = {}
    for case in range(cases):
        dim = int(rng.integers(2, 4))
        nd = [int(rng.integers(2, 14)), int(rng.integers(1, 12)), int(rng.integers(1, 9)) if dim == 3 else 1]
        T = int(rng.choice([1, 1, 2, 3, 6]))
        h = float(rng.choice([1.0, 0.5, 2.0]))
        off = rng.integers(0, 8, size=(T, dim)) / 8.0 * h  # dyadic offsets inside the cube
        if case % 3 == 2:
            off = off + rng.uniform(-0.01, 0.01, size=off.shape) * h  # near-lattice: tested mode
        rmin = float(rng.choice([1.0, 1.5, 2.0, 2.5, 3.0])) * h * float(rng.choice([1.0, 1.0, 0.75]))
        k, j, i = np.meshgrid(np.arange(nd[2]), np.arange(nd[1]), np.arange(nd[0]), indexing="ij")
        cube = np.stack([i.ravel(), j.ravel(), k.ravel()], 1)[:, :dim].astype(np.float64) * h
        c = (cube[:, None, :] + off[None, :, :]).reshape(-1, dim) + 0.25 * h
        c = np.ascontiguousarray(c)
        ref = oracle.build_bruteforce(c, rmin)
        f = tf.tf_build_filter(torch.from_numpy(c).cuda(), rmin)
        p = f.stats()["path"]
        paths[p] = paths.get(p, 0) + 1
        rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
        ok = (np.array_equal(rowptr, ref.rowptr) and np.array_equal(cols, ref.cols) and np.array_equal(vals, ref.vals)
              and np.allclose(hs, ref.hs, rtol=1e-12, atol=0))
        if not ok:
            bad += 1
            print(f"MISMATCH case {case}: dim {dim} cubes {nd} T {T} h {h} rmin {rmin} path {p}", flush=True)
        f.close()
    print(f"lattice soak: {cases} cases, paths {paths}, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
