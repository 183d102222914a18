"""Medium-large random clouds (1-4M points, 2D and 3D, clustered and uniform, 20-90 neighbours per
point) through the default path and the per-bin kernels, the whole CSR compared bit for bit with the
oracle's cell list, both filters within 1e-10. python tools/large_soak.py [cases]."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    rng = np.random.default_rng(99)
    bad = 0
    for case in range(cases):
        dim = 2 + case % 2
        n = int(rng.integers(1_000_000, 4_000_000))
        target = float(rng.uniform(20, 90))  # neighbours per point
        if dim == 2:
            side = np.sqrt(n)
            rmin = np.sqrt(target / np.pi)
        else:
            side = n ** (1.0 / 3.0)
            rmin = (target * 3.0 / (4.0 * np.pi)) ** (1.0 / 3.0)
        c = rng.uniform(0, side, (n, dim))
        if case % 3 == 2:  # a denser region: rows several times the mean
            k = n // 10
            c[:k] = rng.uniform(0, side / 8, (k, dim))
        c = np.ascontiguousarray(c)
        t0 = time.time()
        ref = oracle.build_celllist(c, float(rmin))
        t1 = time.time()
        cd = torch.from_numpy(c).cuda()
        x = rng.uniform(0.001, 1.0, n)
        dc = -rng.uniform(0.0, 1.0, n)
        for path in ("auto", "cell_list_bins"):
            f = tf.tf_build_filter(cd, float(rmin), path=path)
            rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
            ok = (np.array_equal(rowptr, ref.rowptr) and np.array_equal(cols, ref.cols) and
                  np.array_equal(vals, ref.vals) and np.allclose(hs, ref.hs, rtol=1e-12, atol=0))
            if path == "auto":
                s = f.sensitivity(torch.from_numpy(x).cuda(), torch.from_numpy(dc).cuda()).cpu().numpy()
                rs = oracle.apply_sensitivity(ref, x, dc)
                ok = ok and bool(np.all(np.abs(s - rs) <= 1e-10 * np.abs(rs)))
            print(f"case {case} dim {dim} n {n:,} nnz {ref.nnz:,} maxrow {int(np.diff(ref.rowptr).max())} "
                  f"path {path}->{f.stats()['path']} groups {f.stats()['groups']} ok {ok} (oracle {t1 - t0:.0f} s)",
                  flush=True)
            bad += not ok
            f.close()
    print(f"large soak: {cases} cases x 2 paths, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
