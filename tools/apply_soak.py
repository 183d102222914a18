"""Soak run of the apply kernels alone on random CSR matrices (tf_filter_from_csr): row lengths from a
heavy-tailed mix (1-10, 20-120, occasional rows of thousands of entries, longer than a staging window),
random ascending columns, positive weights -- sensitivity, density, both-in-one-pass (bitwise the separate
calls), random row ranges and row prefixes, against the oracle's row loops (1e-10).
python tools/apply_soak.py [cases]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402


def rel_ok(g, r, tol=1e-10):
    scale = np.where(r != 0, np.abs(r), np.abs(r).max() if r.size else 1.0)
    return bool(np.all(np.abs(g - r) <= tol * scale))


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 120
    rng = np.random.default_rng(2718)
    bad = 0
    for case in range(cases):
        n = int(rng.integers(1, 120000)) if case % 5 else int(rng.integers(1, 200))
        kind = rng.choice(4, size=n, p=[0.55, 0.4, 0.045, 0.005])
        lens = np.where(kind == 0, rng.integers(1, 11, n), np.where(kind == 1, rng.integers(20, 121, n),
                        np.where(kind == 2, rng.integers(200, 900, n), rng.integers(2500, 9000, n))))
        lens = np.minimum(lens, n).astype(np.int64)
        if case % 7 == 0:
            lens[:] = int(rng.integers(1, min(n, 200) + 1))  # uniform rows
        rowptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=rowptr[1:])
        nnz = int(rowptr[-1])
        cols = np.empty(nnz, dtype=np.int32)
        for r in range(n):  # ascending distinct columns in a window around the row (index-local, like H)
            L = int(lens[r])
            w = min(n, max(L, int(L * rng.uniform(1.0, 4.0))))
            lo = int(np.clip(r - w // 2, 0, n - w))
            cols[rowptr[r]:rowptr[r + 1]] = np.sort(rng.choice(w, size=L, replace=False)) + lo
        vals = rng.uniform(0.0, 2.0, nnz)
        hs = np.maximum(np.add.reduceat(vals, rowptr[:-1]), 1e-3)
        H = oracle.CSR(rowptr, cols, vals, hs)
        x = rng.uniform(0.0005, 1.0, n)  # some below the 1e-3 floor
        dc = -rng.uniform(0.0, 1.0, n)
        rs, rd = oracle.apply_sensitivity(H, x, dc), oracle.apply_density(H, x)
        f = tf.tf_filter_from_csr(rowptr, cols, vals, hs)
        xd, dcd = torch.from_numpy(x).cuda(), torch.from_numpy(dc).cuda()
        s, d = f.sensitivity(xd, dcd), f.density(xd)
        ok = rel_ok(s.cpu().numpy(), rs) and rel_ok(d.cpu().numpy(), rd)
        sb, db = f.both(xd, dcd)
        ok = ok and torch.equal(sb, s) and torch.equal(db, d)
        r0, r1 = sorted(int(v) for v in rng.integers(0, n + 1, 2))
        so, do = torch.full_like(xd, 5.0), torch.full_like(xd, 5.0)
        tf.tf_sensitivity_filter_range(f, xd, dcd, so, r0, r1)
        tf.tf_density_filter_range(f, xd, do, r0, r1)
        ok = ok and torch.equal(so[r0:r1], s[r0:r1]) and torch.equal(do[r0:r1], d[r0:r1])
        sp = f.sensitivity(xd, dcd, rows=r1)
        ok = ok and torch.equal(sp[:r1], s[:r1])
        if not ok:
            bad += 1
            print(f"MISMATCH case {case}: n {n} nnz {nnz} longest {int(lens.max())} range [{r0},{r1})", flush=True)
        f.close()
    print(f"apply soak: {cases} random CSR matrices, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
