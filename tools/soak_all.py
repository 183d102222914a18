"""Soak run across the library on random inputs (beyond the fixed cases of the test suite), each checked
against the oracle: (a) applies on random clouds -- sensitivity, density, both-in-one-pass (bitwise the
separate calls), row ranges, the host-buffer pipeline; (b) the matrix-free stencil and periodic-lattice
filters on random grids; (c) the OC update (bitwise); (d) the sharded filter with random shard counts.
python tools/soak_all.py [cases]."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402
import synth  # noqa: E402
from test_gpu_fuzz import cloud  # noqa: E402

BAD = []


def rel_ok(g, r, tol=1e-10):
    scale = np.where(r != 0, np.abs(r), np.abs(r).max() if r.size else 1.0)
    return bool(np.all(np.abs(g - r) <= tol * scale))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(ok, what):
    if not ok:
        BAD.append(what)
        print("MISMATCH", what, flush=True)


def soak_applies(seed, rng):
    c, rmin = cloud(1000 + seed)
    n = c.shape[0]
    ref = oracle.build_celllist(c, rmin)
    x = rng.uniform(0.001, 1.0, n)
    dc = -rng.uniform(0.0, 1.0, n) * (1.0 if seed % 3 else 3.0 * x * x)
    rs, rd = oracle.apply_sensitivity(ref, x, dc), oracle.apply_density(ref, x)
    f = tf.tf_build_filter(dev(c), rmin)
    xd, dcd = dev(x), dev(dc)
    s, d = f.sensitivity(xd, dcd), f.density(xd)
    check(rel_ok(s.cpu().numpy(), rs) and rel_ok(d.cpu().numpy(), rd), f"applies seed {seed}")
    sb, db = f.both(xd, dcd)
    check(torch.equal(sb, s) and torch.equal(db, d), f"both seed {seed}")
    r0, r1 = sorted(int(v) for v in rng.integers(0, n + 1, 2))
    so, do = torch.full_like(xd, 7.0), torch.full_like(xd, 7.0)
    tf.tf_sensitivity_filter_range(f, xd, dcd, so, r0, r1)
    tf.tf_density_filter_range(f, xd, do, r0, r1)
    check(torch.equal(so[r0:r1], s[r0:r1]) and torch.equal(do[r0:r1], d[r0:r1]), f"range [{r0},{r1}) seed {seed}")
    if seed % 4 == 0:
        hs_, hd_ = tf.tf_filter_iteration_host(f, x, dc)
        check(np.array_equal(np.asarray(hs_), s.cpu().numpy()) and np.array_equal(np.asarray(hd_), d.cpu().numpy()),
              f"host pipeline seed {seed}")
    f.close()


def soak_matrix_free(seed, rng):
    dim = int(rng.integers(2, 4))
    nx, ny = int(rng.integers(1, 40)), int(rng.integers(1, 25))
    nz = int(rng.integers(1, 12)) if dim == 3 else 1
    h = float(rng.choice([1.0, 0.5, 2.0, 0.75]))
    rmin = float(rng.uniform(0.6, 3.4)) * h
    T = int(rng.choice([1, 1, 2, 3, 6]))
    off = np.full((1, dim), 0.5) if T == 1 else rng.integers(0, 8, size=(T, dim)) / 8.0
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cube = np.stack([i.ravel(), j.ravel(), k.ravel()], 1)[:, :dim].astype(np.float64)
    c = np.ascontiguousarray(((cube[:, None, :] + off[None, :, :]) * h).reshape(-1, dim))
    n = c.shape[0]
    ref = oracle.build_bruteforce(c, rmin) if n <= 20000 else oracle.build_celllist(c, rmin)
    x = rng.uniform(0.001, 1.0, n)
    dc = -rng.uniform(0.0, 1.0, n)
    try:
        f = tf.tf_build_stencil(dim, nx, ny, nz, h, rmin) if (T == 1 and seed % 2 == 0) else \
            tf.tf_build_lattice(dim, nx, ny, nz, h, off, rmin)
    except tf.TopofiltError as e:
        if "too large" in str(e):  # documented refusal (reach / types beyond the shared-memory tile)
            return
        raise
    s, d = f.sensitivity(dev(x), dev(dc)).cpu().numpy(), f.density(dev(x)).cpu().numpy()
    check(f.nnz == ref.nnz and rel_ok(s, oracle.apply_sensitivity(ref, x, dc)) and rel_ok(d, oracle.apply_density(ref, x)),
          f"matrix-free seed {seed}: dim {dim} grid {nx}x{ny}x{nz} T {T} h {h} rmin {rmin:.3f}")
    f.close()


def soak_oc(seed, rng):
    n = int(rng.integers(1, 300000))
    x = rng.uniform(0.001, 1.0, n)
    dc = -rng.uniform(0.0, 10.0 ** rng.uniform(-6, 3), n)
    vf = float(rng.uniform(0.05, 0.95))
    move = float(rng.choice([0.2, 0.05, 0.5]))
    ro, lo, io = oracle.oc_update(x, dc, vf, move=move)
    g, lm, it = tf.tf_oc_update(dev(x), dev(dc), vf, move=move)
    check(np.array_equal(g.cpu().numpy(), ro) and float(lm[0]) == lo and int(it[0]) == io, f"oc seed {seed} n {n}")


def soak_sharded(seed, rng):
    from paper_2012_08208_b200 import sharded
    c, rmin = cloud(2000 + seed)
    n = c.shape[0]
    world = int(rng.integers(2, 9))
    x = rng.uniform(0.001, 1.0, n)
    dc = -rng.uniform(0.0, 1.0, n)
    ref = oracle.build_celllist(c, rmin)
    hub = sharded.LoopbackTransport(world)
    cd = dev(c)
    sens, dens = np.full_like(x, np.nan), np.full_like(x, np.nan)
    errs = []

    def work(k):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                sf = sharded.ShardedFilter(cd, rmin, k, world, hub.endpoint(k))
                ids = sf.plan.owned_ids.long()
                s = sf.sensitivity(dev(x)[ids], dev(dc)[ids]).clone()
                d = sf.density(dev(x)[ids]).clone()
                torch.cuda.current_stream().synchronize()
                idn = ids.cpu().numpy()
                sens[idn], dens[idn] = s.cpu().numpy(), d.cpu().numpy()
                sf.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            hub.barrier.abort()

    th = [threading.Thread(target=work, args=(k,)) for k in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        check(False, f"sharded seed {seed} world {world}: {errs[0]!r}")
        return
    check(rel_ok(sens, oracle.apply_sensitivity(ref, x, dc)) and rel_ok(dens, oracle.apply_density(ref, x)),
          f"sharded seed {seed} world {world}")


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(777)
    if len(sys.argv) > 2 and sys.argv[2] == "sharded":  # sharded runs only
        for seed in range(cases):
            soak_sharded(5000 + seed, rng)
        print(f"soak: {cases} sharded runs, {len(BAD)} mismatches")
        sys.exit(1 if BAD else 0)
    for seed in range(cases):
        soak_applies(seed, rng)
        soak_matrix_free(seed, rng)
        soak_matrix_free(10000 + seed, rng)
        soak_oc(seed, rng)
        if seed % 3 == 0:
            soak_sharded(seed, rng)
    print(f"soak: {cases} rounds (applies, both, ranges, host pipeline, matrix-free x2, OC, sharded every 3rd), "
          f"{len(BAD)} mismatches")
    sys.exit(1 if BAD else 0)


if __name__ == "__main__":
    main()
