"""Soak run of the Helmholtz PDE filter (NEXT-3) on random jittered triangle and tetrahedron meshes with
random radii, against the oracle (oracle/helmholtz.py: scipy assembly + sparse direct solve): system
pattern exact, A / M / node weights / volumes within 1e-13, filtered fields within 1e-9 of max|s~|.
python tools/helmholtz_soak.py [cases]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import helmholtz as hz  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402
import synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(31337)
    bad = 0
    for case in range(cases):
        if case % 2 == 0:
            nx, ny = int(rng.integers(1, 50)), int(rng.integers(1, 40))
            nodes, cells = synth.tri_mesh(nx, ny, str(rng.choice(["right", "left", "right/left"])),
                                          jitter=float(rng.uniform(0, 0.3)), stream=500 + case)
            name = f"tri {nx}x{ny}"
        else:
            nx, ny, nz = int(rng.integers(1, 16)), int(rng.integers(1, 12)), int(rng.integers(1, 10))
            nodes, cells = synth.kuhn_mesh(nx, ny, nz, jitter=float(rng.uniform(0, 0.25)), stream=500 + case)
            name = f"kuhn {nx}x{ny}x{nz}"
        R = float(rng.choice([0.0, 0.1, 0.433, 0.9, 2.5, 7.0]))
        sigma = rng.uniform(-1.0, 1.0, cells.shape[0])
        A, M, W, vol = hz.system(nodes, cells, R)
        ref, _ = hz.helmholtz_filter(nodes, cells, R, sigma)
        h = tf.tf_helmholtz_build(dev(nodes), dev(cells), R)
        rowptr, cols, vA, vM, Wg, volg = (t.cpu().numpy() for t in h.system())
        ok = np.array_equal(rowptr, A.indptr) and np.array_equal(cols, A.indices)
        ok = ok and np.allclose(vA, A.data, rtol=1e-13, atol=1e-13 * np.abs(A.data).max())
        ok = ok and np.allclose(vM, M.data, rtol=1e-13, atol=1e-13 * np.abs(M.data).max())
        ok = ok and np.allclose(Wg, W, rtol=1e-13) and np.allclose(volg, vol, rtol=1e-13)
        out, info = h.filter(dev(sigma), rtol=1e-12)
        inf = h.decode_info(info)
        err = float(np.abs(out.cpu().numpy() - ref).max())
        ok = ok and inf["converged"] and err <= 1e-9 * max(1.0, float(np.abs(ref).max()))
        if not ok:
            bad += 1
            print(f"MISMATCH case {case}: {name} cells {cells.shape[0]} R {R} err {err:.3e} info {inf}", flush=True)
        h.close()
    print(f"helmholtz soak: {cases} cases, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
