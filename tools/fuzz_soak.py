"""Soak run of the seeded fuzz clouds (tests/test_gpu_fuzz.py::cloud) beyond the 24 seeds of the test
suite, through each fill kernel of the group path (TOPOFILT_CL_FILL=walk3 / split) and the default
rule: whole CSR bit-exact against the oracle. python tools/fuzz_soak.py [first_seed last_seed]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402
from test_gpu_fuzz import cloud  # noqa: E402


def main():
    a = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 264
    bad = 0
    for seed in range(a, b):
        c, rmin = cloud(seed)
        ref = oracle.build_celllist(c, rmin)
        cd = torch.from_numpy(c).cuda()
        for kern in ("", "walk3", "split"):
            os.environ["TOPOFILT_CL_FILL"] = kern
            f = tf.tf_build_filter(cd, rmin, path="cell_list")
            rowptr, cols, vals, hs = (t.cpu().numpy() for t in f.csr())
            ok = (np.array_equal(rowptr, ref.rowptr) and np.array_equal(cols, ref.cols) and
                  np.array_equal(vals, ref.vals) and np.allclose(hs, ref.hs, rtol=1e-12, atol=0))
            if not ok:
                bad += 1
                print(f"MISMATCH seed {seed} kernel '{kern}' n {c.shape[0]} dim {c.shape[1]} rmin {rmin} "
                      f"groups {f.stats()['groups']}", flush=True)
            f.close()
    print(f"fuzz soak: seeds [{a}, {b}) x 3 kernel choices, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
