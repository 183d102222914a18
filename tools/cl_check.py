"""Quick check of the group cell-list build against the per-bin kernels (bitwise CSR) and its
timing: python tools/cl_check.py [cfg ...] (default 4 5). One JSON line per config."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_08208_b200 as tf  # noqa: E402
import synth  # noqa: E402


def timed(cd, rmin, path, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        f = tf.tf_build_filter(cd, rmin, path=path)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        f.close()
    return float(np.median(ts)), ts


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [4, 5]
    for cfg in cfgs:
        c, _, _, rmin = synth.workload(cfg)
        cd = torch.from_numpy(c).cuda()
        n, dim = c.shape
        fg = tf.tf_build_filter(cd, rmin, path="cell_list")
        st = fg.stats()
        fb = tf.tf_build_filter(cd, rmin, path="cell_list_bins")
        same = all(torch.equal(a, b) for a, b in zip(fg.csr()[:3], fb.csr()[:3]))
        hsd = float((fg.csr()[3] - fb.csr()[3]).abs().max() / fb.csr()[3].abs().max())
        nnz = fg.nnz
        fg.close()
        fb.close()
        mg, tg = timed(cd, rmin, "cell_list")
        mb, tb = timed(cd, rmin, "cell_list_bins")
        byt = 8 * dim * n + 12 * nnz + 8 * (n + 1) + 8 * n
        print(json.dumps({"config": cfg, "n": n, "nnz": nnz, "bitwise_equal": same, "hs_rel": hsd,
                          "groups": st["groups"], "max_union": st["max_candidates"],
                          "groups_ms": round(mg, 4), "bins_ms": round(mb, 4), "speedup": round(mb / mg, 3),
                          "groups_frac_8tbs": byt / (mg * 1e-3) / 8e12,
                          "all_groups_ms": [round(t, 3) for t in tg]}), flush=True)


if __name__ == "__main__":
    main()
