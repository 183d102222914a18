"""Ablation: the paper's all-pairs build (TF_BUILD_DENSE: every pair of midpoints visited, as its
Euclidean distance matrix does, PAPER.md:390-396 / 442-445) against the cell-list build on the same
B200: python tools/dense_probe.py -> one JSON line per input (median of 3 builds each, CUDA events).
Inputs: configs 1, 2 and 4-like jittered clouds of growing size (the all-pairs cost is O(n^2))."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_08208_b200 as tf  # noqa: E402
import synth  # noqa: E402


def timed(cd, rmin, path, reps=3):
    f = tf.tf_build_filter(cd, rmin, path=path)  # warm-up
    nnz = f.nnz
    f.close()
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
    return float(np.median(ts)), nnz


def main():
    cases = [("c1 quads 60x20", synth.workload(1)[0], 1.5), ("c2 triangles 300x100", synth.workload(2)[0], 2.5),
             ("paper 180x60 right/left triangles (PAPER.md:332)", synth.tri_grid(180, 60, "right/left"), 2.0),
             ("jittered 600x300 (config-4 recipe)", synth.ground_structure(4, 600, 300)[0], 3.0),
             ("jittered 800x400 (config-4 recipe)", synth.ground_structure(4, 800, 400)[0], 3.0),
             ("c3 hex 160x80x80", synth.workload(3)[0], 2.0)]
    for name, c, rmin in cases:
        cd = torch.from_numpy(np.ascontiguousarray(c)).cuda()
        n = c.shape[0]
        td, nnz = timed(cd, rmin, "dense", reps=3 if n < 500000 else 1)
        tc, _ = timed(cd, rmin, "cell_list")
        print(json.dumps({"input": name, "n": n, "nnz": nnz, "dense_ms": round(td, 3), "cell_list_ms": round(tc, 3),
                          "pairs_per_s_dense": 2.0 * n * n / (td * 1e-3), "speedup_cell_list": round(td / tc, 1),
                          "edm_bytes_fp64": 8.0 * n * n}), flush=True)


if __name__ == "__main__":
    main()
