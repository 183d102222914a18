"""Time tf_build_filter on each build path (lattice vs cell list) for the lattice configs.

python tools/build_paths.py [cfg ...]   (default: 1 2 3 5) -> one JSON line per (config, path):
median build ms over 5 repetitions (CUDA events on the build stream, after one warm-up),
nnz/s and the fraction of 8 TB/s on the build's algorithmic bytes.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_08208_b200 as tf  # noqa: E402
import synth  # noqa: E402


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5]
    for cfg in cfgs:
        c, _, _, rmin = synth.workload(cfg)
        cd = torch.from_numpy(c).cuda()
        n, dim = c.shape
        for path in os.environ.get("BUILD_PATHS", "lattice,cell_list").split(","):
            try:
                f = tf.tf_build_filter(cd, rmin, path=path)
            except tf.TopofiltError as e:  # e.g. the lattice path asked for on a non-lattice cloud
                print(json.dumps({"config": cfg, "path": path, "skipped": str(e)[:120]}), flush=True)
                continue
            nnz, got = f.nnz, f.stats()["path"]
            f.close()
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                f = tf.tf_build_filter(cd, rmin, path=path)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
                f.close()
            ms = float(np.median(ts))
            byt = 8 * dim * n + 12 * nnz + 8 * (n + 1) + 8 * n
            print(json.dumps({"config": cfg, "path": got, "n": n, "nnz": nnz, "build_ms": round(ms, 4),
                              "nnz_per_s": nnz / (ms * 1e-3), "gbps": byt / (ms * 1e-3) / 1e9,
                              "frac_8tbs": byt / (ms * 1e-3) / 8e12, "all_ms": [round(t, 4) for t in ts]}),
                  flush=True)


if __name__ == "__main__":
    main()
