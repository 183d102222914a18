"""Mid-size apply probe (configs 3 and 4): cold CUDA-event times of the sensitivity and density
applies (median of 9, L2 flushed), plus the same calls back to back for an ncu capture
(`python tools/apply_mid_probe.py ncu`)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2012_08208_b200 as tf  # noqa: E402
import synth  # noqa: E402
from tools.bench_configs import timed  # noqa: E402


def main():
    ncu = len(sys.argv) > 1 and sys.argv[1] == "ncu"
    dev = torch.device("cuda:0")
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    for cfg in (3, 4):
        c, x, dc, rmin = synth.workload(cfg)
        n = c.shape[0]
        f = tf.tf_build_filter(torch.from_numpy(c).to(dev), rmin)
        xd, dcd = torch.from_numpy(x).to(dev), torch.from_numpy(dc).to(dev)
        out = torch.empty_like(xd)
        if ncu:
            for _ in range(2):
                flush.add_(1.0)
                f.sensitivity(xd, dcd, out=out)
                flush.add_(1.0)
                f.density(xd, out=out)
            torch.cuda.synchronize()
            continue
        s = timed(lambda: f.sensitivity(xd, dcd, out=out), 9, flush)
        d = timed(lambda: f.density(xd, out=out), 9, flush)
        nnz = f.nnz
        sb = 12 * nnz + 8 * (n + 1) + 32 * n
        db = 12 * nnz + 8 * (n + 1) + 24 * n
        print(json.dumps({"config": cfg, "sens_us": s * 1e6, "dens_us": d * 1e6,
                          "sens_frac_8tbs": sb / s / 8e12, "dens_frac_8tbs": db / d / 8e12,
                          "plan": {"group": None}}), flush=True)
        f.close()


if __name__ == "__main__":
    main()
