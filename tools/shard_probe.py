"""NEXT-4 projection on one GPU: config 5 cut into W slabs by the device plan (tf_shard_plan);
for the middle rank of each W, the local filter (owned + halo rows) is built with the library
and its owned-row applies (interior rows + boundary rows, tf_*_filter_range, as ShardedFilter
runs them; all local rows beside) are timed (CUDA events, cold L2), next to the halo it receives
per apply and the unsharded filter's applies. The exchange is not run here (one GPU); its time is projected at
the measured NVLink peer-copy rate of B200_PROFILING.md (770 GB/s per direction), so the
printed per-iteration times are projections, labelled as such.
Usage: python tools/shard_probe.py [W ...]   (default 2 4 8; one JSON line per W)"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402
from paper_2012_08208_b200 import sharded  # noqa: E402
from tools.bench_configs import timed  # noqa: E402

PEER_GBS = 770.0  # measured NVLink peer copy per direction (B200_PROFILING.md)


def main():
    worlds = [int(a) for a in sys.argv[1:]] or [2, 4, 8]
    dev = torch.device("cuda:0")
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    c, x, dc, rmin = synth.workload(5)
    n = c.shape[0]
    f = tf.tf_build_filter(torch.from_numpy(c).to(dev), rmin)
    xd, dcd = torch.from_numpy(x).to(dev), torch.from_numpy(dc).to(dev)
    out = torch.empty_like(xd)
    full_s = timed(lambda: f.sensitivity(xd, dcd, out=out), 5, flush)
    full_d = timed(lambda: f.density(xd, out=out), 5, flush)
    f.close()
    print(json.dumps({"world": 1, "n": n, "sens_us": full_s * 1e6, "dens_us": full_d * 1e6}), flush=True)
    for world in worlds:
        rank = world // 2  # a middle slab: halo on both faces
        cdev = torch.from_numpy(c).to(dev)
        p = sharded.ShardPlan(cdev, rmin, world, rank)
        loc = p.local_ids.long().cpu().numpy()
        lf = tf.tf_build_filter(torch.from_numpy(np.ascontiguousarray(c[loc])).to(dev), rmin)
        xl, dcl = torch.from_numpy(x[loc]).to(dev), torch.from_numpy(dc[loc]).to(dev)
        ol = torch.empty_like(xl)
        ls_all = timed(lambda: lf.sensitivity(xl, dcl, out=ol), 5, flush)
        ld_all = timed(lambda: lf.density(xl, out=ol), 5, flush)

        def sens_split():
            tf.tf_sensitivity_filter_range(lf, xl, dcl, ol, 0, p.n_interior)
            tf.tf_sensitivity_filter_range(lf, xl, dcl, ol, p.n_interior, p.n_owned)

        def dens_split():
            tf.tf_density_filter_range(lf, xl, ol, 0, p.n_interior)
            tf.tf_density_filter_range(lf, xl, ol, p.n_interior, p.n_owned)
        ls = timed(sens_split, 5, flush)  # owned rows, interior then boundary (two launches)
        ld = timed(dens_split, 5, flush)
        sent = int(sum(p.send))
        halo_bytes_sens = 16 * max(p.n_halo, sent)  # x and dc, the larger direction
        xch = halo_bytes_sens / (PEER_GBS * 1e9)
        proj_iter = ls + ld + 2 * xch
        print(json.dumps({
            "world": world, "rank": rank, "n_owned": p.n_owned, "n_interior": p.n_interior, "n_halo": p.n_halo,
            "halo_frac": p.n_halo / p.n_owned,
            "local_nnz": lf.nnz, "sens_us": ls * 1e6, "dens_us": ld * 1e6,
            "sens_us_all_local_rows": ls_all * 1e6, "dens_us_all_local_rows": ld_all * 1e6,
            "halo_mb_per_sens_apply": halo_bytes_sens / 1e6,
            "exchange_us_projected": xch * 1e6,
            "iteration_us_projected": proj_iter * 1e6,
            "speedup_projected_vs_1gpu": (full_s + full_d) / proj_iter,
            "note": "local applies measured on one B200 (interior + boundary launches); exchange projected at "
                    "770 GB/s and not credited with the overlap the interior rows give it",
        }), flush=True)
        lf.close()
        p.close()


if __name__ == "__main__":
    main()
