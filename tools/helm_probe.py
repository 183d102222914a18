"""Helmholtz solve cost split on the config-5 mesh: time at maxit = 1, 2, K (cold L2) ->
per-iteration cost (slope) and the fixed phases (projection, initial residual, nodal mean).
Usage: python tools/helm_probe.py [ncu]  (ncu: one solve only, for a profiler capture)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402
from tools.bench_configs import timed  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    nodes, cells = synth.kuhn_mesh(200, 100, 100)
    n = cells.shape[0]
    h = tf.tf_helmholtz_build(torch.from_numpy(nodes).to(dev), torch.from_numpy(cells).to(dev),
                              tf.helmholtz_radius(1.5))
    x = torch.from_numpy(synth.density(5, n)).to(dev)
    dc = torch.from_numpy(synth.sensitivity(5, synth.density(5, n))).to(dev)
    out = torch.empty_like(x)
    info = h._info(dev)
    if len(sys.argv) > 1 and sys.argv[1] == "ncu":
        h.sensitivity(x, dc, out=out, info=info)
        torch.cuda.synchronize()
        return
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    res = {}
    for k in (1, 2, 19):
        h.sensitivity(x, dc, out=out, info=info, rtol=1e-30, maxit=k)
        res[k] = timed(lambda: h.sensitivity(x, dc, out=out, info=info, rtol=1e-30, maxit=k), 10, flush=flush)
        print(f"maxit {k}: {res[k] * 1e6:.1f} us ({h.decode_info(info)['iterations']} iterations)")
    per = (res[19] - res[1]) / 18
    print(f"per iteration {per * 1e6:.1f} us; fixed phases {(res[1] - per) * 1e6:.1f} us")


if __name__ == "__main__":
    main()
