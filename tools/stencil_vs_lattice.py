"""Regular-grid stencil (k_stencil) vs the lattice kernel with one type at offset 1/2 (k_lattice),
configs 1 and 3, cold L2: which matrix-free kernel to use for single-type grids."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402
from tools.bench_configs import timed  # noqa: E402

flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
for cfg, (dim, nx, ny, nz) in ((1, (2, 60, 20, 1)), (3, (3, 160, 80, 80))):
    c, x, dc, rmin = synth.workload(cfg)
    xd, dd = torch.from_numpy(x).cuda(), torch.from_numpy(dc).cuda()
    out = torch.empty_like(xd)
    fs = tf.tf_build_stencil(dim, nx, ny, nz, 1.0, rmin)
    fl = tf.tf_build_lattice(dim, nx, ny, nz, 1.0, np.full((1, dim), 0.5), rmin)
    a = fs.sensitivity(xd, dd).cpu().numpy()
    b = fl.sensitivity(xd, dd).cpu().numpy()
    rel = float(np.max(np.abs(a - b) / np.abs(a)))
    for name, f in (("stencil", fs), ("lattice", fl)):
        f.sensitivity(xd, dd, out=out)
        ts = timed(lambda: f.sensitivity(xd, dd, out=out), 20, flush=flush)
        td = timed(lambda: f.density(xd, out=out), 20, flush=flush)
        print(f"config {cfg} {name}: sensitivity {ts * 1e6:.1f} us, density {td * 1e6:.1f} us (max rel diff {rel:.1e})")
