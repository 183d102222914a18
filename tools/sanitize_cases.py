"""Small cases for compute-sanitizer runs (memcheck / racecheck / synccheck / initcheck):
configs 1 and 2, random clouds of awkward sizes, duplicates, a one-bin dense case that takes
the large-neighbourhood + row-sort path, and both applies (incl. the cooperative launch)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402

cases = [
    (synth.centroids(1), 1.5),
    (synth.tri_grid(60, 20, "right"), 2.5),
    (synth.random_points(11, 1, 3, 0, 1), 1.0),
    (synth.random_points(12, 2, 2, 0, 1), 1.0),
    (synth.random_points(13, 31, 3, 0, 3), 1.2),
    (synth.random_points(14, 33, 2, 0, 3), 1.2),
    (synth.random_points(15, 1000, 3, 0, 10), 1.3),
    (np.repeat(synth.random_points(16, 50, 3, 0, 3), 3, axis=0), 1.0),
    (synth.random_points(17, 3500, 2, 0, 1), 5.0),   # one bin, > shared-memory cap: row-sort path
    (synth.kuhn_tets(6, 4, 3), 1.5),
]
for c, rmin in cases:
    c = np.ascontiguousarray(c, dtype=np.float64)
    n = c.shape[0]
    f = tf.tf_build_filter(torch.from_numpy(c).cuda(), rmin)
    x = torch.from_numpy(synth.uniform(21, 0, n, 0.001, 1.0)).cuda()
    dc = torch.from_numpy(-synth.uniform(22, 0, n, 0.0, 1.0)).cuda()
    s = f.sensitivity(x, dc)
    d = f.density(x)
    torch.cuda.synchronize()
    assert torch.isfinite(s).all() and torch.isfinite(d).all()
    f.close()
print("sanitize cases OK")
