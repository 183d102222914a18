"""One lattice sensitivity apply on config 5 (for an ncu capture of k_lattice)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402

c, x, dc, rmin = synth.workload(5)
xd, dd = torch.from_numpy(x).cuda(), torch.from_numpy(dc).cuda()
f = tf.tf_build_lattice(3, 200, 100, 100, 1.0, synth.kuhn_lattice_offsets(), rmin)
o = torch.empty_like(xd)
f.sensitivity(xd, dd, out=o)
torch.cuda.synchronize()
print("ok")
