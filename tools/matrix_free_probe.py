"""One matrix-free sensitivity apply per variant (ncu capture of k_stencil / k_lattice):
config 3 regular-grid stencil and config 5 BoxMesh lattice."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402

for cfg in (3, 5):
    c, x, dc, rmin = synth.workload(cfg)
    xd, dd = torch.from_numpy(x).cuda(), torch.from_numpy(dc).cuda()
    f = (tf.tf_build_stencil(3, 160, 80, 80, 1.0, rmin) if cfg == 3 else
         tf.tf_build_lattice(3, 200, 100, 100, 1.0, synth.kuhn_lattice_offsets(), rmin))
    o = torch.empty_like(xd)
    f.sensitivity(xd, dd, out=o)
    torch.cuda.synchronize()
    f.close()
print("ok")
