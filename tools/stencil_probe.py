"""Run the config-3 stencil applies a few times (ncu target)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402

c, x, dc, rmin = synth.workload(3)
xd, dcd = torch.from_numpy(x).cuda(), torch.from_numpy(dc).cuda()
f = tf.tf_build_stencil(3, 160, 80, 80, 1.0, rmin)
for _ in range(4):
    f.sensitivity(xd, dcd)
    f.density(xd)
torch.cuda.synchronize()
print("ok")
