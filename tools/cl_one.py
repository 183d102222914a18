"""One cell-list build of config N (default 5) through the group kernels, for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2012_08208_b200 as tf  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
path = sys.argv[2] if len(sys.argv) > 2 else "cell_list"
c, _, _, rmin = synth.workload(cfg)
f = tf.tf_build_filter(torch.from_numpy(c).cuda(), rmin, path=path)
torch.cuda.synchronize()
print(cfg, path, f.nnz, f.stats())
