"""The apply calls are stream-ordered and capture-safe: a CUDA graph of a whole filter
iteration (sensitivity + density, incl. the cooperative launch and its stream-ordered
scratch) replays with the same results -- how launch-bound small problems should be run."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", [1, 2])
def test_graph_capture_replay(cfg):
    import paper_2012_08208_b200 as tf
    c, x, dc, rmin = synth.workload(cfg)
    dev = torch.device("cuda")
    f = tf.tf_build_filter(torch.from_numpy(c).to(dev), rmin)
    xs, dcs = torch.from_numpy(x).to(dev), torch.from_numpy(dc).to(dev)
    s_ref = f.sensitivity(xs, dcs).clone()
    d_ref = f.density(xs).clone()
    os_, od = torch.empty_like(xs), torch.empty_like(xs)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):  # warm-up on the capture stream (attributes, occupancy queries)
        f.sensitivity(xs, dcs, out=os_)
        f.density(xs, out=od)
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f.sensitivity(xs, dcs, out=os_)
        f.density(xs, out=od)
    for _ in range(5):
        os_.zero_()
        od.zero_()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(os_, s_ref) and torch.equal(od, d_ref)
