"""Concurrent use from several host threads: builds of different sizes and dimensions run at the same
time on different streams (the sharded filter does this with one thread per shard). The kernels'
dynamic shared-memory limit is a per-function, process-wide attribute; setting it per launch to the
exact size let one thread lower it under another thread's launch ("invalid argument", found by
tools/soak_all.py). Every build must succeed and match the oracle bit for bit."""
import threading

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_concurrent_builds_of_different_sizes():
    import paper_2012_08208_b200 as tf
    assert torch.cuda.is_available()
    cases = [
        (synth.ground_structure(4, 400, 200)[0], 3.0),                      # 2D, small unions (k_cl_fill4)
        (synth.random_points(7101, 6000, 2, 0.0, 40.0), 1.7),               # 2D, other sizes
        (synth.kuhn_mesh(10, 8, 6, jitter=0.1, stream=5)[0], 1.5),          # 3D (k_cl_fill3)
        (synth.random_points(7102, 9000, 3, 0.0, 14.0), 1.2),
        (synth.random_points(7103, 2500, 3, 0.0, 6.0), 0.9),
        (np.concatenate([synth.random_points(7104, 1200, 2, 0.0, 1.0),      # dense cluster: long rows, large smem
                         synth.random_points(7105, 800, 2, 0.0, 30.0)]), 0.8),
        (synth.hex_grid(14, 9, 7), 2.0),                                    # lattice path
        (synth.tri_grid(50, 30, "right/left"), 2.0),
    ]
    refs = [oracle.build_celllist(c, r) for c, r in cases]
    errs = []
    start = threading.Barrier(len(cases))

    def work(k):
        try:
            c, rmin = cases[k]
            with torch.cuda.stream(torch.cuda.Stream()):
                cd = torch.from_numpy(np.ascontiguousarray(c)).cuda()
                start.wait()
                for it in range(6):
                    f = tf.tf_build_filter(cd, rmin, path="auto" if it % 2 else "cell_list")
                    rowptr, cols, vals, _ = (t.cpu().numpy() for t in f.csr())
                    assert np.array_equal(rowptr, refs[k].rowptr), (k, it)
                    assert np.array_equal(cols, refs[k].cols), (k, it)
                    assert np.array_equal(vals, refs[k].vals), (k, it)
                    f.close()
        except BaseException as e:  # noqa: BLE001
            errs.append((k, e))
            start.abort()

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
