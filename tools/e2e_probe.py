"""Probe the host-buffer path on config 5: raw pinned H2D/D2H bandwidth and the wall time of
tf_filter_iteration_host (library from TOPOFILT_LIB, default the in-tree one).
Usage: python tools/e2e_probe.py [iterations]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2012_08208_b200 as tf  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    c, x, dc, rmin = synth.workload(5)
    n = x.shape[0]
    pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
    xp, dcp = pin(x), pin(dc)
    os_, od = torch.empty(n, dtype=torch.float64).pin_memory(), torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for name, fn in [("h2d", lambda: d.copy_(xp, non_blocking=True)), ("d2h", lambda: os_.copy_(d, non_blocking=True))]:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(iters):
            fn()
        torch.cuda.synchronize()
        t = (time.perf_counter() - t0) / iters
        print(f"{name}: {8 * n / t / 1e9:.1f} GB/s ({t * 1e3:.2f} ms per {8 * n / 1e6:.0f} MB)")
    # both directions at once on two streams (the pipeline's upload and download overlap)
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")
    su, sd = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        with torch.cuda.stream(su):
            d.copy_(xp, non_blocking=True)
        with torch.cuda.stream(sd):
            od.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / iters
    print(f"h2d+d2h concurrent: {8 * n / t / 1e9:.1f} GB/s each way ({t * 1e3:.2f} ms per {8 * n / 1e6:.0f} MB each)")
    f = tf.tf_build_filter_host(pin(c).numpy(), rmin)
    for _ in range(2):
        tf.tf_filter_iteration_host(f, xp.numpy(), dcp.numpy(), os_.numpy(), od.numpy())
    ts = []
    for _ in range(iters):
        t0 = time.perf_counter()
        tf.tf_filter_iteration_host(f, xp.numpy(), dcp.numpy(), os_.numpy(), od.numpy())
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"{os.environ.get('TOPOFILT_LIB', 'in-tree')}: iteration_host median {ts[len(ts) // 2] * 1e3:.2f} ms "
          f"min {ts[0] * 1e3:.2f} max {ts[-1] * 1e3:.2f}")
    f.close()



def step_probe(reps=4):
    """Whole e2e step as bench.py times it: build from host centroids, 20 iterations, free."""
    c, x, dc, rmin = synth.workload(5)
    n = x.shape[0]
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    cp, xp, dcp = pin(c), pin(x), pin(dc)
    os_, od = pin(x.copy()), pin(x.copy())
    for r in range(reps):
        t0 = time.perf_counter()
        f = tf.tf_build_filter_host(cp, rmin)
        t1 = time.perf_counter()
        tf.tf_filter_iteration_host(f, xp, dcp, os_, od)
        t2 = time.perf_counter()
        for _ in range(19):
            tf.tf_filter_iteration_host(f, xp, dcp, os_, od)
        t3 = time.perf_counter()
        f.close()
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        print(f"step {r}: build_host {1e3 * (t1 - t0):.1f} ms, first iteration {1e3 * (t2 - t1):.1f} ms, "
              f"19 more {1e3 * (t3 - t2):.1f} ms, close {1e3 * (t4 - t3):.1f} ms")



if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "step":
        step_probe()
    else:
        main()
