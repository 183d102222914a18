"""Concurrent applies on ONE handle from several host threads (each on its own stream, distinct outputs;
include/topofilt.h: the handle is immutable after build): sensitivity, density, both-in-one-pass, row
ranges and the matrix-free handles, results bitwise those of the same calls made alone.
python tools/thread_soak.py [rounds]."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_08208_b200 as tf  # noqa: E402
import synth  # noqa: E402


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    bad = []
    handles = [
        ("c3 hex (lattice build)", tf.tf_build_filter(torch.from_numpy(synth.workload(3)[0]).cuda(), 2.0)),
        ("jittered 600x300 (cell list)", tf.tf_build_filter(torch.from_numpy(
            np.ascontiguousarray(synth.ground_structure(4, 600, 300)[0])).cuda(), 3.0)),
        ("stencil 60x40x30", tf.tf_build_stencil(3, 60, 40, 30, 1.0, 2.0)),
    ]
    for name, f in handles:
        n = f.n
        T = 8
        xs = [torch.from_numpy(synth.uniform(900 + k, 0, n, 0.001, 1.0)).cuda() for k in range(T)]
        dcs = [-torch.from_numpy(synth.uniform(950 + k, 0, n, 0.0, 1.0)).cuda() for k in range(T)]
        alone = []
        for k in range(T):
            s, d = f.sensitivity(xs[k], dcs[k]).clone(), f.density(xs[k]).clone()
            alone.append((s, d))
        torch.cuda.synchronize()
        for rnd in range(rounds):
            start = threading.Barrier(T)

            def work(k):
                try:
                    with torch.cuda.stream(torch.cuda.Stream()):
                        start.wait()
                        for it in range(5):
                            s, d = f.sensitivity(xs[k], dcs[k]), f.density(xs[k])
                            if name.startswith("stencil") or it % 2:
                                sb, db = s, d
                            else:
                                sb, db = f.both(xs[k], dcs[k])
                            torch.cuda.current_stream().synchronize()
                            if not (torch.equal(s, alone[k][0]) and torch.equal(d, alone[k][1]) and
                                    torch.equal(sb, alone[k][0]) and torch.equal(db, alone[k][1])):
                                bad.append((name, rnd, k, it))
                except BaseException as e:  # noqa: BLE001
                    bad.append((name, rnd, k, repr(e)))
                    start.abort()

            th = [threading.Thread(target=work, args=(k,)) for k in range(T)]
            for t in th:
                t.start()
            for t in th:
                t.join()
        f.close()
    print(f"thread soak: {len(handles)} handles x {rounds} rounds x 8 threads x 5 iterations, {len(bad)} problems")
    for b in bad[:10]:
        print("  ", b)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
