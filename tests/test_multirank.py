"""World-size-2 gloo tests (CPU) of bench.py's multi-rank host logic: rank/world handling,
max-over-ranks timing, whole-job aggregation and rank-0-only output (DESIGN.md §7:
replicas only -- every rank runs an independent replica, no data-path collective)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    import numpy as np

    import oracle
    import synth

    dist = bench.init_dist("gloo")
    ws, r, _ = bench.dist_env()
    # each replica does the same (CPU) filter work on the same seeded inputs
    c = synth.quad_grid(20, 10)
    H = oracle.build_celllist(c, 1.5)
    x = synth.density(2, c.shape[0])
    out = oracle.apply_density(H, x)
    local_time = 1.0 + rank  # rank 1 is the slow one
    t = bench.reduce_max(local_time, dist, device="cpu")
    val = bench.aggregate(100.0, ws, t)
    q.put((r, ws, t, val, float(out.sum())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_reduce_and_aggregate():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res.sort()
    (r0, w0, t0, v0, s0), (r1, w1, t1, v1, s1) = res
    assert (r0, r1) == (0, 1) and w0 == w1 == 2
    assert t0 == t1 == 2.0  # max over ranks
    assert v0 == v1 == 100.0 * 2 / 2.0  # all ranks' units / slowest time
    assert s0 == s1  # replicas compute identical results


def test_reference_arm_rank_gating(tmp_path):
    """`bench.py --impl reference` under a 2-rank launch: rank 0 prints one JSON line, the
    other rank exits 0 without work."""
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "1", "--warmup", "0", "--cpu-rows", "200"], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == ""
    env["RANK"] = "0"
    env["LOCAL_RANK"] = "0"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "1", "--warmup", "0", "--cpu-rows", "200"], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
