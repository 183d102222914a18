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


def _halo_worker(rank, world, port, q):
    """NEXT-4 transport: every rank posts one send per peer and one receive per peer through
    DistTransport (batch_isend_irecv) over gloo, with the sharded filter's buffer layout
    ([x | dc] per peer, sizes differing per pair), then waits; received values are checked."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2012_08208_b200 import sharded

    dist.init_process_group("gloo", rank=rank, world_size=world)
    size = lambda a, b: 3 + 5 * a + 7 * b  # noqa: E731  points rank a sends to rank b
    val = lambda a, b, m: torch.arange(2 * m, dtype=torch.float64) + 1000.0 * a + 100.0 * b  # noqa: E731
    sends = {j: val(rank, j, size(rank, j)) for j in range(world) if j != rank}
    recvs = {j: torch.zeros(2 * size(j, rank), dtype=torch.float64) for j in range(world) if j != rank}
    sharded.DistTransport().exchange(sends, recvs).wait()
    ok = all(bool(torch.equal(recvs[j], val(j, rank, size(j, rank)))) for j in recvs)
    q.put((rank, ok, sum(t.numel() for t in recvs.values()), sorted(recvs)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, ok, nh, srcs in res:
        assert ok and nh > 0 and rank not in srcs
