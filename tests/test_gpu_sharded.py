"""NEXT-4 end to end on one GPU: W shards of one filter problem run as threads of one process,
each calling ShardedFilter.sensitivity / density (device plan, local build, tf_halo_pack, the
exchange through LoopbackTransport, interior rows then boundary rows with tf_*_filter_range); the
assembled owned rows equal the unsharded filter and the oracle to 1e-10 (only the summation order
differs). The NCCL transport (DistTransport) is the same interface; the gloo test in
tests/test_multirank.py exercises it across processes."""
import threading

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL = 1e-10


@pytest.fixture(scope="module")
def tf():
    assert torch.cuda.is_available()
    import paper_2012_08208_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def assert_rel(g, r, what):
    scale = np.where(r != 0, np.abs(r), np.abs(r).max())
    bad = np.abs(g - r) > RTOL * scale
    assert not bad.any(), f"{what}: {bad.sum()} of {r.size} outside {RTOL}"


def run_shards(c, rmin, x, dc, world, iters=2):
    """Every shard in its own thread (own CUDA stream); returns the assembled global outputs."""
    from paper_2012_08208_b200 import sharded
    hub = sharded.LoopbackTransport(world)
    cd = dev(c)
    sens, dens = np.full_like(x, np.nan), np.full_like(x, np.nan)
    errs = []
    stats = {}

    def work(k):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                sf = sharded.ShardedFilter(cd, rmin, k, world, hub.endpoint(k))
                ids = sf.plan.owned_ids.long()
                xo, dco = dev(x)[ids], dev(dc)[ids]
                for _ in range(iters):  # repeated calls reuse the buffers
                    s = sf.sensitivity(xo, dco).clone()
                    d = sf.density(xo).clone()
                torch.cuda.current_stream().synchronize()
                idn = ids.cpu().numpy()
                sens[idn] = s.cpu().numpy()
                dens[idn] = d.cpu().numpy()
                stats[k] = (sf.plan.n_interior, sf.plan.n_owned, sf.plan.n_halo)
                sf.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            hub.barrier.abort()

    th = [threading.Thread(target=work, args=(k,)) for k in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return sens, dens, stats


@pytest.mark.parametrize("case,world", [("c2", 2), ("c3", 4), ("kuhn_jitter", 3), ("random", 8),
                                        ("ground", 2), ("c3", 13)])
def test_sharded_equals_unsharded_and_oracle(tf, case, world):
    if case == "kuhn_jitter":
        c = synth.kuhn_mesh(12, 8, 6, jitter=0.15, stream=77)[0]
        rmin = 1.5
    elif case == "random":
        c = synth.random_points(909, 30000, 3, 0.0, 30.0)
        rmin = 1.7
    elif case == "ground":
        c = synth.ground_structure(4, 400, 300)[0]
        rmin = 3.0
    else:
        c, _, _, rmin = synth.workload(int(case[1]))
    n = c.shape[0]
    x = synth.uniform(910, 0, n, 0.001, 1.0)
    dc = -synth.uniform(911, 0, n, 0.5, 1.5) * x * x
    sens, dens, stats = run_shards(c, rmin, x, dc, world)
    assert sum(v[1] for v in stats.values()) == n
    assert any(v[0] < v[1] for v in stats.values()) or world == 1  # boundary rows exist
    f = tf.tf_build_filter(dev(c), rmin)
    assert_rel(sens, f.sensitivity(dev(x), dev(dc)).cpu().numpy(), f"{case}/{world} vs unsharded sensitivity")
    assert_rel(dens, f.density(dev(x)).cpu().numpy(), f"{case}/{world} vs unsharded density")
    f.close()
    if n <= 200_000:
        ref = oracle.build_celllist(c, rmin)
        assert_rel(sens, oracle.apply_sensitivity(ref, x, dc), f"{case}/{world} vs oracle sensitivity")
        assert_rel(dens, oracle.apply_density(ref, x), f"{case}/{world} vs oracle density")


def test_filter_range_matches_full(tf):
    """tf_*_filter_range: rows [r0, r1) bitwise the full call's, for ranges starting inside a row
    block, empty ranges and the whole range."""
    c = synth.random_points(912, 50000, 3, 0.0, 40.0)
    rmin = 1.6
    n = c.shape[0]
    f = tf.tf_build_filter(dev(c), rmin)
    x, dc = dev(synth.uniform(913, 0, n, 0.001, 1.0)), dev(-synth.uniform(914, 0, n, 0.0, 1.0))
    full_s, full_d = f.sensitivity(x, dc), f.density(x)
    for r0, r1 in [(0, n), (1234, 1234), (1, 17), (777, 40001), (n - 5, n)]:
        out_s, out_d = torch.full_like(x, float("nan")), torch.full_like(x, float("nan"))
        tf.tf_sensitivity_filter_range(f, x, dc, out_s, r0, r1)
        tf.tf_density_filter_range(f, x, out_d, r0, r1)
        assert torch.equal(out_s[r0:r1], full_s[r0:r1]) and torch.equal(out_d[r0:r1], full_d[r0:r1])
    with pytest.raises(tf.TopofiltError):
        tf.tf_density_filter_range(f, x, torch.empty_like(x), 5, 3)
    f.close()


def test_sharded_empty_ranks(tf):
    """More shards than distinct cut coordinates: some ranks own nothing (no local filter) but
    still take part in the exchange; the assembled result is still the oracle's."""
    rng = np.random.default_rng(21)
    n = 3000
    c = np.stack([rng.integers(0, 3, n).astype(np.float64) * 0.9, rng.uniform(0, 1.0, n) * 0.5], 1)
    rmin = 1.0
    x = synth.uniform(915, 0, n, 0.001, 1.0)
    dc = -synth.uniform(916, 0, n, 0.5, 1.5)
    sens, dens, stats = run_shards(c, rmin, x, dc, 5)
    assert sum(v[1] for v in stats.values()) == n
    assert any(v[1] == 0 for v in stats.values())
    ref = oracle.build_celllist(c, rmin)
    assert_rel(sens, oracle.apply_sensitivity(ref, x, dc), "empty ranks sensitivity")
    assert_rel(dens, oracle.apply_density(ref, x), "empty ranks density")
