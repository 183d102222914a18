"""NEXT-4 on the GPU: the slab-sharded filter (paper_2012_08208_b200/sharded.py) emulated with K
shards in one process on one GPU -- every shard builds its local filter with the library,
packs its boundary values with tf_halo_pack, receives its halo from the other shards' packed
buffers and applies the library filter; the assembled owned rows equal the unsharded filter
and the oracle to 1e-10 (only the summation order differs). The transport itself (NCCL/gloo
point-to-point) is exercised by tests/test_multirank.py."""
import ctypes

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


def emulate(tf, c, rmin, x, dc, world):
    from paper_2012_08208_b200 import sharded
    plans = sharded.make_plans(c, world, rmin)
    shards = [sharded.ShardedFilter(c, rmin, k, world, plan=plans[k]) for k in range(world)]
    xo = [dev(x[p.owned]) for p in plans]
    dco = [dev(dc[p.owned]) for p in plans]
    sens, dens = np.empty_like(x), np.empty_like(x)
    packs = [sh.pack(xo[k], dco[k]) for k, sh in enumerate(shards)]
    for k, sh in enumerate(shards):
        rec = {j: packs[j][k] for j in sh.plan.halo_from}
        sens[plans[k].owned] = sh.apply_with_halo(xo[k], dco[k], rec).cpu().numpy()
    packs = [sh.pack(xo[k]) for k, sh in enumerate(shards)]
    for k, sh in enumerate(shards):
        rec = {j: packs[j][k] for j in sh.plan.halo_from}
        dens[plans[k].owned] = sh.apply_with_halo(xo[k], None, rec, density=True).cpu().numpy()
    for sh in shards:
        sh.close()
    return sens, dens, plans


@pytest.mark.parametrize("case,world", [("c2", 2), ("c3", 4), ("kuhn", 3), ("random", 8), ("c3", 13)])
def test_sharded_equals_unsharded(tf, case, world):
    if case == "kuhn":
        c, rmin = synth.kuhn_tets(30, 20, 16), 1.5
        x = synth.uniform(910, 0, c.shape[0], 0.001, 1.0)
        dc = (-3.0 * (x * x)) * synth.uniform(911, 0, c.shape[0], 0.5, 1.5)
    elif case == "random":
        c, rmin = synth.random_points(912, 200_000, 3, 0.0, 40.0), 1.2
        x = synth.uniform(913, 0, c.shape[0], 0.001, 1.0)
        dc = -synth.uniform(914, 0, c.shape[0], 0.0, 1.0)
    else:
        c, x, dc, rmin = synth.workload(int(case[1]))
    sens, dens, plans = emulate(tf, c, rmin, x, dc, world)
    assert sum(p.n_halo for p in plans) > 0
    f = tf.tf_build_filter(dev(c), rmin)
    assert_rel(sens, f.sensitivity(dev(x), dev(dc)).cpu().numpy(), f"{case}/{world} sharded sensitivity")
    assert_rel(dens, f.density(dev(x)).cpu().numpy(), f"{case}/{world} sharded density")
    f.close()
    if case in ("c2", "kuhn"):
        H = oracle.build_celllist(c, rmin)
        assert_rel(sens, oracle.apply_sensitivity(H, x, dc), "oracle sensitivity")
        assert_rel(dens, oracle.apply_density(H, x), "oracle density")


def test_halo_pack(tf):
    src = synth.uniform(915, 0, 10_000, -1.0, 1.0)
    idx = np.asarray(synth.sample_rows(3, 10_000, 777), dtype=np.int32)
    d = torch.empty(idx.shape[0], dtype=torch.float64, device="cuda")
    s, i = dev(src), dev(idx)
    tf._check(tf.lib().tf_halo_pack(ctypes.c_void_p(s.data_ptr()), ctypes.c_void_p(i.data_ptr()), idx.shape[0],
                                    ctypes.c_void_p(d.data_ptr()), None))
    assert np.array_equal(d.cpu().numpy(), src[idx])
    assert tf.lib().tf_halo_pack(None, None, 0, None, None) == tf.TF_OK  # m = 0: no-op
    with pytest.raises(tf.TopofiltError):
        tf._check(tf.lib().tf_halo_pack(ctypes.c_void_p(src.ctypes.data), ctypes.c_void_p(i.data_ptr()), 5,
                                        ctypes.c_void_p(d.data_ptr()), None))
    with pytest.raises(tf.TopofiltError):
        tf._check(tf.lib().tf_halo_pack(ctypes.c_void_p(s.data_ptr()), ctypes.c_void_p(i.data_ptr()), -1,
                                        ctypes.c_void_p(d.data_ptr()), None))
