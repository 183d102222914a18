"""NEXT-4: the device slab partition (tf_shard_plan, shard.cu) checked against brute-force
neighbour sets: owned sets partition [0, n); every neighbour of an owned point is local (owned rows
complete); interior points have no neighbour outside their slab; halo lists equal the senders'
send lists in order; equal coordinates along the cut axis never straddle a cut; balance; the plan
of config 5 on 8 ranks in well under 5 ms."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sh():
    assert torch.cuda.is_available()
    from paper_2012_08208_b200 import sharded
    return sharded


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def neighbours(c, rmin):
    d2 = ((c[:, None, :] - c[None, :, :]) ** 2).sum(-1)
    return d2 < rmin * rmin


@pytest.mark.parametrize("name,c,rmin,world", [
    ("random3d_w2", synth.random_points(901, 1500, 3, 0.0, 10.0), 1.3, 2),
    ("random3d_w5", synth.random_points(902, 1500, 3, 0.0, 10.0), 1.3, 5),
    ("thin_slabs_w12", synth.random_points(903, 1200, 2, 0.0, 6.0), 1.5, 12),  # slabs thinner than rmin
    ("kuhn_w4", synth.kuhn_tets(8, 5, 4), 1.5, 4),                             # ties on slab bounds
    ("quads_w3", synth.quad_grid(30, 10), 2.5, 3),
    ("w1", synth.random_points(904, 300, 2, 0.0, 5.0), 1.0, 1),
])
def test_plan_partition_and_complete_halo(sh, name, c, rmin, world):
    n = c.shape[0]
    cd = dev(c)
    plans = [sh.ShardPlan(cd, rmin, world, k) for k in range(world)]
    nb = neighbours(c, rmin)
    own = np.concatenate([p.owned_ids.cpu().numpy() for p in plans])
    assert np.array_equal(np.sort(own), np.arange(n))  # owned sets partition [0, n)
    owner = np.empty(n, np.int64)
    for p in plans:
        owner[p.owned_ids.cpu().numpy()] = p.rank
    for p in plans:
        loc = p.local_ids.cpu().numpy()
        assert np.unique(loc).shape[0] == loc.shape[0]
        inter, bnd = loc[:p.n_interior], loc[p.n_interior:p.n_owned]
        assert np.all(np.diff(inter) > 0) and np.all(np.diff(bnd) > 0)
        have = np.zeros(n, bool)
        have[loc] = True
        need = nb[loc[:p.n_owned]].any(axis=0)
        assert not (need & ~have).any(), name  # owned rows are complete
        # interior points: every neighbour owned by this rank
        if p.n_interior:
            assert np.all(owner[nb[inter].any(axis=0)] == p.rank), name
        assert p.recv[p.rank] == 0 and p.send[p.rank] == 0
        for j in range(world):
            h0, h1 = p.halo_range(j)
            g = loc[h0:h1]
            assert np.all(np.diff(g) > 0) and np.all(owner[g] == j)
            q = plans[j]
            s0, s1 = q.send_range(p.rank)
            sent = q.local_ids.cpu().numpy()[q.send_idx[s0:s1].cpu().numpy()]
            assert np.array_equal(sent, g), name  # the sender lists exactly these, in this order
    if world == 1:
        assert plans[0].n_halo == 0 and plans[0].n_interior == n
    ax = plans[0].axis
    for v in np.unique(c[:, ax]):
        assert np.unique(owner[c[:, ax] == v]).shape[0] == 1
    for p in plans:
        p.close()


def test_plan_balanced(sh):
    c = synth.random_points(905, 200000, 3, 0.0, 50.0)
    cd = dev(c)
    sizes = [sh.ShardPlan(cd, 1.5, 8, k).n_owned for k in range(8)]
    assert sum(sizes) == 200000
    assert max(sizes) - min(sizes) <= 0.01 * 200000 / 8  # histogram cuts: within 1% of n/W


def test_plan_config5_cost(sh):
    c, _, _, rmin = synth.workload(5)
    cd = dev(c)
    sh.ShardPlan(cd, rmin, 8, 3).close()  # warm-up
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    p = sh.ShardPlan(cd, rmin, 8, 3)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    assert p.n_owned == 1_500_000 and 0 < p.n_interior < p.n_owned
    assert ms < 5.0, f"plan took {ms:.2f} ms"
    p.close()
