"""NEXT-4 host logic (paper_2012_08208_b200/sharded.py): the slab partition and halo plans,
checked against brute-force neighbour sets (no GPU needed)."""
import numpy as np
import pytest

import synth


def plans_mod():
    # the package loads its library on CPU too (no kernel runs here)
    from paper_2012_08208_b200 import sharded
    return sharded


def neighbours(c, rmin):
    d2 = ((c[:, None, :] - c[None, :, :]) ** 2).sum(-1)
    return d2 < rmin * rmin


@pytest.mark.parametrize("name,c,rmin,world", [
    ("random3d_w2", synth.random_points(901, 1500, 3, 0.0, 10.0), 1.3, 2),
    ("random3d_w5", synth.random_points(902, 1500, 3, 0.0, 10.0), 1.3, 5),
    ("thin_slabs_w12", synth.random_points(903, 1200, 2, 0.0, 6.0), 1.5, 12),   # slabs thinner than rmin
    ("kuhn_w4", synth.kuhn_tets(8, 5, 4), 1.5, 4),                              # ties on slab bounds
    ("quads_w3", synth.quad_grid(30, 10), 2.5, 3),
    ("w1", synth.random_points(904, 300, 2, 0.0, 5.0), 1.0, 1),
])
def test_plans_partition_and_complete_halo(name, c, rmin, world):
    m = plans_mod()
    plans = m.make_plans(c, world, rmin)
    n = c.shape[0]
    own = np.concatenate([p.owned for p in plans])
    assert np.array_equal(np.sort(own), np.arange(n))          # owned sets partition [0, n)
    nb = neighbours(c, rmin)
    for p in plans:
        assert np.all(np.diff(p.owned) > 0)
        loc = p.local_ids()
        assert np.unique(loc).shape[0] == loc.shape[0]          # no duplicates
        have = np.zeros(n, bool)
        have[loc] = True
        # every neighbour of every owned point is local: the owned rows are complete
        need = nb[p.owned].any(axis=0)
        assert not (need & ~have).any(), name
        assert p.rank not in p.halo_from
        for j, g in p.halo_from.items():
            assert np.all(np.diff(g) > 0)
            # the sender's plan lists exactly these points, in this order
            assert np.array_equal(plans[j].owned[plans[j].send_to[p.rank]], g)
    if world == 1:
        assert plans[0].n_halo == 0
    # equal coordinates along the cut axis never straddle a cut
    ax = plans[0].axis
    owner = np.empty(n, np.int64)
    for p in plans:
        owner[p.owned] = p.rank
    for v in np.unique(c[:, ax]):
        assert np.unique(owner[c[:, ax] == v]).shape[0] == 1


def test_plans_balanced():
    m = plans_mod()
    c = synth.random_points(905, 20000, 3, 0.0, 50.0)
    plans = m.make_plans(c, 8, 1.5)
    sizes = np.array([p.n_owned for p in plans])
    assert sizes.max() - sizes.min() <= 1
