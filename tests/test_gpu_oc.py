"""NEXT-1 on the GPU: the OC update with bisection (tf_oc_update) against the oracle, bitwise
(same correctly rounded element formula, exact-sum decisions: DESIGN.md R15)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tf():
    assert torch.cuda.is_available()
    import paper_2012_08208_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n,vf,seed", [(1, 0.5, 1), (7, 0.4, 2), (1000, 0.3, 3), (100_003, 0.45, 4),
                                       (1_000_000, 0.5, 5)])
def test_oc_matches_oracle(tf, n, vf, seed):
    d = synth.uniform(400 + seed, 0, n, 0.001, 1.0)
    dc = -synth.uniform(500 + seed, 0, n, 0.0, 2.0)
    ref, lref, itref = oracle.oc_update(d, dc, vf)
    xn, lm, it = tf.tf_oc_update(dev(d), dev(dc), vf)
    assert int(it.item()) == itref
    assert float(lm.item()) == lref
    np.testing.assert_array_equal(xn.cpu().numpy(), ref)


def test_oc_in_place_and_params(tf):
    n = 50_000
    d = synth.uniform(601, 0, n, 0.001, 1.0)
    dc = -synth.uniform(602, 0, n, 0.0, 1.0)
    ref, lref, _ = oracle.oc_update(d, dc, 0.35, move=0.1, l1=0.0, l2=1000.0, tol=1e-6)
    xd = dev(d)
    _, lm, _ = tf.tf_oc_update(xd, dev(dc), 0.35, move=0.1, l2=1000.0, tol=1e-6, x_new=xd)
    np.testing.assert_array_equal(xd.cpu().numpy(), ref)
    assert float(lm.item()) == lref


def test_design_iteration_filter_then_oc(tf):
    """One optimisation-iteration tail on config 3: sensitivity filter (a8) then the OC update,
    against the oracle chain."""
    c, x, dc, rmin = synth.workload(3)
    H = oracle.build_celllist(c, rmin)
    dcf = oracle.apply_sensitivity(H, x, dc)
    ref, lref, _ = oracle.oc_update(x, dcf, 0.5)
    f = tf.tf_build_filter(dev(c), rmin)
    xd = dev(x)
    dcf_g = f.sensitivity(xd, dev(dc))
    xn, lm, _ = tf.tf_oc_update(xd, dcf_g, 0.5)
    # the filtered sensitivities agree to 1e-10 (not bitwise), so compare the updated densities
    # to the same tolerance and the multipliers to the bisection tolerance
    np.testing.assert_allclose(xn.cpu().numpy(), ref, rtol=1e-9, atol=1e-12)
    assert abs(float(lm.item()) - lref) <= 1e-4


def test_oc_rejects_bad_args(tf):
    d = dev(np.full(10, 0.5))
    with pytest.raises(tf.TopofiltError):
        tf.tf_oc_update(d, dev(np.full(10, -1.0)), -0.5)
    with pytest.raises(tf.TopofiltError):
        tf.tf_oc_update(d, dev(np.full(10, -1.0)), 0.5, l1=5.0, l2=1.0)


@pytest.mark.parametrize("cfg,penal", [(2, 3.0), (3, 3.0), (4, 2.5)])
def test_sensitivity_from_energy(tf, cfg, penal):
    """NEXT-2: dc evaluated inside the sensitivity filter's fused pass from element energies."""
    c, x, dc, rmin = synth.workload(cfg)
    U = synth.uniform(800 + cfg, 0, x.shape[0], 0.0, 2.0)
    H = oracle.build_celllist(c, rmin)
    ref = oracle.apply_sensitivity(H, x, oracle.compliance_sensitivity(x, U, penal))
    f = tf.tf_build_filter(dev(c), rmin)
    got = tf.tf_sensitivity_filter_energy(f, dev(x), dev(U), penal).cpu().numpy()
    scale = np.where(ref != 0, np.abs(ref), np.abs(ref).max())
    assert np.all(np.abs(got - ref) <= 1e-10 * scale)


@pytest.mark.parametrize("case", ["no_progress", "exhausted", "x_above_4"])
def test_oc_termination_and_flags(tf, case):
    """Reading R23 and the bracket-exhausted flag, bitwise with the oracle; x outside [0, 1]
    (x > 4, where a 64-bit fixed-point sum would saturate) still matches the exact oracle."""
    n = 5000
    rng = np.random.default_rng(3)
    if case == "no_progress":
        d, dc, kw = np.full(n, 0.5), np.full(n, -1.0e4), dict(tol=1e-13)
        vf = 0.5
    elif case == "exhausted":
        d, dc, kw = rng.uniform(0.5, 1.0, n), -rng.uniform(0.5, 1.5, n), dict(l2=1e-6, tol=1e-12)
        vf = 0.1
    else:
        d, dc, kw = rng.uniform(4.5, 6.0, n), -rng.uniform(0.5, 1.5, n), dict(move=0.2)
        vf = 2.0
    ref, lref, itref, flref = oracle.oc_update(d, dc, vf, flags=True, **kw)
    xn, lm, it, fl = tf.tf_oc_update(dev(d), dev(dc), vf, flags=True, **kw)
    assert int(it.item()) == itref and int(fl.item()) == flref
    assert float(lm.item()) == lref
    np.testing.assert_array_equal(xn.cpu().numpy(), ref)
    if case != "x_above_4":
        assert flref != 0
