"""Pins for the NEXT-1 oracle (OC update with bisection, listing 380-385)."""
import numpy as np
import pytest

import oracle
import synth


def paper_listing(density, sensitivity, volfrac, num_cells):
    """The paper's listing, verbatim numpy; returns the decisions too."""
    l1, l2, move = 0, 100000, 0.2
    decisions = []
    while l2 - l1 > 1e-4:
        l_mid = 0.5 * (l2 + l1)
        density_new = np.maximum(0.001, np.maximum(density - move, np.minimum(1.0, np.minimum(density + move, density * np.sqrt(-sensitivity / l_mid)))))
        up = sum(density_new) - volfrac * num_cells > 0
        decisions.append(bool(up))
        l1, l2 = (l_mid, l2) if up else (l1, l_mid)
    return density_new, l_mid, decisions


@pytest.mark.parametrize("n,volfrac,seed", [(50, 0.5, 1), (400, 0.3, 2), (1000, 0.15, 3), (777, 0.4, 4)])
def test_oc_matches_paper_listing(n, volfrac, seed):
    """Same l_mid sequence and bitwise-identical density_new as the printed listing (whose
    rounded-sum decisions agree with the exact ones away from ties)."""
    d = synth.uniform(100 + seed, 0, n, 0.001, 1.0)
    dc = -synth.uniform(200 + seed, 0, n, 0.0, 2.0)
    ref, lref, dec = paper_listing(d, dc, volfrac, n)
    x, lm, it = oracle.oc_update(d, dc, volfrac)
    assert it == len(dec) == 30
    assert lm == lref
    np.testing.assert_array_equal(x, ref)


def test_oc_closed_form_uniform():
    """Uniform d and dc: d*sqrt(-dc/l) = volfrac at l* = -dc d^2 / volfrac^2 (inside the move
    limits), so the bisection converges to l* within its tolerance."""
    n, d0, dc0, vf = 64, 0.5, -0.8, 0.45
    x, lm, it = oracle.oc_update(np.full(n, d0), np.full(n, dc0), vf)
    lstar = -dc0 * d0 * d0 / (vf * vf)
    assert abs(lm - lstar) <= 2e-4
    assert np.all(x == x[0]) and abs(x[0] - vf) < 1e-4


def test_oc_invariants():
    n = 5000
    d = synth.uniform(301, 0, n, 0.001, 1.0)
    dc = -synth.uniform(302, 0, n, 0.0, 3.0)
    vf = 0.45  # feasible: between the move-limit extremes sum(max(.001, d-.2)) and sum(min(1, d+.2))
    x, lm, it = oracle.oc_update(d, dc, vf)
    assert np.all(x >= 0.001) and np.all(x <= 1.0)
    assert np.all(x >= d - 0.2)  # move limit m = 0.2 (Eq. update)
    assert np.all(x <= np.maximum(0.001, np.minimum(1.0, d + 0.2)))
    # volume constraint met up to the bisection tolerance's effect
    assert abs(x.sum() - vf * n) < 1e-3 * n
    # sum of density_new is nonincreasing in the multiplier
    sums = [oracle.oc_update(d, dc, 0.3, l1=l, l2=l, tol=1.0)[0].sum() for l in (0.01, 0.1, 1.0, 10.0)]
    assert all(a >= b for a, b in zip(sums, sums[1:]))


def test_compliance_sensitivity_matches_listing():
    """NEXT-2 oracle: the paper's listing evaluated verbatim by numpy."""
    x = synth.uniform(701, 0, 1000, 0.001, 1.0)
    U = synth.uniform(702, 0, 1000, 0.0, 5.0)
    for penal in (3.0, 1.0, 2.5):
        ref = -penal * (x) ** (penal - 1) * U
        np.testing.assert_allclose(oracle.compliance_sensitivity(x, U, penal), ref, rtol=4e-16, atol=0)
    # p = 1: dc = -U exactly
    np.testing.assert_array_equal(oracle.compliance_sensitivity(x, U, 1.0), -U)


def test_termination_rule_no_progress():
    """Reading R23: with tol below the fp64 spacing near lambda* the listing's loop never ends;
    the oracle stops when l_mid rounds to l1 or l2 and flags it (bit 1)."""
    n = 64
    d = np.full(n, 0.5)
    dc = np.full(n, -1.0e4)  # lambda* = -dc d^2 / vf^2 = 1e4 at vf = 0.5: spacing there ~1.8e-12
    x, lm, it, fl = oracle.oc_update(d, dc, 0.5, tol=1e-13, flags=True)
    assert fl & 2
    assert it < 4096
    assert np.nextafter(lm, np.inf) - lm > 1e-13 or np.nextafter(lm, -np.inf) - lm < -1e-13


def test_bracket_exhausted_flag():
    """Every step moving l1 up (the volume constraint still violated at l2) sets bit 0; a normal
    run sets no flag."""
    n = 100
    d = np.full(n, 0.9)
    dc = np.full(n, -1.0)
    x, lm, it, fl = oracle.oc_update(d, dc, 0.1, l2=1e-6, tol=1e-12, flags=True)
    assert fl == 1
    assert x.sum() > 0.1 * n
    _, _, _, fl2 = oracle.oc_update(d, dc, 0.8, flags=True)  # reachable within the move limit
    assert fl2 == 0
