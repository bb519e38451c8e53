"""Parity at the benchmarked scale (BASELINE config 4, the 584 x 584 tube skirt, and
config 5's 317^2 drape), against the CPU oracle.

The headline number is measured on a regime no small test reaches: 1.03 mm row
spacing (about d_hat), so nearly every primitive sits in the barrier band and a CCD
site carries ~30 M candidate pairs.  These tests check the device path at that
size and spacing:

* every subset / motion-free CCD site the step takes is re-derived by the full
  broad phase (CS_VERIFY_STATIC_SITE) on the 584^2 skirt;
* the broad phase of one real site (the motion of a step) equals the oracle's
  set (reference collision/bvh.py:207-292), all ~30 M pairs;
* full CCD and the distance march of the step path (site filter + worklists,
  reference collision/ccd.py:138-266) are bitwise on every pair that can touch
  within the site's motion plus a 1 M random sample of the rest;
* partial CCD (collision/partial.py:149-204) and the witness
  (collision/geometry.py:115-148) are bitwise on a 1 M sample;
* one full step, teacher forced, against OracleSimulation on a skirt band with
  the bench's spacing (584 around x 64 down), and two contact steps of a config-5
  drape (100 K vertices).

Run by `pytest -m gpu` on the B200 box (the oracle runs on its host cores).
"""

import numpy as np
import pytest

from oracle import narrow as ON
from oracle.broad import broad_phase as oracle_broad
from oracle.stepper import OracleSimulation, Pairs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SAMPLE = 1_000_000


def _keys_sorted(kind, idx):
    k = Pairs(np.asarray(kind), np.asarray(idx, np.int64)).keys()
    return k[np.lexsort(k.T[::-1])]


def _chunks(n, size=2_000_000):
    for a in range(0, n, size):
        yield slice(a, min(n, a + size))


@pytest.fixture(scope="module")
def skirt584(cuda):
    """584^2 skirt after two verified steps; returns (sim, oracle clone, xw0, xw1):
    the world positions before / after the third step (one step of real motion)."""
    import os

    import paper_2403_19272_b200 as P
    from paper_2403_19272_b200 import scenes as S

    os.environ["CS_VERIFY_STATIC_SITE"] = "1"
    try:
        sim = S.skirt_scene(P.StepConfig(h=1.0 / 200.0), around=584, down=584, eigensolver="device")
        verified = served = 0
        for _ in range(2):
            sim.step()
            c = sim.last_report_c
            served += c.subset_sites + c.static_sites
            verified += c.verified_sites
            assert c.verified_sites >= c.subset_sites + c.static_sites
        assert served >= 2 and verified >= served, (served, verified)
    finally:
        os.environ.pop("CS_VERIFY_STATIC_SITE", None)
    x0, o0 = sim.state.x.copy(), np.array(sim.obstacle_x, copy=True)
    sim.step()
    x1, o1 = sim.state.x.copy(), np.array(sim.obstacle_x, copy=True)
    ref = OracleSimulation.from_simulation(sim)
    return sim, ref, sim.world(x0, o0), sim.world(x1, o1)


@pytest.fixture(scope="module")
def site584(skirt584):
    """The device CCD site of that motion (step path: broad phase, site filter,
    worklists): pairs, full-CCD TOIs, distance-march TOIs."""
    sim, ref, xw0, xw1 = skirt584
    pairs, toi, filt = sim._full_ccd_site(xw0, xw1)
    assert len(pairs) > 10_000_000, len(pairs)     # the bench regime: tens of millions of pairs
    return pairs, toi, filt


def test_skirt584_broad_phase_set_equals_oracle(skirt584, site584):
    sim, ref, xw0, xw1 = skirt584
    pairs, _, _ = site584
    kind, idx = oracle_broad(xw0, xw1, ref.topo, sim.config.d_hat)
    assert len(kind) == len(pairs), (len(kind), len(pairs))
    got = _keys_sorted(pairs.kind, pairs.idx)
    exp = _keys_sorted(kind, idx)
    assert np.array_equal(got, exp)
    assert not (np.diff(got, axis=0) == 0).all(axis=1).any(), "duplicate rows"


def _reachable(kind, idx, xw0, xw1, dist0, d_hat):
    """Pairs that can come within reach during the site: witness distance at the start
    no larger than both sides' largest displacement plus the barrier band."""
    disp = np.linalg.norm(xw1 - xw0, axis=1)
    side_a = np.where(kind == 0, disp[idx[:, 0]], np.maximum(disp[idx[:, 0]], disp[idx[:, 1]]))
    side_b = np.where(kind == 0, np.maximum(np.maximum(disp[idx[:, 1]], disp[idx[:, 2]]), disp[idx[:, 3]]),
                      np.maximum(disp[idx[:, 2]], disp[idx[:, 3]]))
    return dist0 <= 2.0 * (side_a + side_b) + 4.0 * d_hat


def test_skirt584_ccd_site_bitwise(skirt584, site584):
    """full_ccd and distance_toi of the device step path vs the oracle, bit for bit."""
    import paper_2403_19272_b200 as P

    sim, ref, xw0, xw1 = skirt584
    pairs, toi, filt = site584
    kind, idx = pairs.kind, pairs.idx
    _, _, _, dist0 = P.pair_witness(kind, idx, xw0)
    near = np.flatnonzero(_reachable(kind, idx, xw0, xw1, dist0, sim.config.d_hat))
    hits = np.flatnonzero(~np.isnan(toi) | ~np.isnan(filt))
    assert np.isin(hits, near).all(), "a device hit outside the reachable set"
    # every device hit, 1.5 M of the reachable pairs (where a wrongly filtered pair would
    # hide) and 0.5 M of all pairs
    rng = np.random.default_rng(584)
    sel = np.union1d(np.union1d(hits, rng.choice(near, min(len(near), 1_500_000), replace=False)),
                     rng.choice(len(kind), SAMPLE // 2, replace=False))
    for sl in _chunks(len(sel)):
        s = sel[sl]
        e_toi = ON.full_ccd(kind[s], idx[s], xw0, xw1)
        e_flt = ON.distance_toi(kind[s], idx[s], xw0, xw1, floor_frac=1.0 - sim.config.alpha)
        np.testing.assert_array_equal(toi[s], e_toi)
        np.testing.assert_array_equal(filt[s], e_flt)
    assert len(near) > 100_000, len(near)


def test_skirt584_partial_ccd_and_witness_bitwise(skirt584, site584):
    """partial_ccd over the site's pairs for the real step motion and for a 1 mm
    random perturbation of it (which flips many pair offsets, so the active set is
    large); every device-active pair (up to 500 K) + a 1 M random sample vs the oracle."""
    import paper_2403_19272_b200 as P

    sim, ref, xw0, xw1 = skirt584
    pairs, _, _ = site584
    rng = np.random.default_rng(5840)
    samples = P.default_samples(sim.config.samples)
    xw1p = xw1 + rng.uniform(-1e-3, 1e-3, xw1.shape)
    n_active = 0
    for xe in (xw1, xw1p):
        got_all = P.partial_ccd(pairs.kind, pairs.idx, xw0, xe, samples)
        act = np.flatnonzero(got_all)
        n_active = max(n_active, len(act))
        s = np.union1d(act[rng.permutation(len(act))[:500_000]], rng.choice(len(pairs), SAMPLE, replace=False))
        exp = ON.partial_ccd(pairs.kind[s], pairs.idx[s], xw0, xe, sim.config.samples)
        np.testing.assert_array_equal(got_all[s], exp)
    assert n_active > 10_000, n_active
    s = np.sort(rng.choice(len(pairs), SAMPLE, replace=False))
    kind, idx = pairs.kind[s], pairs.idx[s]
    for got_w, exp_w in zip(P.pair_witness(kind, idx, xw1), ON.witness(kind, idx, xw1)):
        np.testing.assert_array_equal(got_w, exp_w)


def test_skirt_band_step_teacher_forced(cuda):
    """One full step (warm start, three CCD sites, LG loop, NDB, exit line search) at the
    bench's spacing: a 584-around x 64-down band of the skirt (same 1.03 mm rows and
    body motion, 37 K vertices), from a GPU-settled state, vs OracleSimulation."""
    import paper_2403_19272_b200 as P
    from paper_2403_19272_b200 import scenes as S

    down = 64
    sim = S.skirt_scene(P.StepConfig(h=1.0 / 200.0), around=584, down=down, length=0.6 * (down - 1) / 583)
    for _ in range(3):
        sim.step()
    for _ in range(1):
        ref = OracleSimulation.from_simulation(sim)
        r = sim.step()
        rr = ref.step()
        assert r.active_pairs == rr["active_pairs"] > 0
        assert r.lg_iterations == rr["lg_iterations"]
        assert r.full_ccd_calls == rr["full_ccd_calls"]
        assert r.rf_triggered == rr["rf_triggered"]
        assert abs(r.toi_exit - rr["toi_exit"]) <= 1e-12
        assert np.abs(sim.state.x - ref.state.x).max() <= 1e-9


def test_drape317_contact_steps_teacher_forced(cuda):
    """BASELINE config 5 (one 100 K-vertex drape of the batch, material 0): free fall
    to first contact on the device, then two contact steps vs OracleSimulation."""
    import paper_2403_19272_b200 as P
    from paper_2403_19272_b200 import scenes as S

    sim = S.drape_scene(0, resolution=317, config=P.StepConfig(h=1.0 / 200.0), eigensolver="device")
    engaged = 0
    for _ in range(40):
        r = sim.step()
        if r.active_pairs > 0:
            engaged += 1
            if engaged >= 2:
                break
    assert engaged >= 2, "the drape never reached the sphere"
    for _ in range(2):
        ref = OracleSimulation.from_simulation(sim)
        r = sim.step()
        rr = ref.step()
        assert r.active_pairs == rr["active_pairs"] > 0
        assert r.lg_iterations == rr["lg_iterations"]
        assert r.full_ccd_calls == rr["full_ccd_calls"]
        assert r.rf_triggered == rr["rf_triggered"]
        assert np.abs(sim.state.x - ref.state.x).max() <= 1e-9
