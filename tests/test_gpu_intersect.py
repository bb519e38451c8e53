"""GPU intersection check (the penetration-free invariant) vs the oracle's restatement
of reference oracles.py:83-131, and the verify mode it backs (stepper.py:614-621)."""

import numpy as np
import pytest

from oracle.intersect import intersecting_pairs

pytestmark = pytest.mark.gpu


def _rows(a):
    return {tuple(int(v) for v in r) for r in a}


@pytest.mark.parametrize("jitter,seed", [(0.0, 0), (0.01, 1), (0.03, 2), (0.06, 3)])
def test_intersections_equal_oracle(cuda, jitter, seed):
    import paper_2403_19272_b200 as P

    sim = P.build_scene("sphere_drape", resolution=16, size=0.6, config=P.StepConfig(r_bar=8, r=4))
    rng = np.random.default_rng(seed)
    xw = sim.world(sim.state.x)
    n = sim.mesh.vertex_count
    xw[:n] += jitter * rng.normal(size=(n, 3))
    xw[:n, 2] -= 0.17 * (jitter > 0)                # push part of the cloth into the sphere
    got = sim.intersecting_pairs(xw)
    ref = intersecting_pairs(xw, sim.bvh.triangles)
    assert _rows(got) == _rows(ref)
    assert len(got) == len(ref)
    if jitter > 0:
        assert len(ref) > 0


def test_verify_mode_raises_and_keeps_state(cuda):
    import paper_2403_19272_b200 as P

    cfg = P.StepConfig(verify=True, r_bar=8, r=4)
    sim = P.build_scene("sphere_drape", resolution=12, size=0.6, config=cfg)
    for _ in range(2):
        rep = sim.step()
        assert rep.penetration_free
    st = sim.state
    x = st.x.copy()
    x[:, 2] -= 0.17                                  # cloth plane now cuts the sphere
    sim.state = P.SimState(x=x, x_dot=np.zeros_like(x), x_prev=x.copy(), delta_f=np.zeros_like(x),
                           step_index=st.step_index)
    before = sim._step_index
    with pytest.raises(P.PenetrationError) as err:
        sim.step()
    dump = err.value.state_dump
    assert len(dump["pairs"]) > 0 and dump["x"].shape == x.shape
    assert sim._step_index == before
    assert np.array_equal(sim.state.x, x)             # state untouched by the failed step
