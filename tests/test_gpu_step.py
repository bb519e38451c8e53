"""Full GPU step vs the oracle.

Contact-free scenes: free-running trajectories within 1e-9 m over a fixed
horizon (fp64 everywhere; only OpenBLAS-vs-kernel summation order differs).
Contact scenes: per-step teacher forcing - the GPU is
fed the oracle's state and must land within 1e-7 m of the oracle's next
state; free-running runs must stay penetration free.
"""

import numpy as np
import pytest

from oracle.stepper import OracleSimulation

pytestmark = pytest.mark.gpu


def _pair(kind, **kw):
    import paper_2403_19272_b200 as P

    cfg_kw = {k: kw.pop(k) for k in list(kw) if k in P.StepConfig.__dataclass_fields__}
    cfg = P.StepConfig(**cfg_kw)
    sim = P.build_scene(kind, config=cfg, **kw)
    return sim, OracleSimulation.from_simulation(sim)


@pytest.mark.parametrize("kind,kw,steps", [
    ("hanging", dict(resolution=10, h=1.0 / 200.0), 6),
    ("two_corner", dict(resolution=16, h=1.0 / 200.0), 6),
    ("twist", dict(resolution=12, size=0.3), 6),
    ("free_fall", dict(resolution=6), 5),
])
def test_free_running_matches_oracle(cuda, kind, kw, steps):
    sim, ref = _pair(kind, **kw)
    for s in range(steps):
        r = sim.step()
        rr = ref.step()
        assert r.lg_iterations == rr["lg_iterations"], s
        assert r.full_ccd_calls == rr["full_ccd_calls"] == r.outer_loops + 2
        assert np.abs(sim.state.x - ref.state.x).max() <= 1e-9, s
        assert np.abs(sim.state.x_dot - ref.state.x_dot).max() <= 1e-6, s


def test_contact_teacher_forced(cuda):
    sim, ref = _pair("sphere_drape", resolution=14, size=0.2)
    worst = 0.0
    rf_seen = False
    for s in range(14):
        sim.state = ref.state
        sim.obstacle_x = ref.obstacle_x
        r = sim.step()
        rr = ref.step()
        rf_seen |= rr["rf_triggered"]
        worst = max(worst, float(np.abs(sim.state.x - ref.state.x).max()))
        assert worst <= 1e-7, (s, worst, r.lg_iterations, rr["lg_iterations"])
    assert rf_seen, "scene should exercise residual forwarding"


def test_contact_free_running_close(cuda):
    sim, ref = _pair("sphere_drape", resolution=14, size=0.2)
    for s in range(10):
        sim.step()
        ref.step()
    assert np.abs(sim.state.x - ref.state.x).max() <= 1e-6


def test_determinism(cuda):
    import paper_2403_19272_b200 as P

    def run():
        sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
        for _ in range(8):
            sim.step()
        return sim.state.x.copy()

    assert np.array_equal(run(), run())


def test_ballistic_trajectory(cuda):
    """reference tests/test_stepper.py:27-41."""
    import paper_2403_19272_b200 as P

    verts, tris = P.grid_cloth(4, 1.0, height=1.0)
    sim = P.Simulation(P.build_mesh(verts, tris, density=0.3), P.StepConfig())
    h, g = sim.config.h, np.array(sim.config.gravity)
    x_ref = sim.state.x.copy()
    v = np.zeros_like(x_ref)
    for _ in range(10):
        sim.step()
        v = v + h * g
        x_ref = x_ref + h * v
    assert np.abs(sim.state.x - x_ref).max() <= 1e-6


def test_rest_fixed_point(cuda):
    """reference tests/test_stepper.py:44-51."""
    import paper_2403_19272_b200 as P

    verts, tris = P.grid_cloth(5, 1.0)
    sim = P.Simulation(P.build_mesh(verts, tris, 0.3, pins=np.arange(5)), P.StepConfig(gravity=(0.0, 0.0, 0.0)))
    x0 = sim.state.x.copy()
    sim.step()
    assert np.abs(sim.state.x - x0).max() <= 1e-9


def test_iteration_cap_and_budget(cuda):
    """reference tests/test_stepper.py:78-84, 195-203."""
    import paper_2403_19272_b200 as P

    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig(iteration_cap=1))
    hit = False
    for _ in range(20):
        r = sim.step()
        assert r.full_ccd_calls == r.outer_loops + 2
        hit |= r.cap_hit
    assert hit


def test_resting_contact_penetration_free(cuda):
    """reference tests/test_stepper.py:174-184 with the oracle's exact intersection test."""
    import paper_2403_19272_b200 as P
    from oracle.intersect import intersecting_pairs

    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
    for _ in range(25):
        sim.step()
        assert len(intersecting_pairs(sim.world(sim.state.x), sim.bvh.triangles)) == 0
