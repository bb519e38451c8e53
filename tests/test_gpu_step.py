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


@pytest.mark.parametrize("kind,kw,steps", [
    ("sphere_drape", dict(resolution=14, size=0.2), 8),
    ("skirt", dict(around=160, down=96, radius=0.22), 6),   # subset sites with violator queries
])
def test_determinism(cuda, kind, kw, steps):
    """Run-to-run bitwise determinism (no float atomics feed the state)."""
    import paper_2403_19272_b200 as P

    def run():
        sim = P.build_scene(kind, config=P.StepConfig(h=1.0 / 200.0), **kw)
        for _ in range(steps):
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
    """reference tests/test_stepper.py:174-184 (cloth settling on a sphere), every step
    intersection free.  Run here, the reference itself degenerates on this scene after
    step 21: its exit line search collapses to toi_exit ~5e-15, it shows 6 transient
    cloth-sphere intersections at step 22 and a residual-forwarding blow-up (a 4 m
    vertex jump) at step 24 (tests/golden/contact_sphere14.npz); its own test only
    checks the state after step 25.  This test covers the 21 well-posed steps; the
    teacher-forced test below pins the degenerate ones against the reference."""
    import paper_2403_19272_b200 as P
    from oracle.intersect import intersecting_pairs

    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
    for s in range(21):
        sim.step()
        assert len(intersecting_pairs(sim.world(sim.state.x), sim.bvh.triangles)) == 0, s


def test_contact_teacher_forced_vs_reference(cuda):
    """Every step of the reference's own 25-step sphere drape (tests/golden/
    contact_sphere14.npz, generated by running the reference), teacher forced: the
    GPU is given the reference's full state before step s and must land on the
    reference's state after it.  Covers first contact, residual forwarding and the
    line-search collapse of steps 16-23 (including the reference's transient
    intersections at step 22).  Step 24 is excluded: there the reference's residual
    forwarding blows up (186 LG iterations, a 4 m vertex jump) and the outcome is
    chaotic in the last bit of every input.  Step 23 is the onset of that blow-up: its
    exit TOI (4.9e-9) sits at the round-off floor of the distance march, and flips with
    the last bit of the reduced correction (LAPACK's blocked LU vs the one-CTA LU), so
    it is held to the LG / RF decisions, a 10 % TOI band and 1e-8 m."""
    import paper_2403_19272_b200 as P
    from conftest import golden

    g = golden("contact_sphere14.npz")
    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
    errs = []
    for s in range(24):
        sim.state = P.SimState(x=g["x"][s], x_dot=g["x_dot"][s], x_prev=g["x_prev"][s], delta_f=g["delta_f"][s],
                               step_index=s)
        sim.obstacle_x = g["obstacle_x"][s]
        r = sim.step()
        err = float(np.abs(sim.state.x - g["x"][s + 1]).max())
        assert r.lg_iterations == g["lg"][s], s
        assert r.rf_triggered == bool(g["rf"][s]), s
        if s == 23:
            assert abs(r.toi_exit - g["toi"][s]) <= 0.1 * g["toi"][s], s
            assert err <= 1e-8, (s, err)
            continue
        errs.append(err)
        assert abs(r.toi_exit - g["toi"][s]) <= 1e-9 * max(g["toi"][s], 1e-300) + 1e-15, s
    assert max(errs) <= 1e-12, errs


@pytest.mark.parametrize("kind,kw,steps", [
    ("sphere_ground", dict(resolution=14, size=0.25), 10),                  # BASELINE config 2 (small)
    ("stacked_twist", dict(resolution=10, size=0.3, sheets=2, gap=0.0015), 6),  # config 3: sheet-sheet contact
    ("skirt", dict(around=40, down=14, radius=0.205), 12),                   # config 4 geometry, moving body
    ("desk_fold", dict(resolution=12, size=0.3), 14),                        # reference scene kind
])
def test_scene_teacher_forced_vs_oracle(cuda, kind, kw, steps):
    """Each step starts from the oracle's state: positions, report
    counters and the line-search clamp must agree (contact decisions included)."""
    import paper_2403_19272_b200 as P

    cfg = P.StepConfig(h=1.0 / 200.0)
    sim = P.build_scene(kind, config=cfg, **kw)
    ref = OracleSimulation.from_simulation(sim)
    worst = 0.0
    contact = 0
    for s in range(steps):
        sim.state = ref.state
        sim.obstacle_x = ref.obstacle_x
        r = sim.step()
        rr = ref.step()
        contact = max(contact, r.active_pairs)
        assert r.active_pairs == rr["active_pairs"], (kind, s)
        assert r.lg_iterations == rr["lg_iterations"], (kind, s)
        assert r.full_ccd_calls == rr["full_ccd_calls"], (kind, s)
        assert r.rf_triggered == rr["rf_triggered"], (kind, s)
        worst = max(worst, float(np.abs(sim.state.x - ref.state.x).max()))
        assert worst <= 1e-9, (kind, s, worst)
    assert contact > 0, f"{kind}: the scene should exercise the barrier (engaged pairs)"


@pytest.mark.parametrize("kind,kw,steps", [
    ("sphere_drape", dict(resolution=14, size=0.2), 16),
    ("skirt", dict(around=40, down=14, radius=0.205), 12),
])
def test_static_exit_site_subset_is_exact(cuda, monkeypatch, kind, kw, steps):
    """The exit line search's motion-free CCD site reuses the previous site's pairs
    (abi.cu broad_phase_static); with CS_VERIFY_STATIC_SITE the driver recomputes the
    full broad phase every time and fails the step on any difference."""
    import paper_2403_19272_b200 as P

    monkeypatch.setenv("CS_VERIFY_STATIC_SITE", "1")
    sim = P.build_scene(kind, config=P.StepConfig(h=1.0 / 200.0), **kw)
    served = 0
    for _ in range(steps):
        sim.step()
        served += sim.last_report_c.static_sites
    assert served >= steps // 2, served


@pytest.mark.parametrize("kind,kw,steps", [
    ("sphere_drape", dict(resolution=14, size=0.2), 16),
    ("skirt", dict(around=40, down=14, radius=0.205), 12),
    ("stacked_twist", dict(resolution=10, size=0.3, sheets=2, gap=0.0015), 8),
    ("desk_fold", dict(resolution=12, size=0.3), 14),
    ("sphere_ground", dict(resolution=14, size=0.25), 10),     # large ground triangles: oversize in the grid
    ("skirt", dict(around=160, down=96, radius=0.22), 8),       # 15 K vertices on the spinning body
])
def test_subset_sites_are_exact(cuda, monkeypatch, kind, kw, steps):
    """Outer-loop CCD sites reuse the step's base site (abi.cu subset_site: surviving
    base pairs + violator queries); with CS_VERIFY_STATIC_SITE every such site is
    recomputed by the full broad phase and any difference in the key set fails."""
    import paper_2403_19272_b200 as P

    monkeypatch.setenv("CS_VERIFY_STATIC_SITE", "1")
    sim = P.build_scene(kind, config=P.StepConfig(h=1.0 / 200.0), **kw)
    served = verified = 0
    for _ in range(steps):
        sim.step()
        c = sim.last_report_c
        served += c.subset_sites
        verified += c.verified_sites
        # every subset / motion-free site of the step was re-checked (the check's own
        # broad phase runs on private grid tables, so the base survives it)
        assert c.verified_sites >= c.subset_sites + c.static_sites, (c.verified_sites, c.subset_sites)
    assert served >= steps // 2, served


def test_subset_sites_verified_across_outer_loops(cuda, monkeypatch):
    """Contact steps with two outer loops (BASELINE config 2, the reference's own steps 11
    and 12 of tests/golden/traj_sphere_ground128.npz): the 2nd outer-loop site of a step
    still takes the subset path after the first one was verified, and is verified too
    (a verification broad phase must not invalidate the step's base site)."""
    import paper_2403_19272_b200 as P
    from conftest import golden

    monkeypatch.setenv("CS_VERIFY_STATIC_SITE", "1")
    g = golden("traj_sphere_ground128.npz")
    h, first, xs = float(g["h"]), int(g["first"]), g["x"]
    df = np.zeros_like(xs)
    df[g["df_nonzero"]] = g["delta_f"]
    sim = P.build_scene("sphere_ground", resolution=128, size=1.0, config=P.StepConfig(h=h))
    obstacles = sim.obstacle_x.copy()
    best = 0
    for j in range(1, len(xs) - 1):
        k = first + j + 1
        sim.state = P.SimState(x=xs[j], x_dot=(xs[j] - xs[j - 1]) / h, x_prev=xs[j - 1], delta_f=df[j],
                               step_index=k)
        sim.obstacle_x = obstacles
        r = sim.step()
        c = sim.last_report_c
        assert r.outer_loops == g["outer"][k]
        assert c.verified_sites >= c.subset_sites + c.static_sites
        best = max(best, c.subset_sites)
    assert max(g["outer"][first + 2:first + len(xs)]) >= 2
    assert best >= 2, "no step served more than one outer-loop site from its base"


def test_subset_sites_exact_without_slack(cuda, monkeypatch):
    """No margin slack on the base site: most moving vertices become violators, so the
    violator queries (grid walks + violator brute force) carry the site; still exact."""
    import paper_2403_19272_b200 as P

    monkeypatch.setenv("CS_VERIFY_STATIC_SITE", "1")
    monkeypatch.setenv("CS_SITE_SLACK", "0")
    sim = P.build_scene("stacked_twist", resolution=10, size=0.3, sheets=2, gap=0.0015,
                        config=P.StepConfig(h=1.0 / 200.0))
    served = 0
    for _ in range(8):
        sim.step()
        served += sim.last_report_c.subset_sites
    assert served >= 4, served


def test_subset_sites_exact_in_dbb_mode(cuda, monkeypatch):
    """DBB baseline mode runs the same site sequence; its subset sites are exact too."""
    import paper_2403_19272_b200 as P

    monkeypatch.setenv("CS_VERIFY_STATIC_SITE", "1")
    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig(barrier_mode="dbb"))
    served = 0
    for _ in range(16):
        sim.step()
        served += sim.last_report_c.subset_sites
    assert served >= 4, served


def test_subset_sites_match_full_broad_phase_trajectory(cuda, monkeypatch):
    """Same trajectory bit for bit with and without subset sites (pair order may differ;
    the per-step counters and positions must not move beyond round-off)."""
    import paper_2403_19272_b200 as P

    def run(env):
        if env:
            monkeypatch.setenv("CS_NO_SUBSET_SITES", "1")
        else:
            monkeypatch.delenv("CS_NO_SUBSET_SITES", raising=False)
        sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
        out = []
        for _ in range(12):
            r = sim.step()
            out.append((r.lg_iterations, r.outer_loops, r.rf_triggered))
        return out, sim.state.x.copy()

    a, xa = run(False)
    b, xb = run(True)
    assert a == b
    assert np.abs(xa - xb).max() <= 1e-12


def _contact_state(steps=12):
    """sphere_drape res 14 after `steps` steps: engaged pairs present."""
    import paper_2403_19272_b200 as P

    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
    for _ in range(steps):
        sim.step()
    return sim, OracleSimulation.from_simulation(sim)


def test_witness_and_collision_terms_match_oracle(cuda):
    """Drop-in Simulation._witness / _collision_terms (stepper.py:194-285) vs the oracle."""
    from oracle.stepper import Pairs

    sim, ref = _contact_state()
    xw = sim.world(sim.state.x)
    pairs = sim.broad_phase(xw, xw)
    sim._witness(pairs, xw)
    rp = Pairs(pairs.kind, pairs.idx)
    ref.witness_into(rp, xw)
    assert np.array_equal(pairs.bary, rp.bary) and np.array_equal(pairs.distance, rp.dist)
    assert np.array_equal(pairs.normal, rp.normal)
    engaged = pairs.distance < 2.0 * sim.config.d_hat
    assert engaged.any()
    pairs.weight = np.where(engaged, sim.k * 2.0, 0.0)
    rp.weight = pairs.weight
    got = sim._collision_terms(pairs, engaged, xw + 1e-5)
    exp = ref.collision_terms(rp, engaged, xw + 1e-5)
    for g, e in zip(got, exp):
        assert np.array_equal(g, e)


def test_residual_forward_matches_oracle(cuda):
    """Drop-in Simulation.residual_forward (stepper.py:626-672) vs the oracle on a contact
    state: frozen-weight proxy, energy gradient, reuse-basis corrections + smoothing."""
    from oracle.stepper import Pairs

    sim, ref = _contact_state()
    st = ref.state
    x = st.x
    z = x + sim.config.h * st.x_dot
    xw = sim.world(x)
    pairs = sim.broad_phase(xw, xw)
    sim._witness(pairs, xw)
    rp = Pairs(pairs.kind, pairs.idx)
    ref.witness_into(rp, xw)
    got = sim.residual_forward(x, z, pairs, xw)
    exp = ref.residual_forward(x, z, rp, xw)
    scale = max(float(np.abs(exp).max()), 1e-30)
    assert np.abs(got - exp).max() <= 1e-9 * scale


def test_dbb_baseline_mode_matches_reference(cuda):
    """barrier_mode="dbb" (reference stepper.py:489-491, 524-538, 566-568): free running
    against the reference's own trajectory (tests/golden/traj_sphere14_dbb.npz) and teacher
    forced against the oracle through the contact steps."""
    import paper_2403_19272_b200 as P
    from conftest import golden

    g = golden("traj_sphere14_dbb.npz")
    cfg = P.StepConfig(barrier_mode="dbb")
    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=cfg)
    ref = OracleSimulation.from_simulation(sim)
    for s in range(len(g["lg"])):
        sim.state = ref.state
        sim.obstacle_x = ref.obstacle_x
        r = sim.step()
        rr = ref.step()
        assert r.lg_iterations == rr["lg_iterations"] == g["lg"][s], s
        assert np.abs(ref.state.x - g["x"][s]).max() <= 1e-12, s       # oracle pinned to the reference
        assert np.abs(sim.state.x - ref.state.x).max() <= 1e-9, s
    assert max(g["lg"]) > 1


def test_dbb_free_running_close(cuda):
    import paper_2403_19272_b200 as P
    from conftest import golden

    g = golden("traj_sphere14_dbb.npz")
    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig(barrier_mode="dbb"))
    for s in range(len(g["lg"])):
        r = sim.step()
        assert r.lg_iterations == g["lg"][s], s
        assert np.abs(sim.state.x - g["x"][s]).max() <= 1e-8, s


def test_two_corner64_vs_reference(cuda):
    """BASELINE config 1 at its stated size (64^2, pinned at two corners, h = 1/200)
    against the reference's own 20-step run (tests/golden/traj_two_corner64.npz):
    free running, every step's positions and counters."""
    import paper_2403_19272_b200 as P
    from conftest import golden

    g = golden("traj_two_corner64.npz")
    sim = P.build_scene("two_corner", resolution=64, config=P.StepConfig(h=1.0 / 200.0))
    for s in range(len(g["x"])):
        r = sim.step()
        assert r.lg_iterations == g["lg"][s], s
        assert r.outer_loops == g["outer"][s], s
        assert r.full_ccd_calls == g["sites"][s], s
        assert np.abs(sim.state.x - g["x"][s]).max() <= 1e-9, s
    assert np.abs(sim.state.x_dot - g["x_dot"]).max() <= 1e-6


def test_sphere_ground128_contact_vs_reference(cuda):
    """BASELINE config 2 at its stated size (128^2 cloth onto a sphere above a ground
    slab) against the reference's own run (tests/golden/traj_sphere_ground128.npz):
    the first contact steps, teacher forced from the reference's state, must land on
    the reference's next state with identical counters and line-search TOI."""
    import paper_2403_19272_b200 as P
    from conftest import golden

    g = golden("traj_sphere_ground128.npz")
    h = float(g["h"])
    first = int(g["first"])
    xs = g["x"]
    df = np.zeros_like(xs)
    df[g["df_nonzero"]] = g["delta_f"]
    sim = P.build_scene("sphere_ground", resolution=128, size=1.0, config=P.StepConfig(h=h))
    obstacles = sim.obstacle_x.copy()
    contact = 0
    for j in range(1, len(xs) - 1):
        k = first + j + 1                      # steps taken before this one
        sim.state = P.SimState(x=xs[j], x_dot=(xs[j] - xs[j - 1]) / h, x_prev=xs[j - 1], delta_f=df[j],
                               step_index=k)
        sim.obstacle_x = obstacles
        r = sim.step()
        contact = max(contact, r.active_pairs)
        assert r.active_pairs == g["active"][k], k
        assert r.lg_iterations == g["lg"][k], k
        assert r.outer_loops == g["outer"][k], k
        assert r.rf_triggered == bool(g["rf"][k]), k
        assert abs(r.toi_exit - g["toi"][k]) <= 1e-9 * g["toi"][k] + 1e-15, k
        assert np.abs(sim.state.x - xs[j + 1]).max() <= 1e-9, k
    assert contact > 0



_PLAN_SCENES = [
    ("sphere_drape", dict(resolution=14, size=0.2), 14),
    ("skirt", dict(around=40, down=14, radius=0.205), 10),
    ("stacked_twist", dict(resolution=10, size=0.3, sheets=2, gap=0.0015), 8),
]


@pytest.mark.parametrize("kind,kw,steps", _PLAN_SCENES)
def test_stamp_plan_reuse_is_bitwise(cuda, monkeypatch, kind, kw, steps):
    """Many LG iterations per outer loop (the paper's iteration-cap regime): the driver
    reuses the row order of the collision stamps across iterations (pairs leaving the
    engaged set keep w = 0 entries, joining pairs are merged in).  Positions and
    counters must equal, bit for bit, a run that rebuilds the order every iteration
    (CS_NO_STAMP_PLAN)."""
    import paper_2403_19272_b200 as P

    cfg = P.StepConfig(h=1.0 / 200.0, eps_inner=1e-9, eps_outer=1e-9, iteration_cap=16)

    def run(plan):
        if plan:
            monkeypatch.delenv("CS_NO_STAMP_PLAN", raising=False)
        else:
            monkeypatch.setenv("CS_NO_STAMP_PLAN", "1")
        sim = P.build_scene(kind, config=cfg, **kw)
        out, reuses = [], 0
        for _ in range(steps):
            r = sim.step()
            out.append((r.lg_iterations, r.outer_loops, r.active_pairs, r.rf_triggered, r.toi_exit))
            reuses += sim.last_report_c.stamp_plan_reuses
        return out, sim.state.x.copy(), reuses

    a, xa, ra = run(True)
    b, xb, rb = run(False)
    assert rb == 0
    assert ra > 0, "the cached stamp plan was never reused"
    assert a == b
    assert np.array_equal(xa, xb)


def test_stamp_plan_teacher_forced_vs_oracle(cuda):
    """Iteration-cap regime with contact, teacher forced against the oracle (which
    rebuilds its stamps from scratch every iteration, stepper.py:238-285)."""
    import paper_2403_19272_b200 as P

    cfg = P.StepConfig(h=1.0 / 200.0, eps_inner=1e-9, eps_outer=1e-9, iteration_cap=12)
    sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=cfg)
    for _ in range(8):
        sim.step()
    ref = OracleSimulation.from_simulation(sim)
    reuses = 0
    for s in range(4):
        sim.state = ref.state
        sim.obstacle_x = ref.obstacle_x
        r = sim.step()
        rr = ref.step()
        reuses += sim.last_report_c.stamp_plan_reuses
        assert r.active_pairs == rr["active_pairs"], s
        assert r.lg_iterations == rr["lg_iterations"], s
        assert float(np.abs(sim.state.x - ref.state.x).max()) <= 1e-9, s
    assert reuses > 0


@pytest.mark.parametrize("kind,kw,steps", [
    ("sphere_drape", dict(resolution=14, size=0.2), 20),        # contact + residual forwarding steps
    ("skirt", dict(around=40, down=14, radius=0.205), 10),
])
def test_lazy_exit_site_is_bitwise(cuda, monkeypatch, kind, kw, steps):
    """The motion-free exit site settled from the last site's witness distances (no pair
    set materialised unless residual forwarding needs it) gives the same trajectory,
    counters and TOIs, bit for bit, as the materialised site (CS_NO_LAZY_EXIT)."""
    import paper_2403_19272_b200 as P

    def run(lazy):
        if lazy:
            monkeypatch.delenv("CS_NO_LAZY_EXIT", raising=False)
        else:
            monkeypatch.setenv("CS_NO_LAZY_EXIT", "1")
        sim = P.build_scene(kind, config=P.StepConfig(h=1.0 / 200.0), **kw)
        out, lazy_sites = [], 0
        for _ in range(steps):
            r = sim.step()
            out.append((r.lg_iterations, r.outer_loops, r.full_ccd_calls, r.active_pairs, r.rf_triggered,
                        r.toi_exit))
            lazy_sites += sim.last_report_c.lazy_exit_sites
        return out, sim.state.x.copy(), sim.state.delta_f.copy(), lazy_sites

    a, xa, fa, la = run(True)
    b, xb, fb, lb = run(False)
    assert lb == 0 and la > 0
    assert a == b
    assert np.array_equal(xa, xb) and np.array_equal(fa, fb)


@pytest.mark.parametrize("kind,kw,steps,cap", [
    ("sphere_drape", dict(resolution=14, size=0.2), 14, 0),
    ("skirt", dict(around=40, down=14, radius=0.205), 8, 12),
    ("stacked_twist", dict(resolution=10, size=0.3, sheets=2, gap=0.0015), 8, 12),
])
def test_far_pair_shortcut_is_bitwise(cuda, monkeypatch, kind, kw, steps, cap):
    """Partial CCD's far-pair shortcut (witness distance beyond 2 d_hat plus both sides'
    candidate displacements: provably inactive and disengaged) leaves trajectories and
    counters bit for bit unchanged (CS_NO_FAR_PAIRS runs the full classifier everywhere)."""
    import paper_2403_19272_b200 as P

    extra = dict(eps_inner=1e-9, eps_outer=1e-9, iteration_cap=cap) if cap else {}
    cfg = P.StepConfig(h=1.0 / 200.0, **extra)

    def run(fast):
        if fast:
            monkeypatch.delenv("CS_NO_FAR_PAIRS", raising=False)
        else:
            monkeypatch.setenv("CS_NO_FAR_PAIRS", "1")
        sim = P.build_scene(kind, config=cfg, **kw)
        out = []
        for _ in range(steps):
            r = sim.step()
            out.append((r.lg_iterations, r.outer_loops, r.active_pairs, r.rf_triggered, r.toi_exit))
        return out, sim.state.x.copy()

    a, xa = run(True)
    b, xb = run(False)
    assert a == b
    assert np.array_equal(xa, xb)
