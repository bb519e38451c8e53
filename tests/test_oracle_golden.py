"""CPU: the oracle reproduces the REAL reference's outputs (tests/golden, made by
tests/golden/make_golden.py from /root/reference) - this is what pins the oracle.

Pair sets, row order, CCD TOIs/hit sets, partial-CCD classes, witnesses, the
rhs and the rank-2 smoother are compared bitwise.  Stages that go through
OpenBLAS (reduced/warm-start corrections, whole trajectories) are bitwise on
the build host and checked to 1e-12 so the suite also holds on a host whose
BLAS kernel differs.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import narrow as N
from oracle import solver as S
from oracle.broad import WorldTopology, broad_phase
from oracle.stepper import OracleSimulation


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return False
    if a.dtype.kind == "f":
        na, nb = np.isnan(a), np.isnan(b)
        return np.array_equal(na, nb) and np.array_equal(a[~na], b[~nb])
    return np.array_equal(a, b)


def test_fit_constants_match_kernel_literals():
    """csrc/narrow.cu kFit hex literals == numpy's inv(vander) (reference ccd.py:22)."""
    hexes = [["0x1.0p+0", "0x0.0p+0", "0x0.0p+0", "0x0.0p+0"],
             ["-0x1.6000000000001p+2", "0x1.2p+3", "-0x1.1fffffffffffcp+2", "0x1.0p+0"],
             ["0x1.2000000000001p+3", "-0x1.68p+4", "0x1.1ffffffffffffp+4", "-0x1.2p+2"],
             ["-0x1.2000000000001p+2", "0x1.bp+3", "-0x1.bp+3", "0x1.2p+2"]]
    lit = np.array([[float.fromhex(h) for h in row] for row in hexes])
    assert np.array_equal(lit, N.FIT)


def test_full_ccd_golden():
    g = golden("narrow.npz")
    assert same(N.full_ccd(g["kind"], g["idx"], g["x0"], g["x1"]), g["toi"])
    assert same(N.full_ccd(g["kind_n"], g["idx"], g["y0"], g["y1"]), g["toi_n"])
    assert (~np.isnan(g["toi"])).sum() > 50


def test_full_ccd_single_pair_golden():
    g = golden("narrow.npz")
    got = [N.full_ccd(g["kind"][i:i + 1], np.array([[0, 1, 2, 3]]), g["x0"][4 * i:4 * i + 4],
                      g["x1"][4 * i:4 * i + 4])[0] for i in range(200)]
    assert same(np.array(got), g["toi_single"])


def test_distance_toi_golden():
    g = golden("narrow.npz")
    for f in (0.2, 1.0 - 0.8):
        assert same(N.distance_toi(g["kind"], g["idx"], g["x0"], g["x1"], floor_frac=f), g[f"dist_{f!r}"])
        assert same(N.distance_toi(g["kind_n"], g["idx"], g["y0"], g["y1"], floor_frac=f), g[f"dist_n_{f!r}"])


@pytest.mark.parametrize("count", [1, 3, 6])
def test_partial_ccd_golden(count):
    g = golden("narrow.npz")
    x1 = g["x0"] + 0.4 * (g["x1"] - g["x0"])
    assert same(N.partial_ccd(g["kind"], g["idx"], g["x0"], x1, count), g[f"partial_{count}"])
    assert same(N.partial_ccd(g["kind_n"], g["idx"], g["y0"], g["y1"], count), g[f"partial_n_{count}"])


def test_pair_witness_golden():
    g = golden("narrow.npz")
    p1, p2, bary, dist = N.witness(g["kind_n"], g["idx"], g["y0"])
    assert same(p1, g["w_p1"]) and same(p2, g["w_p2"]) and same(bary, g["w_bary"]) and same(dist, g["w_dist"])


def test_ccd_known_answers():
    """reference tests/test_ccd.py:7-50, 144-167."""
    x0 = np.array([[0.25, 0.25, -1.0], [0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    x1 = x0.copy()
    x1[0, 2] = 1.0
    one = np.array([[0, 1, 2, 3]])
    assert np.isclose(N.full_ccd(np.array([0]), one, x0, x1)[0], 0.5, atol=1e-9)
    r1 = x0.copy()
    r1[0, 2] = -3.0
    assert not N.partial_ccd(np.array([0]), one, x0, r1, 3).any()
    assert N.partial_ccd(np.array([0]), one, x0, x1, 3).all()


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_broad_phase_golden_rows_and_order(k):
    g = golden(f"broad_{k}.npz")
    topo = WorldTopology.build(g["tris"], g["tri_static"])
    kind, idx = broad_phase(g["x0"], g["x1"], topo, float(g["margin"]))
    assert np.array_equal(kind, g["kind"])
    assert np.array_equal(idx, g["idx"])


def _twist16():
    from paper_2403_19272_b200 import StepConfig
    from paper_2403_19272_b200.scenes import scene_parts

    cfg = StepConfig(h=1.0 / 200.0)
    return OracleSimulation.from_parts(scene_parts("twist", resolution=16, size=0.5, config=cfg), cfg)


def test_solver_stages_golden():
    g = golden("solver.npz")
    o = _twist16()
    b0, d0 = S.assemble_rhs(o.sys, o.mesh, o.el, g["z"], g["x"], g["pins"])
    b1, d1 = S.assemble_rhs(o.sys, o.mesh, o.el, g["z"], g["x"], g["pins"], g["ids"], g["w"], g["tg"])
    assert same(b0, g["b0"]) and same(d0, g["d0"]) and same(b1, g["b1"]) and same(d1, g["d1"])
    assert same(S.ajacobi_smooth(o.sys, g["bb"], g["xx"], 32, 0.0, g["dl"]), g["smooth"])
    nf = o.mesh.free.size
    for key, delta in (("rc0", np.zeros(nf)), ("rc1", g["dl"]), ("rc2", g["big"])):
        got, red = S.reduced_correction(o.sub, o.sys, g["bb"], g["xx"], delta)
        assert np.abs(got - g[key]).max() <= 1e-12 * np.abs(g[key]).max(), key
    assert bool(red.fallback) == bool(g["rc2_fallback"])
    ws = S.warmstart_correction(o.sub, o.sys, g["bb"], g["xx"])
    assert np.abs(ws - g["ws"]).max() <= 1e-12 * np.abs(g["ws"]).max()


@pytest.mark.parametrize("tag,kind,cfg_kw,scene_kw", [
    ("hanging10", "hanging", dict(h=1.0 / 200.0), dict(resolution=10)),
    ("sphere14", "sphere_drape", {}, dict(resolution=14, size=0.2)),
    ("sphere14_dbb", "sphere_drape", {"barrier_mode": "dbb"}, dict(resolution=14, size=0.2)),
    ("twist10", "twist", {}, dict(resolution=10, size=0.3)),
    ("two_corner64", "two_corner", dict(h=1.0 / 200.0), dict(resolution=64)),
])
def test_trajectory_golden(tag, kind, cfg_kw, scene_kw):
    from paper_2403_19272_b200 import StepConfig
    from paper_2403_19272_b200.scenes import scene_parts

    g = golden(f"traj_{tag}.npz")
    cfg = StepConfig(**cfg_kw)
    o = OracleSimulation.from_parts(scene_parts(kind, config=cfg, **scene_kw), cfg)
    for s in range(len(g["x"])):
        rep = o.step()
        assert rep["lg_iterations"] == g["lg"][s]
        assert np.abs(o.state.x - g["x"][s]).max() <= 1e-12, (tag, s)


def test_intersection_oracle_pinned_to_reference_counts():
    """oracle/intersect.py against the reference's own per-step intersection counts of
    its 25-step sphere drape (tests/golden/contact_sphere14.npz: oracle_intersect run by
    the reference on its states; steps 22-24 carry its transient intersections)."""
    from oracle.intersect import intersecting_pairs
    from paper_2403_19272_b200 import StepConfig
    from paper_2403_19272_b200.scenes import scene_parts

    g = golden("contact_sphere14.npz")
    parts = scene_parts("sphere_drape", resolution=14, size=0.2, config=StepConfig())
    n = parts["mesh"].vertex_count
    ov, ot = parts["obstacles"][0]
    tris = np.concatenate([parts["mesh"].triangles, np.asarray(ot) + n])
    counts = g["intersections"]
    assert counts.max() > 0
    for s in range(len(counts)):
        xw = np.concatenate([g["x"][s + 1], g["obstacle_x"][s + 1]])
        assert len(intersecting_pairs(xw, tris)) == counts[s], s


def test_float_sat_golden_and_exact_arithmetic():
    """The float 17-axis SAT restatement reproduces the reference's verdicts on its
    near-degenerate pair mix bit for bit, and is conservative against the exact rational
    test as the reference requires (tests/test_harness.py:166-181)."""
    from oracle.intersect import exact_separation_margin, tri_tri_intersect, tri_tri_intersect_exact

    g = golden("stages.npz")
    p, q = g["sat_p"], g["sat_q"]
    got = tri_tri_intersect(p, q)
    assert np.array_equal(got, g["sat"])
    for i in range(0, len(p), 5):
        ex = tri_tri_intersect_exact(p[i], q[i])
        assert ex == bool(g["sat_exact"][i])
        if got[i] != ex:
            assert got[i] and not ex
            scale = float(np.abs(np.concatenate([p[i], q[i]])).max()) + 1.0
            assert exact_separation_margin(p[i], q[i]) <= 1e-12 * scale
