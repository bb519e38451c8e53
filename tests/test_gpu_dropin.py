"""Module-level drop-ins (reference clothsim/__init__.py:3-32, collision/__init__.py:1-5)
run on the device: the reference's own stage values (tests/golden/stages.npz, made by
running the reference) and restatements of the reference tests that exercise them
(pkg/tests/test_partial_ccd.py, test_geometry.py, test_smoothing.py, test_subspace.py,
test_constraints.py, test_bvh.py, test_harness.py)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G(cuda):
    return golden("stages.npz")


def test_coplanarity_coefficients_bitwise(G):
    import paper_2403_19272_b200 as P

    assert np.array_equal(P.coplanarity_coefficients(G["kind"], G["idx"], G["x0"], G["x1"]), G["coef"])
    for i in range(50):      # m = 1 takes OpenBLAS's single-row path
        got = P.coplanarity_coefficients(G["kind"][i:i + 1], np.array([[0, 1, 2, 3]]), G["x0"][4 * i:4 * i + 4],
                                         G["x1"][4 * i:4 * i + 4])
        assert np.array_equal(got[0], G["coef_single"][i]), i


def test_query_q_bitwise(G):
    import paper_2403_19272_b200 as P

    assert np.array_equal(P.query_q(G["kind"], G["idx"], G["x0"], G["x1"], G["lam_shared"]), G["q_shared"])
    assert np.array_equal(P.query_q(G["kind"], G["idx"], G["x0"], G["x1"], G["lam_pair"]), G["q_pair"])


def test_query_q_reference_cases(cuda):
    """reference tests/test_partial_ccd.py:32-53."""
    import paper_2403_19272_b200 as P

    x = np.array([[0.25, 0.25, 1.0], [0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    assert np.isclose(P.query_q(np.array([0]), np.array([[0, 1, 2, 3]]), x, x, np.array([[0.25, 0.25]]))[0, 0], 1.0)
    x0 = np.array([[0.25, 0.25, -1.0], [0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    x1 = x0.copy()
    x1[0, 2] = 1.0
    kind, idx = np.array([0]), np.array([[0, 1, 2, 3]])
    assert np.isclose(P.query_q(kind, idx, x0, x1, np.array([[0.25, 0.25]]))[0, 0], -1.0)
    t = P.full_ccd(kind, idx, x0, x1)[0]
    assert np.isclose(P.query_q(kind, idx, x0, x1, np.array([[0.25, 0.25]]))[0, 0], (t - 1.0) / t, atol=1e-9)
    assert P.partial_ccd(kind, idx, x0, x1, P.default_samples(3)).all()


def test_closest_points_and_boxes_bitwise(G):
    import paper_2403_19272_b200 as P

    q = G["x0"][G["idx"]]
    n = len(q)
    got = np.concatenate([np.asarray(a).reshape(n, -1) for a in P.point_triangle_closest(q[:, 0], q[:, 1], q[:, 2],
                                                                                          q[:, 3])], 1)
    assert np.array_equal(got, G["ptc"])
    got = np.concatenate([np.asarray(a).reshape(n, -1) for a in P.segment_segment_closest(q[:, 0], q[:, 1], q[:, 2],
                                                                                           q[:, 3])], 1)
    assert np.array_equal(got, G["ssc"])
    lo, hi = P.swept_boxes(G["x0"][G["idx"]], G["x1"][G["idx"]], 1e-3)
    assert np.array_equal(lo, G["sb_lo"]) and np.array_equal(hi, G["sb_hi"])
    # reference tests/test_geometry.py:27-33
    t = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    c, b, d = P.point_triangle_closest(np.array([[0.25, 0.25, 0.5]]), t[None, 0], t[None, 1], t[None, 2])
    assert np.allclose(d, 0.5) and np.allclose(b, [[0.25, 0.25]]) and np.allclose(c, [[0.25, 0.25, 0.0]])


def test_dbb_weights(G):
    """Device log barrier vs the reference's values (CUDA's log vs numpy's: <= 4 ulp),
    plus reference tests/test_partial_ccd.py:146-160."""
    import paper_2403_19272_b200 as P

    w = P.dbb_weight(G["dbb_d"], 1e-3, 3.0)
    g = P.dbb_weight_gradient(G["dbb_d"], 1e-3, 3.0)
    np.testing.assert_allclose(w, G["dbb_w"], rtol=1e-15, atol=0)
    np.testing.assert_allclose(g, G["dbb_g"], rtol=1e-14, atol=0)
    d_hat = 1e-3
    assert P.dbb_weight(d_hat, d_hat, 1.0) == 0.0 and P.dbb_weight(2 * d_hat, d_hat, 1.0) == 0.0
    vals = P.dbb_weight(np.array([1e-7, 1e-6, 1e-5, 1e-4]), d_hat, 1.0)
    assert (np.diff(vals) < 0).all()
    assert P.dbb_weight(1e-200, d_hat, 1.0) > 50 * P.dbb_weight(1e-6, d_hat, 1.0)
    gg = P.dbb_weight_gradient(np.array([d_hat / 2]), d_hat, 1.0)
    fd = (P.dbb_weight(d_hat / 2 + 1e-9, d_hat, 1.0) - P.dbb_weight(d_hat / 2 - 1e-9, d_hat, 1.0)) / 2e-9
    assert np.isclose(gg[0], fd, rtol=1e-5)
    with pytest.raises(FloatingPointError):
        P.dbb_weight(np.array([1e-4, 0.0]), d_hat, 1.0)
    with pytest.raises(ValueError):
        P.dbb_weight(1e-4, d_hat, 0.0)


def test_lattice_samples_golden(G):
    import paper_2403_19272_b200 as P

    for dom in ("triangle", "box"):
        for iv in (0.3, 0.1):
            assert np.array_equal(P.lattice_samples(iv, dom), G[f"lattice_{dom}_{iv}"])


def test_device_sat_vs_reference_and_exact(G):
    """tri_tri_intersect on the device: the reference's float verdicts bit for bit on the
    near-degenerate mix, never a false negative against the rational SAT
    (reference tests/test_harness.py:166-181, oracles.py:51-80)."""
    import paper_2403_19272_b200 as P
    from oracle.intersect import exact_separation_margin

    p, q = G["sat_p"], G["sat_q"]
    got = P.tri_tri_intersect(p, q)
    assert np.array_equal(got, G["sat"])
    exact = G["sat_exact"]
    assert not (exact & ~got).any(), "false negative against exact arithmetic"
    for i in np.flatnonzero(got & ~exact):
        scale = float(np.abs(np.concatenate([p[i], q[i]])).max()) + 1.0
        assert exact_separation_margin(p[i], q[i]) <= 1e-12 * scale
    for i in range(0, len(p), 25):
        assert P.tri_tri_intersect_exact(p[i], q[i]) == bool(exact[i])


def test_oracle_intersect_matches_reference_counts(cuda):
    """oracle_intersect (device) on the reference's own sphere-drape states reproduces its
    per-step intersection counts (tests/golden/contact_sphere14.npz)."""
    import paper_2403_19272_b200 as P
    from paper_2403_19272_b200.scenes import scene_parts

    g = golden("contact_sphere14.npz")
    parts = scene_parts("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
    n = parts["mesh"].vertex_count
    tris = np.concatenate([parts["mesh"].triangles, np.asarray(parts["obstacles"][0][1]) + n])
    for s in range(len(g["intersections"])):
        xw = np.concatenate([g["x"][s + 1], g["obstacle_x"][s + 1]])
        assert len(P.oracle_intersect(xw, tris)) == g["intersections"][s], s


def _random_spd_system(n, rng):
    import paper_2403_19272_b200 as P

    A = rng.normal(size=(n, n)) * (rng.random((n, n)) < 0.2)
    A = A + A.T
    A = A + np.diag(np.abs(A).sum(axis=1) + 1.0)
    H = sp.csr_matrix(A)
    return P.GlobalSystem(H=H, H_fp=sp.csr_matrix((n, 0)), diag=H.diagonal().copy(), mass_over_h2=np.ones(n))


def test_smoothing_dropins(cuda, rng):
    """reference tests/test_smoothing.py:24-78: one aggregated step == two Jacobi steps
    (with and without collision diagonal and damping), diagonal systems converge,
    divergence raises SmootherDivergence."""
    import paper_2403_19272_b200 as P

    diag = np.array([2.0, 3.0, 4.0])
    system = P.GlobalSystem(H=sp.csr_matrix(np.diag(diag)), H_fp=sp.csr_matrix((3, 0)), diag=diag,
                            mass_over_h2=np.ones(3))
    b = np.array([[2.0], [6.0], [12.0]])
    assert np.allclose(P.ajacobi_smooth(system, b, np.zeros((3, 1)), iterations=2), b / diag[:, None])
    for trial in range(20):
        n = int(rng.integers(5, 60))
        system = _random_spd_system(n, rng)
        b = rng.normal(size=(n, 3))
        x0 = rng.normal(size=(n, 3))
        delta = rng.uniform(0.0, 1.0, size=n) if trial % 2 else None
        omega = 0.0 if trial % 3 else float(rng.uniform(0.1, 0.9))
        x1 = P.jacobi_step(system, b, x0, omega=omega, diag_delta=delta)
        x2 = P.jacobi_step(system, b, x1, omega=omega, diag_delta=delta)
        agg = P.ajacobi_smooth(system, b, x0, iterations=2, omega=omega, diag_delta=delta)
        assert np.abs(agg - x2).max() <= 1e-12 * max(float(np.abs(x2).max()), 1.0)
    n = 40
    A = sp.csr_matrix(np.abs(np.full((n, n), -1.0)) * -1 + np.diag(np.full(n, 2.0)))
    system = P.GlobalSystem(H=A, H_fp=sp.csr_matrix((n, 0)), diag=A.diagonal().copy(), mass_over_h2=np.ones(n))
    with pytest.raises(P.SmootherDivergence):
        P.ajacobi_smooth(system, np.ones((n, 1)), np.zeros((n, 1)), iterations=400, omega=0.0)
    with pytest.raises(ValueError):
        P.ajacobi_smooth(system, np.ones((n, 1)), np.zeros((n, 1)), iterations=2, diag_delta=np.full(n, -5.0))


def _small_system():
    import paper_2403_19272_b200 as P

    verts, tris = P.grid_cloth(6, 1.0)
    mesh = P.build_mesh(verts, tris, density=0.3, pins=np.arange(6))
    el = P.build_elastic(mesh, 160.0, 3e-4)
    return mesh, el, P.assemble_global(mesh, el, h=1.0 / 150.0)


def test_subspace_dropins(cuda, rng):
    """reference tests/test_subspace.py:104-186 and the oracle's solver stages."""
    import paper_2403_19272_b200 as P
    from oracle import solver as O

    mesh, el, system = _small_system()
    rest = mesh.rest_positions[mesh.free]
    sub = P.build_subspace(system, rest, r_bar=10, r=5)
    assert np.array_equal(P.reduced_update(sub, np.zeros(0, dtype=int), np.zeros(0)), np.zeros((5, 5)))
    got = P.reduced_update(sub, np.array([7]), np.array([2.0]))
    assert np.allclose(got, 2.0 * np.outer(sub.V[7], sub.V[7]))
    with pytest.raises(ValueError):
        P.reduced_update(sub, np.array([7]), np.array([-1.0]))
    sub8 = P.build_subspace(system, rest, r_bar=10, r=8)
    dl = rng.normal(size=(8, 8))
    dl = dl @ dl.T
    red = P.build_reduced(sub8, dl, rhs_scale=2.5)
    A = np.diag(sub8.eigenvalues_r) + dl
    rhs = rng.normal(size=(8, 3))
    sol = red.solve(rhs)
    assert np.linalg.norm(A @ sol - rhs) / np.linalg.norm(rhs) <= 1e-6
    assert np.allclose(sol, np.linalg.solve(A, rhs), atol=1e-8) and red.beta == 2.5
    # reduced_correction / warmstart_correction vs the oracle (fp64, 1e-12)
    nf = rest.shape[0]
    b = rng.normal(size=(nf, 3))
    x = rest + 0.01 * rng.normal(size=(nf, 3))
    delta = np.where(rng.random(nf) < 0.3, rng.uniform(1.0, 50.0, nf), 0.0)
    got, reduced = P.reduced_correction(sub, system, b, x, delta)
    exp = O.reduced_correction(sub, system, b, x, delta)
    exp = exp[0] if isinstance(exp, tuple) else exp
    assert np.abs(got - exp).max() <= 1e-12 * max(np.abs(exp).max(), 1.0)
    again, _ = P.reduced_correction(sub, system, b, got, delta, reduced)   # reuse within an iteration
    res0 = np.linalg.norm(b - system.H @ got - delta[:, None] * got)
    res1 = np.linalg.norm(b - system.H @ again - delta[:, None] * again)
    assert res1 <= res0 * (1 + 1e-9)
    w = P.warmstart_correction(sub, system, b, x)
    we = O.warmstart_correction(sub, system, b, x)
    assert np.abs(w - we).max() <= 1e-12 * max(np.abs(we).max(), 1.0)


def test_assemble_rhs_dropin_bitwise(cuda, rng):
    """assemble_rhs(system, mesh, elastic, z, x, pinned_positions, ...) bitwise the oracle
    (constraints.py:229-256), with pin targets that differ from x's pinned rows."""
    import paper_2403_19272_b200 as P
    from oracle import solver as O

    mesh, el, system = _small_system()
    n = mesh.vertex_count
    x = mesh.rest_positions + 0.01 * rng.normal(size=(n, 3))
    z = mesh.rest_positions + 0.01 * rng.normal(size=(n, 3))
    pins = mesh.rest_positions[mesh.pinned] + 0.02
    ids = rng.choice(n, 40)
    w = rng.uniform(0.1, 5.0, 40)
    t = rng.normal(size=(40, 3))
    for args in ((), (ids, w, t)):
        got = P.assemble_rhs(system, mesh, el, z, x, pins, *args)
        exp = O.assemble_rhs(system, mesh, el, z, x, pins, *args)
        assert np.array_equal(got[0], exp[0]) and np.array_equal(got[1], exp[1])


def test_broad_phase_dropin_equals_oracle(cuda, rng):
    """broad_phase(x0, x1, PatchBVH.build(...), margin) on the device equals the oracle's
    set (reference tests/test_bvh.py:28-105 superset + set equality)."""
    import paper_2403_19272_b200 as P
    from oracle.broad import WorldTopology, broad_phase as oracle_broad
    from oracle.stepper import Pairs

    verts, tris = P.grid_cloth(12, 0.3)
    x0 = verts + rng.normal(scale=0.01, size=verts.shape)
    x1 = x0 + rng.normal(scale=0.01, size=verts.shape)
    bvh = P.PatchBVH.build(tris, verts)
    got = P.broad_phase(x0, x1, bvh, 1e-3)
    kind, idx = oracle_broad(x0, x1, WorldTopology.build(tris, np.zeros(len(tris), bool)), 1e-3)
    a = Pairs(got.kind, got.idx).keys()
    b = Pairs(kind, idx).keys()
    assert len(a) == len(b) > 0
    assert np.array_equal(a[np.lexsort(a.T[::-1])], b[np.lexsort(b.T[::-1])])
    # far apart triangles: no pairs (reference test_bvh.py:15-25)
    far = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [10, 10, 10], [11, 10, 10], [10, 11, 10]], float)
    ft = np.array([[0, 1, 2], [3, 4, 5]])
    assert len(P.broad_phase(far, far, P.PatchBVH.build(ft, far), 1e-3)) == 0
