"""GPU broad phase vs the oracle: the candidate pair SET and the edge-edge
orientation must equal the reference's exactly (rows compared as sets; the
device emits them in its own deterministic order)."""

import numpy as np
import pytest

from oracle.broad import WorldTopology, broad_phase as oracle_broad

pytestmark = pytest.mark.gpu


def _rows(kind, idx):
    return {(int(k),) + tuple(int(v) for v in r) for k, r in zip(kind, idx)}


def _scene(res, obstacles, rng, jitter, move):
    import paper_2403_19272_b200 as P

    cfg = P.StepConfig()
    if obstacles:
        sim = P.build_scene("sphere_drape", resolution=res, size=1.0, config=cfg)
    else:
        sim = P.build_scene("hanging", resolution=res, config=cfg)
    st = sim.state
    xw = sim.world(st.x)
    x0 = xw + jitter * rng.normal(size=xw.shape)
    x1 = x0 + move * rng.normal(size=xw.shape)
    return sim, x0, x1


@pytest.mark.parametrize("res,obst,jitter,move,margin", [
    (6, False, 0.08, 0.15, 0.01),        # crumpled (reference tests/test_bvh.py:82-104)
    (12, True, 0.02, 0.05, 0.01),
    (24, True, 0.005, 0.01, 1e-3),
    (40, False, 0.002, 0.004, 1e-3),
])
def test_broad_phase_equals_reference_set(cuda, rng, res, obst, jitter, move, margin):
    sim, x0, x1 = _scene(res, obst, rng, jitter, move)
    got = sim.broad_phase(x0, x1, margin)
    topo = WorldTopology.build(sim.world_triangles, sim.tri_static)
    k_ref, i_ref = oracle_broad(x0, x1, topo, margin)
    assert len(got) == len(k_ref)
    assert _rows(got.kind, got.idx) == _rows(k_ref, i_ref)        # includes EE orientation
    assert len(_rows(got.kind, got.idx)) == len(got)                # no duplicates


def test_broad_phase_far_apart_empty(cuda):
    import paper_2403_19272_b200 as P

    verts = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0],
                      [100.0, 0.0, 0.0], [101.0, 0.0, 0.0], [100.0, 1.0, 0.0]])
    mesh = P.build_mesh(verts, np.array([[0, 1, 2], [3, 4, 5]]), 0.3)
    sim = P.Simulation(mesh, P.StepConfig(r_bar=4, r=2))
    assert len(sim.broad_phase(verts, verts, 1e-3)) == 0
