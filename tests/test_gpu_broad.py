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


def _brute_set(x0, x1, tris, tri_static, margin):
    """Reference set semantics by brute force (reference tests/test_bvh.py:44-80)."""
    vlo = np.minimum(x0, x1) - margin
    vhi = np.maximum(x0, x1) + margin
    tris = np.asarray(tris)
    stack = np.sort(np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]]), axis=1)
    edges, inv = np.unique(stack, axis=0, return_inverse=True)
    estat = np.zeros(len(edges), bool)
    estat[inv.reshape(3, -1).T[tri_static].ravel()] = True
    vstat = np.ones(len(x0), bool)
    vstat[tris[~tri_static].ravel()] = False
    used = np.zeros(len(x0), bool)
    used[tris.ravel()] = True
    tlo, thi = vlo[tris].min(axis=1), vhi[tris].max(axis=1)
    elo, ehi = vlo[edges].min(axis=1), vhi[edges].max(axis=1)
    out = set()
    ov = ((vlo[:, None] <= thi[None]) & (tlo[None] <= vhi[:, None])).all(axis=2)
    for v, f in zip(*np.nonzero(ov)):
        if used[v] and v not in tris[f] and not (vstat[v] and tri_static[f]):
            out.add((0, int(v)) + tuple(sorted(int(z) for z in tris[f])))
    oe = ((elo[:, None] <= ehi[None]) & (elo[None] <= ehi[:, None])).all(axis=2)
    for a, b in zip(*np.nonzero(oe)):
        if a < b and not set(edges[a]) & set(edges[b]) and not (estat[a] and estat[b]):
            out.add((1,) + tuple(sorted([tuple(int(z) for z in edges[a]), tuple(int(z) for z in edges[b])])))
    return out


def _canon(kind, idx):
    out = set()
    for k, r in zip(kind, idx):
        r = [int(z) for z in r]
        if k == 0:
            out.add((0, r[0]) + tuple(sorted(r[1:])))
        else:
            out.add((1,) + tuple(sorted([tuple(sorted(r[:2])), tuple(sorted(r[2:]))])))
    return out


def test_broad_phase_oversize_primitives(cuda, rng):
    """Giant obstacle faces and a vertex swept tens of metres span more grid cells than
    the hash grid enters; the brute-force side must still produce exactly the set."""
    import paper_2403_19272_b200 as P

    verts, tris = P.grid_cloth(8, 0.05)
    ground = np.array([[-100.0, -100.0, -0.002], [100.0, -100.0, -0.002], [100.0, 100.0, -0.002],
                       [-100.0, 100.0, -0.002]])
    gtris = np.array([[0, 1, 2], [0, 2, 3]])
    sim = P.Simulation(P.build_mesh(verts, tris, 0.3), P.StepConfig(r_bar=8, r=4), obstacles=[(ground, gtris)])
    x0 = sim.world(sim.state.x)
    x1 = x0 + 1e-4 * rng.normal(size=x0.shape)
    x1[len(verts) // 2] += np.array([50.0, 3.0, 0.0])   # one vertex sweeps 50 m
    got = sim.broad_phase(x0, x1, 1e-3)
    ref = _brute_set(x0, x1, sim.world_triangles, sim.tri_static, 1e-3)
    assert len(got) == len(ref)
    assert _canon(got.kind, got.idx) == ref


def test_broad_phase_dense_pile(cuda, rng):
    """A cloth crumpled into a 2 cm ball: every grid cell holds hundreds of entries
    (bucket runs beyond the shared-memory staging cap take the long-run path)."""
    import paper_2403_19272_b200 as P

    sim = P.build_scene("hanging", resolution=16, config=P.StepConfig())
    xw = sim.world(sim.state.x)
    x0 = 0.02 * rng.random(size=xw.shape)
    x1 = x0 + 0.005 * rng.normal(size=xw.shape)
    got = sim.broad_phase(x0, x1, 1e-3)
    topo = WorldTopology.build(sim.world_triangles, sim.tri_static)
    k_ref, i_ref = oracle_broad(x0, x1, topo, 1e-3)
    assert len(got) == len(k_ref) > 100_000
    assert _rows(got.kind, got.idx) == _rows(k_ref, i_ref)
