"""Diagnostic: device broad phase vs the oracle set along a simulated trajectory (GPU box)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2403_19272_b200 as P  # noqa: E402
from oracle.broad import WorldTopology, broad_phase as oracle_broad  # noqa: E402
from oracle.intersect import intersecting_pairs  # noqa: E402


def rows(kind, idx):
    return {(int(k),) + tuple(int(v) for v in r) for k, r in zip(kind, idx)}


sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
topo = WorldTopology.build(sim.world_triangles, sim.tri_static)
prev = sim.world(sim.state.x)
for s in range(25):
    sim.step()
    cur = sim.world(sim.state.x)
    got = sim.broad_phase(prev, cur, sim.config.d_hat)
    k, i = oracle_broad(prev, cur, topo, sim.config.d_hat)
    a, b = rows(got.kind, got.idx), rows(k, i)
    bad = intersecting_pairs(cur, sim.bvh.triangles)
    print(s, len(got), len(k), "missing", len(b - a), "extra", len(a - b), "dups", len(got) - len(a),
          "intersections", len(bad), flush=True)
    if b - a:
        print("  missing sample", sorted(b - a)[:5])
    prev = cur
