"""Per-pair cost of the REAL reference broad phase (patch BVH, collision/bvh.py:207-292)
against the oracle port's grid-hash join (oracle/broad.py), same worlds, same
positions, one host thread -- the factor the CPU baseline applies to the port's
broad-phase time so the reference arm reflects the reference's stock code path.

Build container only (imports /root/reference):

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 python tools/calibrate_broad.py

Writes profiles/broad_calibration.json (committed; bench.py reads it).
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("CLOTHSIM_REF", "/root/reference/pkg/src"))

from clothsim.collision import PatchBVH, broad_phase as ref_broad  # noqa: E402

from oracle.broad import WorldTopology, broad_phase as port_broad  # noqa: E402
from paper_2403_19272_b200.scenes import grid_cloth, skirt_parts  # noqa: E402


def timed(fn, reps=2):
    best = float("inf")
    out = None
    for _ in range(reps):
        t = time.perf_counter()
        out = fn()
        best = min(best, time.perf_counter() - t)
    return best, out


def world_cases():
    # BASELINE config 1 world: the 64^2 sheet (flat, 1 cm motion)
    v, t = grid_cloth(64, 1.0)
    yield "config1_grid64", v, v + np.array([0.0, 0.0, -0.01]), t, np.zeros(len(t), bool)
    # a band of the config-4 skirt (bench spacing: 1.03 mm rows) on its body, one step of spin
    p = skirt_parts(around=584, down=24, length=0.6 * 23 / 583)
    cv = p["mesh"].rest_positions
    bv, bt = p["obstacles"][0]
    x0 = np.concatenate([cv, bv])
    ang = np.pi / 200.0
    rot = np.array([[np.cos(ang), -np.sin(ang), 0.0], [np.sin(ang), np.cos(ang), 0.0], [0.0, 0.0, 1.0]])
    x1 = x0 @ rot.T
    tris = np.concatenate([p["mesh"].triangles, bt + len(cv)])
    stat = np.zeros(len(tris), bool)
    stat[len(p["mesh"].triangles):] = True
    yield "skirt_band_584x24", x0, x1, tris, stat


def main():
    d_hat = 1e-3
    cases = []
    for name, x0, x1, tris, stat in world_cases():
        bvh = PatchBVH.build(tris, x0, stat)
        topo = WorldTopology.build(tris, stat)
        t_ref, pr = timed(lambda: ref_broad(x0, x1, bvh, d_hat))
        t_port, (kind, idx) = timed(lambda: port_broad(x0, x1, topo, d_hat))
        assert len(kind) == len(pr.kind), (name, len(kind), len(pr.kind))
        cases.append({"world": name, "pairs": int(len(kind)), "reference_s": t_ref, "port_s": t_port,
                      "reference_us_per_pair": 1e6 * t_ref / max(len(kind), 1),
                      "port_us_per_pair": 1e6 * t_port / max(len(kind), 1), "factor": t_ref / t_port})
        print(cases[-1], flush=True)
    out = {"what": "reference patch-BVH broad phase time / oracle grid-join broad phase time, same inputs, "
                   "1 host thread (OPENBLAS_NUM_THREADS=1)",
           "factor": float(np.exp(np.mean([np.log(c["factor"]) for c in cases]))),
           "factor_max": max(c["factor"] for c in cases), "cases": cases,
           "host": platform.processor() or platform.machine(), "script": "tools/calibrate_broad.py"}
    with open(os.path.join(ROOT, "profiles", "broad_calibration.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
