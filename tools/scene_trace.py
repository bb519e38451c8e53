"""Per-step trace for a BASELINE config scene (diagnostic, GPU box).

    python tools/scene_trace.py sphere_ground 128 40
    python tools/scene_trace.py stacked_twist 256 40
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2403_19272_b200 as P  # noqa: E402

kind, res, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = P.StepConfig(h=1.0 / 200.0)
kw = {"sheets": 2, "gap": 0.005} if kind == "stacked_twist" else {}
if kind == "sphere_drape":      # BASELINE config 5 scene (317^2 drape, material 0)
    kw = {}
t0 = time.time()
sim = P.build_scene(kind, resolution=res, config=cfg, eigensolver="device", **kw)
print("setup_s", round(time.time() - t0, 1), "verts", sim.mesh.vertex_count, flush=True)
tot = 0.0
for i in range(steps):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = sim.step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    tot += dt
    c = sim.last_report_c
    if i % 5 == 4 or i < 3:
        print(json.dumps({"step": i, "ms": round(1e3 * dt, 2), "lg": r.lg_iterations, "outer": r.outer_loops,
                          "rf": r.rf_triggered, "toi": round(r.toi_exit, 4), "active": r.active_pairs,
                          "pairs": c.pairs_max_site, "stages": {k: round(v, 2) for k, v in r.timings.items()}}),
              flush=True)
print("mean ms/step", round(1e3 * tot / steps, 2), "FPS", round(steps / tot, 1))
print("intersecting pairs at end:", len(sim.intersecting_pairs()))
