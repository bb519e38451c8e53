"""Per-step trace of one scene: wall time, stage ms, counters (diagnostic, GPU box)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2403_19272_b200 as P  # noqa: E402
from paper_2403_19272_b200 import scenes as S  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "skirt"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = P.StepConfig(h=1.0 / 200.0)
if which == "skirt":
    sim = S.skirt_scene(cfg, around=584, down=584, eigensolver="device")
else:
    sim = P.build_scene(which, resolution=int(sys.argv[3]) if len(sys.argv) > 3 else 64, config=cfg)
for i in range(steps):
    print(f"--- step {i}", file=sys.stderr, flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = sim.step()
    torch.cuda.synchronize()
    c = sim.last_report_c
    print(json.dumps({"step": i, "wall_ms": round(1e3 * (time.perf_counter() - t0), 2),
                      "stages": {k: round(v, 2) for k, v in r.timings.items()},
                      "lg": r.lg_iterations, "outer": r.outer_loops, "sites": r.full_ccd_calls,
                      "pairs_max": c.pairs_max_site, "active": r.active_pairs, "rf": r.rf_triggered,
                      "toi_exit": r.toi_exit, "launches": c.gpu_launches}), flush=True)
