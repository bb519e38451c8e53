"""Skirt (config 4) in the paper's solver regime (eps 1e-9, 67 LG iterations): 4 default
steps, one untimed paper-regime step, then `--steps` more (for ncu / nsight captures of
the per-iteration kernels; GPU box)."""
import dataclasses
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_19272_b200 as P  # noqa: E402
from paper_2403_19272_b200 import scenes as S  # noqa: E402

steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1
cfg = P.StepConfig(h=1.0 / 200.0)
sim = S.skirt_scene(cfg, around=584, down=584, eigensolver="device")
for _ in range(4):
    sim.step()
sim.config = dataclasses.replace(cfg, eps_inner=1e-9, eps_outer=1e-9, iteration_cap=67)
sim.step()
torch.cuda.synchronize()
for _ in range(steps):
    r = sim.step()
    c = sim.last_report_c
    print("lg", r.lg_iterations, "outer", r.outer_loops, "reuses", c.stamp_plan_reuses, "reduced_fallbacks",
          c.reduced_fallbacks, "host_syncs", c.host_syncs, flush=True)
torch.cuda.synchronize()
