"""Kernel breakdown of the slow late steps of BASELINE config 3 (GPU box)."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2403_19272_b200 as P  # noqa: E402

sim = P.build_scene("stacked_twist", resolution=256, sheets=2, gap=0.005, config=P.StepConfig(h=1.0 / 200.0),
                    eigensolver="device")
for _ in range(27):
    sim.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        sim.step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
