"""Config 3 (stacked twisted 256^2 sheets) after N steps: kernel breakdown of one step
(torch-profiler CUPTI timeline; GPU box).  python tools/twist_profile.py [N]"""
import json
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2403_19272_b200 as P  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 29
sim = P.build_scene("stacked_twist", resolution=256, config=P.StepConfig(h=1.0 / 200.0), eigensolver="device",
                    sheets=2, gap=0.005)
for _ in range(N):
    sim.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = sim.step()
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/twist.json")
ev = json.load(open("gpurun_out/twist.json"))["traceEvents"]
dev = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
by = {}
for e in dev:
    k = e["name"][:70]
    by.setdefault(k, [0, 0.0, 0.0])
    by[k][0] += 1
    by[k][1] += e["dur"]
    by[k][2] = max(by[k][2], e["dur"])
print("step", N, "timings", {k: round(v, 1) for k, v in r.timings.items()})
for k, (c, d, mx) in sorted(by.items(), key=lambda x: -x[1][1])[:15]:
    print(f"{d / 1e3:8.3f} ms {c:4d} max {mx / 1e3:7.3f}  {k}")
