"""Same K skirt steps timed twice from one snapshot (first-execution effects; GPU box)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_19272_b200 as P  # noqa: E402
from paper_2403_19272_b200 import scenes as S  # noqa: E402

sim = S.skirt_scene(P.StepConfig(h=1.0 / 200.0), around=584, down=584, eigensolver="device")
for _ in range(3):
    sim.step()
torch.cuda.synchronize()
st, ob = sim.host_state(), np.array(sim.obstacle_x, copy=True)
for rep in range(3):
    sim.state = st
    sim.obstacle_x = ob
    sim._flush()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    stages = []
    for _ in range(20):
        r = sim.step()
        stages.append(r.timings)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    nf = [t["narrow_full"] for t in stages]
    print(f"pass {rep}: {ms:.2f} ms/step, narrow_full mean {np.mean(nf):.2f} max {np.max(nf):.2f} "
          f"argmax {int(np.argmax(nf))}", flush=True)
