"""A/B step time of the config-4 skirt for two builds of the library (diagnostic, GPU box).
usage: python tools/ab_step.py LIB.so [steps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2403_19272_b200 as P  # noqa: E402
from paper_2403_19272_b200 import _lib  # noqa: E402
from paper_2403_19272_b200 import scenes as S  # noqa: E402

_lib.load(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
sim = S.skirt_scene(P.StepConfig(h=1.0 / 200.0), around=584, down=584, eigensolver="device")
for _ in range(4):
    sim.step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(steps):
    sim.step()
b.record()
torch.cuda.synchronize()
print(f"{sys.argv[1]}: {a.elapsed_time(b) / steps:.3f} ms/step")
