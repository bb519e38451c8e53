import sys
sys.path.insert(0, ".")
import paper_2403_19272_b200 as P
from paper_2403_19272_b200 import scenes as S
sim = S.skirt_scene(P.StepConfig(h=1.0 / 200.0), around=584, down=584, eigensolver="device")
for k in range(4):
    print(f"=== step {k}", file=sys.stderr, flush=True)
    sim.step()
