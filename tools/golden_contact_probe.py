"""Per-step comparison against the reference's own 25-step sphere drape
(tests/golden/contact_sphere14.npz), teacher forced (diagnostic, GPU box)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2403_19272_b200 as P  # noqa: E402
from conftest import golden  # noqa: E402

g = golden("contact_sphere14.npz")
sim = P.build_scene("sphere_drape", resolution=14, size=0.2, config=P.StepConfig())
for s in range(25):
    sim.state = P.SimState(x=g["x"][s], x_dot=g["x_dot"][s], x_prev=g["x_prev"][s], delta_f=g["delta_f"][s],
                           step_index=s)
    sim.obstacle_x = g["obstacle_x"][s]
    try:
        r = sim.step()
    except Exception as e:  # noqa: BLE001
        print(s, "raised", type(e).__name__)
        continue
    err = float(np.abs(sim.state.x - g["x"][s + 1]).max())
    print(f"{s:2d} err {err:.2e} lg {r.lg_iterations}/{g['lg'][s]} rf {int(r.rf_triggered)}/{int(g['rf'][s])} "
          f"toi {r.toi_exit:.17g} / {g['toi'][s]:.17g}")
