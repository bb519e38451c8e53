"""Batch (config 5) end-to-end overhead probe (GPU box): device-timed steps vs the same
steps with each scene's state read back, over the multi-stream Stepper.
    python tools/batch_e2e_probe.py [scenes] [steps]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

scenes = int(sys.argv[1]) if len(sys.argv) > 1 else 16
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sys.argv = [sys.argv[0], "--workload", "batch", "--batch-scenes", str(scenes)]
args = bench.parse()
sims, _ = bench.make_scenes(args, 0, 1)
st = bench.Stepper(sims, args.streams)
st.run(2)
torch.cuda.synchronize()
snap = [(s.host_state(), np.array(s.obstacle_x, copy=True)) for s in sims]
for label, cb in (("no readback", None), ("state.x readback", lambda s: s.state.x), ("no readback", None),
                  ("state.x readback", lambda s: s.state.x)):
    for s, (x, ob) in zip(sims, snap):   # the same steps every time
        s.state = x
        s.obstacle_x = ob
        s._flush()
    torch.cuda.synchronize()
    t = time.perf_counter()
    st.run(steps, on_step=cb)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{label}: {scenes * steps / dt:.1f} scene-steps/s", flush=True)
