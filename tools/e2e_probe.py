import sys, time
sys.path.insert(0, ".")
import torch
import paper_2403_19272_b200 as P
from paper_2403_19272_b200 import scenes as S
sim = S.skirt_scene(P.StepConfig(h=1/200), around=584, down=584, eigensolver="device")
for _ in range(4): sim.step()
torch.cuda.synchronize()
t_step, t_x = [], []
for _ in range(8):
    t0 = time.perf_counter(); sim.step(); torch.cuda.synchronize(); t1 = time.perf_counter()
    x = sim.state.x; t2 = time.perf_counter()
    t_step.append(t1 - t0); t_x.append(t2 - t1)
print("step ms", [round(1e3*v,2) for v in t_step]); print("state.x ms", [round(1e3*v,2) for v in t_x])
t0=time.perf_counter()
for _ in range(20): sim._pin_targets(0.1); sim._obstacle_targets(0.1)
print("targets ms", (time.perf_counter()-t0)/20*1e3)
