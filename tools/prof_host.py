import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch
import paper_2403_19272_b200 as P
from paper_2403_19272_b200 import scenes as S
sim = S.skirt_scene(P.StepConfig(h=1.0 / 200.0), around=584, down=584, eigensolver="device")
for _ in range(3): sim.step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10): sim.step()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(25)
