import sys, time, torch
sys.path.insert(0, ".")
import paper_2403_19272_b200 as P
sim = P.build_scene("sphere_drape", resolution=317, config=P.StepConfig(h=1.0/200.0), eigensolver="device")
out = []
for i in range(30):
    torch.cuda.synchronize(); t = time.perf_counter(); r = sim.step(); torch.cuda.synchronize()
    out.append((i, round(1e3*(time.perf_counter()-t),1), round(r.timings["broad"],1), r.outer_loops, sim.last_report_c.subset_sites))
print(out)
