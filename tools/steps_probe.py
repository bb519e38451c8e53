import sys, time, torch
sys.path.insert(0, ".")
import paper_2403_19272_b200 as P
kind = sys.argv[1] if len(sys.argv) > 1 else "sphere_drape"
res = int(sys.argv[2]) if len(sys.argv) > 2 else 317
kw = {"sheets": 2, "gap": 0.005} if kind == "stacked_twist" else {}
sim = P.build_scene(kind, resolution=res, config=P.StepConfig(h=1.0/200.0), eigensolver="device", **kw)
out = []
for i in range(30):
    torch.cuda.synchronize(); t = time.perf_counter(); r = sim.step(); torch.cuda.synchronize()
    out.append((i, round(1e3*(time.perf_counter()-t),1), round(r.timings["broad"],1), r.outer_loops, sim.last_report_c.subset_sites))
print(out)
print("mean ms over steps 1..:", round(sum(o[1] for o in out[1:]) / (len(out) - 1), 2))
