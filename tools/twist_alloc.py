import sys, time, torch
sys.path.insert(0, ".")
import paper_2403_19272_b200 as P
sim = P.build_scene("stacked_twist", resolution=256, sheets=2, gap=0.005, config=P.StepConfig(h=1.0/200.0), eigensolver="device")
for i in range(30):
    torch.cuda.synchronize(); t = time.perf_counter(); r = sim.step(); torch.cuda.synchronize()
    print(f"[step] {i} {1e3*(time.perf_counter()-t):.1f} ms rf={r.rf_triggered} lg={r.lg_iterations} outer={r.outer_loops}", file=sys.stderr, flush=True)
