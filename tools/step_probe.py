import sys, time
sys.path.insert(0, ".")
import torch
import paper_2403_19272_b200 as P
from paper_2403_19272_b200 import scenes as S
sim = S.skirt_scene(P.StepConfig(h=1.0 / 200.0), around=584, down=584, eigensolver="device")
for k in range(12):
    print(f"=== step {k}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    r = sim.step()
    torch.cuda.synchronize()
    c = sim.last_report_c
    print(f"=== step {k} done {1e3*(time.perf_counter()-t0):.1f} ms rf {r.rf_triggered} outer {r.outer_loops} lg {r.lg_iterations} "
          f"lazy {c.lazy_exit_sites} static {c.static_sites} subset {c.subset_sites} nf {r.timings['narrow_full']:.1f} "
          f"toi {r.toi_exit:.3g}", file=sys.stderr, flush=True)
