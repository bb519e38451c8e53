"""Micro-benchmark of the A-Jacobi smoother (the roofline kernel) on the config-4
skirt: CUDA-event time per SpMV pass, algorithmic GB/s (diagnostic, GPU box)."""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2403_19272_b200 as P  # noqa: E402
from paper_2403_19272_b200 import _lib, scenes as S  # noqa: E402

if len(sys.argv) > 1:  # optional: a specific build of the library (A/B)
    _lib.load(sys.argv[1])

cfg = P.StepConfig(h=1.0 / 200.0)
sim = S.skirt_scene(cfg, around=584, down=584, eigensolver="device")
nf = sim.mesh.free.size
nnz = sim.system.H.nnz
rng = np.random.default_rng(0)
b = torch.as_tensor(rng.standard_normal((nf, 3)), device="cuda")
x = torch.as_tensor(rng.standard_normal((nf, 3)) * 1e-3, device="cuda")
dl = torch.zeros(nf, dtype=torch.float64, device="cuda")
lib = sim._lib
st = torch.cuda.current_stream()
h = ctypes.c_void_p(st.cuda_stream)
for _ in range(3):
    lib.cs_ajacobi_smooth(sim._scene, b.data_ptr(), x.data_ptr(), 32, 0.0, dl.data_ptr(), h)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 50
e0.record(st)
for _ in range(reps):
    rc = lib.cs_ajacobi_smooth(sim._scene, b.data_ptr(), x.data_ptr(), 32, 0.0, dl.data_ptr(), h)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
per_pass = ms / 32 * 1e3
bytes_pass = 12.0 * nnz + 88.0 * nf
print(json.dumps({"ms_per_smooth32": ms, "us_per_pass": per_pass, "GBps": bytes_pass / (per_pass * 1e-6) / 1e9,
                  "nnz": nnz, "nf": nf, "rc": rc}))
