"""Frame-output overhead on the config-4 skirt (GPU box): steps/s of `simulate` with a
frame every `stride` steps vs without frames.   python tools/frames_bench.py [steps] [stride]"""
import sys
import tempfile
import time

sys.path.insert(0, ".")
from paper_2403_19272_b200.cli import simulate  # noqa: E402
from paper_2403_19272_b200.sceneconfig import parse_config  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
stride = int(sys.argv[2]) if len(sys.argv) > 2 else 5
for s in (steps + 1, stride):
    with tempfile.TemporaryDirectory() as d:
        cfg = parse_config(f'name = "skirt"\nsteps = {steps}\n[scene]\nkind = "skirt"\n[solver]\nh = 0.005\n'
                           f'[output]\ndirectory = "{d}"\nframe_stride = {s}\n')
        t = time.perf_counter()
        simulate(cfg, eigensolver="device")
        print(f"frame_stride {s}: {steps} steps incl. setup {time.perf_counter() - t:.2f}s", flush=True)
