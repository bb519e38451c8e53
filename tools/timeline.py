"""Device timeline of a few steps via torch.profiler (CUPTI): busy vs idle time,
largest idle gaps and what precedes them (diagnostic, GPU box)."""
import json
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2403_19272_b200 as P  # noqa: E402
from paper_2403_19272_b200 import scenes as S  # noqa: E402

import dataclasses  # noqa: E402

PAPER = "--paper" in sys.argv   # eps 1e-9, 67 LG iterations (bench.py paper_regime)
TAG = "_paper" if PAPER else ""
cfg = P.StepConfig(h=1.0 / 200.0)
sim = S.skirt_scene(cfg, around=584, down=584, eigensolver="device")
for _ in range(4):
    sim.step()
if PAPER:
    sim.config = dataclasses.replace(cfg, eps_inner=1e-9, eps_outer=1e-9, iteration_cap=67)
    sim.step()  # buffers of the 67-iteration regime sized once, outside the profile
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(int(__import__("os").environ.get("TL_STEPS", "1")) if PAPER else 2):
        sim.step()
    torch.cuda.synchronize()
prof.export_chrome_trace(f"gpurun_out/timeline{TAG}.json")
ev = json.load(open(f"gpurun_out/timeline{TAG}.json"))["traceEvents"]
dev = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
dev.sort(key=lambda e: e["ts"])
t0, t1 = dev[0]["ts"], max(e["ts"] + e["dur"] for e in dev)
busy = sum(e["dur"] for e in dev)
print(f"window {(t1 - t0) / 1e3:.2f} ms, device busy {busy / 1e3:.2f} ms, events {len(dev)}")
by = {}
for e in dev:
    k = e["cat"] + ":" + e["name"][:60]
    by.setdefault(k, [0, 0.0])
    by[k][0] += 1
    by[k][1] += e["dur"]
for k, (c, d) in sorted(by.items(), key=lambda x: -x[1][1])[:70]:
    print(f"{d / 1e3:8.3f} ms {c:5d}  {k}")
gaps = []
end = dev[0]["ts"] + dev[0]["dur"]
prev = dev[0]
for e in dev[1:]:
    if e["ts"] > end:
        gaps.append((e["ts"] - end, prev["name"][:50], e["name"][:50]))
    if e["ts"] + e["dur"] > end:
        end = e["ts"] + e["dur"]
        prev = e
gaps.sort(reverse=True)
print(f"idle total {sum(g[0] for g in gaps) / 1e3:.2f} ms in {len(gaps)} gaps; largest:")
for g in gaps[:25]:
    print(f"  {g[0]:8.1f} us after {g[1]} -> before {g[2]}")
cpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"]
byc = {}
for e in cpu:
    byc.setdefault(e["name"], [0, 0.0])
    byc[e["name"]][0] += 1
    byc[e["name"]][1] += e["dur"]
print("host CUDA runtime calls:")
for k, (c, d) in sorted(byc.items(), key=lambda x: -x[1][1])[:12]:
    print(f"{d / 1e3:8.3f} ms {c:5d}  {k}")

# host runtime calls overlapping the two largest device gaps
gl = []
end = dev[0]["ts"] + dev[0]["dur"]
for e in dev[1:]:
    if e["ts"] > end:
        gl.append((e["ts"] - end, end, e["ts"]))
    end = max(end, e["ts"] + e["dur"])
gl.sort(reverse=True)
for g, a, b in gl[:2]:
    print(f"gap {g:.1f} us [{a:.1f}, {b:.1f}]: host events inside")
    for e in sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("cuda_runtime", "cpu_op", "python_function")
                     and e["ts"] + e.get("dur", 0) >= a and e["ts"] <= b], key=lambda e: e["ts"])[:40]:
        print(f"    {e['ts'] - a:9.1f} +{e.get('dur', 0):8.1f}  {e.get('cat')}: {e['name'][:80]}")

# per-launch durations of kernels named in TL_KERNELS (comma-separated substrings)
import os  # noqa: E402
for sub in filter(None, os.environ.get("TL_KERNELS", "").split(",")):
    sel = [(k, e) for k, e in enumerate(dev) if sub in e["name"]]
    print(f"{sub}: " + ", ".join(f"{e['dur']:.0f}us g{e.get('args', {}).get('grid', ['?'])[0]} "
                                 f"(after {dev[k - 1]['name'][:28] if k else '-'})" for k, e in sel))
