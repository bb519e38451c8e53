"""Summarise ncu reports / launch lists into profiles/*.md (run in the build container).

    python profiles/ncu_summary.py launches gpurun_out/launches.csv
    python profiles/ncu_summary.py full gpurun_out/full_k_query_ee.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Compute (SM) Throughput", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Branch Efficiency", "Executed Ipc Active", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Static Shared Memory Per Block", "Waves Per SM")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__inst_executed_pipe_fp64.sum",
       "smsp__sass_inst_executed_op_global_ld.sum", "lts__t_bytes.sum")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "").replace("cs::", "")
        if name.startswith("k_blk_"):  # setup eigensolver kernels
            continue
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    print("| kernel | launches | total ms | share | avg us |")
    print("|---|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:70]}` | {c} | {t / 1e3:.3f} | {100 * t / tot:.1f}% | {t / c:.1f} |")
    print(f"\ntotal kernel time {tot / 1e3:.3f} ms over the profiled steps")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    name = rows[1][h.index("Kernel Name")]
    print(f"kernel: `{name.split('(')[0]}`  block {rows[1][h.index('Block Size')]} grid {rows[1][h.index('Grid Size')]}")
    seen = set()
    for r in rows[1:]:
        m = r[h.index("Metric Name")]
        if m in KEYS and m not in seen:
            seen.add(m)
            print(f"- {m}: {r[h.index('Metric Value')]} {r[h.index('Metric Unit')]}")
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    for i, m in enumerate(h):
        if m in RAW or m.startswith("smsp__pcsamp_warps_issue_stalled") and not m.endswith("not_issued"):
            try:
                if float(vals[i].replace(",", "")) == 0:
                    continue
            except ValueError:
                pass
            print(f"- {m}: {vals[i]} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
