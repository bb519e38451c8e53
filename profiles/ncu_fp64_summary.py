"""Summarise an ncu raw CSV (profiles/run_ncu_fp64.sh) into a per-kernel roofline table.

    python profiles/ncu_fp64_summary.py gpurun_out/ncu_fp64.csv gpurun_out/fp64_peak.json > profiles/rN_kernel_roofs.md

Per kernel (aggregated over its launches in one bench step):
  * time, DRAM bytes (read + write), achieved DRAM GB/s and fraction of the
    measured HBM peak (MEASURED_PEAKS.json, else 6,542 GB/s);
  * FP64 FLOP = 2 * DFMA + DADD + DMUL thread instructions (predicated on),
    achieved TFLOP/s and fraction of the measured FP64 peak (tools/fp64_peak.cu);
  * FP64 pipe utilisation and SM issue utilisation (ncu's own counters: these
    include DSETP / conversions / MUFU-assisted sqrt & divide sequences that the
    FLOP count omits);
  * the binding roof = the larger of the DRAM fraction and the FP64-pipe
    fraction, and the top warp-stall reasons (cycles per issued instruction).
"""

from __future__ import annotations

import csv
import json
import os
import sys
from collections import OrderedDict

STALLS = ["long_scoreboard", "short_scoreboard", "wait", "math_pipe_throttle", "mio_throttle", "lg_throttle",
          "not_selected", "branch_resolving", "dispatch_stall", "no_instruction", "barrier", "membar", "drain",
          "tex_throttle", "sleeping", "misc"]


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    head = rows[0]
    col = {c: i for i, c in enumerate(head)}
    out = []
    for r in rows[2:]:
        def g(name, default=0.0):
            i = col.get(name)
            if i is None or i >= len(r) or r[i] in ("", "n/a"):
                return default
            try:
                return float(r[i].replace(",", ""))
            except ValueError:
                return default
        name = r[col["Kernel Name"]].split("(")[0].strip()
        if name.startswith("void "):
            name = name[5:]
        name = name.replace("cs::", "")
        d = {
            "name": name,
            "ns": g("gpu__time_duration.sum"),
            "dram": g("dram__bytes_read.sum") + g("dram__bytes_write.sum"),
            "dfma": g("sm__sass_thread_inst_executed_op_dfma_pred_on.sum"),
            "dadd": g("sm__sass_thread_inst_executed_op_dadd_pred_on.sum"),
            "dmul": g("sm__sass_thread_inst_executed_op_dmul_pred_on.sum"),
            "fp64_pipe": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue": g("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
            "dram_pct": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "occ": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "stalls": {s: g(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio") for s in STALLS},
        }
        out.append(d)
    return out


def main():
    csv_path = sys.argv[1]
    peak_path = sys.argv[2] if len(sys.argv) > 2 else None
    fp64_peak = 34.1
    if peak_path and os.path.exists(peak_path):
        fp64_peak = json.load(open(peak_path))["fp64_tflops"]
    hbm_peak = 6542.4
    mp = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        try:
            m = json.load(open(mp))
            for k in ("hbm_copy_gbps", "hbm_gbps", "hbm_burst_gbps"):
                if k in m:
                    hbm_peak = float(m[k])
                    break
        except Exception:
            pass
    launches = [d for d in load(csv_path) if not d["name"].startswith("k_blk_")]  # setup eigensolver
    agg: "OrderedDict[str, dict]" = OrderedDict()
    for d in launches:
        a = agg.setdefault(d["name"], {"n": 0, "ns": 0.0, "dram": 0.0, "flop": 0.0, "w_pipe": 0.0, "w_issue": 0.0,
                                       "w_occ": 0.0, "stalls": {s: 0.0 for s in STALLS}})
        a["n"] += 1
        a["ns"] += d["ns"]
        a["dram"] += d["dram"]
        a["flop"] += 2 * d["dfma"] + d["dadd"] + d["dmul"]
        a["w_pipe"] += d["fp64_pipe"] * d["ns"]
        a["w_issue"] += d["issue"] * d["ns"]
        a["w_occ"] += d["occ"] * d["ns"]
        for s in STALLS:
            a["stalls"][s] += d["stalls"][s] * d["ns"]
    total = sum(a["ns"] for a in agg.values())
    rows = sorted(agg.items(), key=lambda kv: -kv[1]["ns"])
    print(f"# Per-kernel roofs, one config-4 skirt bench step (ncu, cold L2, serialised)\n")
    print(f"Source: `{os.path.basename(csv_path)}` ({len(launches)} launches, {total / 1e6:.2f} ms summed). "
          f"HBM peak {hbm_peak:,.0f} GB/s (MEASURED_PEAKS.json copy bandwidth); FP64 peak {fp64_peak:.1f} TFLOP/s "
          f"(measured, `tools/fp64_peak.cu`: independent DFMA chains, all SMs). FLOP = 2·DFMA + DADD + DMUL "
          f"(thread instructions). `pipe` = ncu FP64-pipe utilisation (includes the DSETP / conversion / "
          f"sqrt / divide sequences the FLOP count leaves out). Bound = the roof with the larger fraction; "
          f"stalls = cycles per issued instruction (top three).\n")
    print("| kernel | launches | µs total | share | DRAM MB | GB/s | HBM frac | GFLOP | TFLOP/s | FP64 frac | "
          "FP64 pipe % | issue % | occ % | bound | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for name, a in rows:
        t = a["ns"] * 1e-9
        gbs = a["dram"] / t / 1e9 if t > 0 else 0.0
        tfl = a["flop"] / t / 1e12 if t > 0 else 0.0
        pipe = a["w_pipe"] / a["ns"] if a["ns"] else 0.0
        issue = a["w_issue"] / a["ns"] if a["ns"] else 0.0
        occ = a["w_occ"] / a["ns"] if a["ns"] else 0.0
        hf = gbs / hbm_peak
        ff = tfl / fp64_peak
        if max(hf, pipe / 100) < 0.3:
            bound = "latency" if issue < 50 else "issue"
        else:
            bound = "HBM" if hf >= pipe / 100 else "FP64 pipe"
        st = {s: v / a["ns"] for s, v in a["stalls"].items()} if a["ns"] else {}
        top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        tops = ", ".join(f"{k} {v:.1f}" for k, v in top)
        print(f"| `{name}` | {a['n']} | {a['ns'] / 1e3:,.1f} | {a['ns'] / total:.1%} | {a['dram'] / 1e6:,.1f} | "
              f"{gbs:,.0f} | {hf:.2f} | {a['flop'] / 1e9:,.2f} | {tfl:.2f} | {ff:.2f} | {pipe:.0f} | {issue:.0f} | "
              f"{occ:.0f} | {bound} | {tops} |")


if __name__ == "__main__":
    main()
