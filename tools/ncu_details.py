"""Key metrics of `ncu --page details --csv` exports (one kernel each)."""
import csv
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Achieved Occupancy",
        "Registers Per Thread", "Grid Size", "Block Size", "Theoretical Occupancy", "Issue Slots Busy",
        "Compute (SM) Throughput", "L2 Cache Throughput"]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    h = rows[0]
    ni, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    seen = {}
    for r in rows[1:]:
        if len(r) > vi and r[ni] in WANT and r[ni] + r[ui] not in seen:
            seen[r[ni] + r[ui]] = f"{r[ni]} {r[vi]} {r[ui]}"
    print(path + ": " + "; ".join(seen.values()))
