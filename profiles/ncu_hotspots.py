"""Top warp-stall SASS lines of one kernel in an ncu report, mapped to source lines.

    python profiles/ncu_hotspots.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
ai, si = h.index("Address"), h.index("Source")
wi = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed") if "Instructions Executed" in h else None
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
def f(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


tot = sum(f(r[wi]) for r in data) or 1.0
print(f"{rep}: {len(data)} SASS lines, {tot:.0f} stall samples")
for r in sorted(data, key=lambda r: -f(r[wi]))[:top]:
    print(f"{f(r[wi]) / tot:6.1%}  {r[si][:90]}")
