"""Per-CUDA-source-line summary of an ncu report (--page source --print-source
cuda,sass --csv): warp-stall samples and executed warp instructions per line.

usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv
       python scripts/ncu_lines.py x.csv [top]
"""
import csv
import os
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = "?"
hdr = None
agg = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r or not r[0].strip().isdigit():
        continue
    try:
        s = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        ie = float(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    agg.append((s, ie, f"{fname}:{r[0]}", r[1].strip()[:100]))
ts = sum(a[0] for a in agg) or 1.0
ti = sum(a[1] for a in agg) or 1.0
print(f"{'stall%':>7s} {'inst%':>7s}  line")
for s, ie, loc, src in sorted(agg, key=lambda x: -x[0])[:top]:
    print(f"{100 * s / ts:6.1f}% {100 * ie / ti:6.1f}%  {loc:22s} {src}")
