"""Aggregate an ncu --page source --csv --print-source sass export by opcode:
share of warp-stall samples and executed instructions per SASS opcode."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
agg, cnt = defaultdict(float), defaultdict(float)
tot = 0.0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        ie = float(r[idx["Instructions Executed"]] or 0)
    except ValueError:
        continue
    src = r[idx["Source"]].split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    op = op.split(".")[0]
    agg[op] += s
    cnt[op] += ie
    tot += s
itot = sum(cnt.values())
print(f"{'opcode':12s} {'stall%':>7s} {'inst%':>7s}")
for op, s in sorted(agg.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{op:12s} {100 * s / tot:6.1f}% {100 * cnt[op] / itot:6.1f}%")
