"""Instruction / stall breakdown of an ncu report by CUDA source line and by
named line ranges (ncu -i rep --page source --csv --print-source cuda,sass).

usage: python scripts/ncu_breakdown.py x.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
fname = "?"
agg, src, st = {}, {}, {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r or not r[0].strip().isdigit():
        continue
    try:
        ie = float(r[hdr["Instructions Executed"]] or 0)
        s = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    key = (fname, int(r[0]))
    agg[key] = agg.get(key, 0.0) + ie
    st[key] = st.get(key, 0.0) + s
    src[key] = r[1].strip()[:80]
tot = sum(agg.values()) or 1.0
tots = sum(st.values()) or 1.0
print(f"total executed warp instructions {tot / 1e9:.2f} G")
for key in sorted(agg, key=lambda x: -agg[x])[:top]:
    print(f"{100 * agg[key] / tot:5.1f}% inst {100 * st[key] / tots:5.1f}% stall  {key[0]}:{key[1]}  {src[key]}")
