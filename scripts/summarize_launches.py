"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python scripts/summarize_launches.py launches.csv [--apply-only]
Prints per-kernel launch count, total ms and share of the listed time.  With
--apply-only, plan-build / harness kernels are excluded so the shares describe
the timed matvec step.
"""
import csv
import re
import sys
from collections import defaultdict

APPLY = ("k_permute", "k_near", "k_s2c", "k_fit", "k_cousin", "k_upward", "k_unpermute")


def short(name: str) -> str:
    m = re.search(r"(k_[A-Za-z0-9_]+)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def main():
    path = sys.argv[1]
    apply_only = "--apply-only" in sys.argv
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        if apply_only and not k.startswith(APPLY):
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(
            r.get("Metric Unit", "ns"), 1e-6)
        agg[k][0] += 1
        agg[k][1] += v * scale
    total = sum(v[1] for v in agg.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total_ms':>12s} {'share':>7s}")
    for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {c:8d} {ms:12.3f} {100 * ms / total:6.1f}%")
    print(f"{'TOTAL':40s} {sum(v[0] for v in agg.values()):8d} {total:12.3f}")


if __name__ == "__main__":
    main()
