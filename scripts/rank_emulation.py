"""Multi-GPU scaling estimate on ONE GPU: build each rank's plan of an R-rank
source partition in turn (the same plan each rank of a torchrun job builds),
time its apply with CUDA events, and report max-over-ranks vs the 1-rank time.
The per-rank field is checked to sum to the 1-GPU field.  (The NCCL all-reduce
of 16 N bytes, ~1 ms at cfg4 over NVLink, is not included.)

usage: python scripts/rank_emulation.py cfg4 8 [reps]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_02857_b200 import ifgf, inputs  # noqa: E402


def timed_apply(plan, a, reps):
    out = plan.apply(a)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        out = plan.apply(a)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return out, min(ts)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    c = inputs.CONFIGS[name]
    pts = torch.from_numpy(c.points()).cuda()
    a = torch.from_numpy(c.densities()).cuda()
    res = {"config": name, "ranks": R}
    full = None
    single = os.environ.get("SKIP_SINGLE") is None  # cfg5 does not fit one GPU
    if single:
        plan = ifgf.Plan(pts, c.k, c.levels, c.Ps, c.Pang)
        full, t1 = timed_apply(plan, a, reps)
        res["t1_ms"] = t1
        full = full.cpu()
        del plan
        torch.cuda.empty_cache()
    acc = torch.zeros(c.n, dtype=torch.complex128)
    ts, ranges, mem = [], [], []
    for r in range(R):
        plan = ifgf.Plan(pts, c.k, c.levels, c.Ps, c.Pang, rank=r, nranks=R)
        part, tr = timed_apply(plan, a, reps)
        st = plan.stats()
        ts.append(tr)
        ranges.append(st["owned_leaf_range"])
        mem.append(st["plan_device_bytes"] / 1e9)
        acc += part.cpu()
        del plan, part
        torch.cuda.empty_cache()
        print(f"rank {r}: {tr:.1f} ms, leaves {ranges[-1]}, plan {mem[-1]:.1f} GB", flush=True)
    res.update({"rank_ms": ts, "max_ms": max(ts), "mean_ms": float(np.mean(ts)),
                "imbalance_max_over_mean": max(ts) / float(np.mean(ts)), "plan_gb_per_rank": mem,
                "points_per_s_estimate": c.n / (max(ts) * 1e-3)})
    if single:
        res.update({"speedup_vs_1": res["t1_ms"] / max(ts), "efficiency": res["t1_ms"] / (R * max(ts)),
                    "sum_vs_full_rel_l2": float(torch.linalg.norm(acc - full) / torch.linalg.norm(full))})
    else:
        tg = torch.from_numpy(inputs.error_targets(c.n, 1000))
        exact = ifgf.direct(pts, c.k, a, tg.cuda()).cpu()
        res["rel_err_vs_direct_1000"] = float(torch.linalg.norm(acc[tg] - exact) / torch.linalg.norm(exact))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
