#!/usr/bin/env python
"""A/B of K7 variants on one config: per-class device times (CUDA events on the
apply stream) and the field's deviation from the first variant.

    python scripts/ab_upward.py cfg4 "IFGF_TC3=0" "IFGF_TC3=1" ...
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2010_02857_b200 import ifgf, inputs  # noqa: E402


def main():
    name = sys.argv[1]
    variants = sys.argv[2:] or [""]
    c = {**inputs.CONFIGS, **inputs.EXTRA_CONFIGS}[name]
    dev = torch.device("cuda:0")
    pts = torch.from_numpy(c.points()).to(dev)
    a = torch.from_numpy(c.densities()).to(dev)
    ref = None
    for v in variants:
        env = dict(kv.split("=") for kv in v.split(",") if kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        plan = ifgf.Plan(pts, c.k, c.levels, c.Ps, c.Pang)
        st = plan.stats()
        out = plan.apply(a)
        plan.apply(a, out)
        torch.cuda.synchronize()
        plan.profile_enable(True)
        plan.profile_read(reset=True)
        reps = 3
        for _ in range(reps):
            plan.apply(a, out)
        prof = plan.profile_read(reset=True)
        plan.profile_enable(False)
        plan.stats()
        o = out.cpu()
        dev_rel = None if ref is None else float(((o - ref).abs().pow(2).sum() / ref.abs().pow(2).sum()).sqrt())
        if ref is None:
            ref = o
        print(json.dumps({"variant": v, "upward_kernel": st["upward_kernel"],
                          "ms": {k2: round(t / reps, 3) for k2, (t, _) in prof.items()},
                          "total_ms": round(sum(t for t, _ in prof.values()) / reps, 3), "rel_vs_first": dev_rel}),
              flush=True)
        del plan, out
        torch.cuda.empty_cache()
        for k2, val in old.items():
            if val is None:
                os.environ.pop(k2, None)
            else:
                os.environ[k2] = val


if __name__ == "__main__":
    main()
