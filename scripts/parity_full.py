#!/usr/bin/env python
"""Full GPU-vs-oracle parity on one BASELINE config, all sources and all N
targets, in the bench's launch configuration (one plan, nranks = 1).

    python scripts/parity_full.py cfg4 [--out profiles/r02/parity_full_cfg4.json]

Checks (BASELINE.json north_star): rel l2(GPU, oracle) <= 1e-11 over all N;
max_l |GPU_l - oracle_l| / rms(oracle); error vs the direct sum (GPU direct
kernel, cross-checked against the oracle's direct sum on 16 targets) on the
1000 seeded targets for both, with eps_GPU <= 1.1 eps_oracle; per-level
relevant-box and relevant-segment counts equal.  The oracle runs on all host
cores (its OpenMP mode is bitwise equal to serial).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2010_02857_b200 import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    from paper_2010_02857_b200 import ifgf

    c = {**inputs.CONFIGS, **inputs.EXTRA_CONFIGS}[args.config]
    pts, a = c.points(), c.densities()
    dev = torch.device("cuda:0")
    res = {"config": args.config, "N": c.n, "k": c.k, "levels": c.levels, "P_s": c.Ps, "P_ang": c.Pang,
           "host_cores": os.cpu_count()}
    t0 = time.perf_counter()
    plan = ifgf.Plan(torch.from_numpy(pts).to(dev), c.k, c.levels, c.Ps, c.Pang)
    got = plan.apply(torch.from_numpy(a).to(dev)).cpu().numpy()
    st = plan.stats()
    res["gpu_plan_apply_s"] = time.perf_counter() - t0
    res["upward_kernel"] = st["upward_kernel"]

    oracle.set_threads(0)
    res["oracle_threads"] = oracle.get_threads()
    t0 = time.perf_counter()
    oplan = oracle.OraclePlan(pts, c.k, c.levels, c.Ps, c.Pang)
    res["oracle_plan_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = oplan.apply(a)
    res["oracle_apply_s"] = time.perf_counter() - t0

    res["rel_l2_gpu_vs_oracle"] = oracle.rel_l2(got, ref)
    rms = float(np.sqrt(np.mean(np.abs(ref) ** 2)))
    res["max_abs_diff_over_rms"] = float(np.max(np.abs(got - ref)) / rms)
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
    res["max_elementwise_rel"] = float(rel.max())
    res["p99999_elementwise_rel"] = float(np.quantile(rel, 0.99999))
    res["levels_equal"] = {}
    for d in range(1, c.levels + 1):
        info = oplan.level_info(d)
        res["levels_equal"][d] = bool(st["nbox"][d] == info["nbox"] and st["nseg"][d] == info["nseg"])
    tg = inputs.error_targets(c.n, 1000)
    exact = ifgf.direct(torch.from_numpy(pts).to(dev), c.k, torch.from_numpy(a).to(dev),
                        torch.from_numpy(tg).to(dev)).cpu().numpy()
    chk = oracle.direct(pts, c.k, a, tg[:16])
    res["direct_gpu_vs_oracle_16"] = oracle.rel_l2(exact[:16], chk)
    res["eps_gpu"] = oracle.rel_l2(got[tg], exact)
    res["eps_oracle"] = oracle.rel_l2(ref[tg], exact)
    res["pass"] = bool(res["rel_l2_gpu_vs_oracle"] <= 1e-11 and res["eps_gpu"] <= 1.1 * res["eps_oracle"]
                       and all(res["levels_equal"].values()) and res["max_abs_diff_over_rms"] <= 1e-10)
    line = json.dumps(res)
    print(line, flush=True)
    if args.out:
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        with open(args.out, "w") as f:
            f.write(line + "\n")
    sys.exit(0 if res["pass"] else 1)


if __name__ == "__main__":
    main()
