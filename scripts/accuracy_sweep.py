"""accuracy / cost of the interpolation orders (P_s, P_ang) and
the leaf size (D) on one GPU.  Prints one JSON object per case: relative l2 error
against the direct sum at 1000 seeded targets, apply time and points/s.

usage: python scripts/accuracy_sweep.py [cfg2]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_02857_b200 import ifgf, inputs  # noqa: E402

base = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
pts = torch.from_numpy(base.points()).cuda()
a = torch.from_numpy(base.densities()).cuda()
tg = torch.from_numpy(inputs.error_targets(base.n, 1000)).cuda()
exact = ifgf.direct(pts, base.k, a, tg)
cases = [(base.levels, ps, pa) for ps, pa in [(2, 3), (3, 3), (3, 5), (5, 5), (5, 7), (7, 7)]]
cases += [(base.levels + 1, 3, 5), (base.levels - 1, 3, 5)]
for D, ps, pa in cases:
    plan = ifgf.Plan(pts, base.k, D, ps, pa)
    out = plan.apply(a)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = plan.apply(a)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    err = float(torch.linalg.norm(out[tg] - exact) / torch.linalg.norm(exact))
    st = plan.stats()
    print(json.dumps({"config": base.name, "N": base.n, "k": base.k, "D": D, "P_s": ps, "P_ang": pa,
                      "rel_err_vs_direct": err, "apply_ms": min(ts), "points_per_s": base.n / (min(ts) * 1e-3),
                      "upward_kernel": st["upward_kernel"]}), flush=True)
    del plan
