"""Per-kernel-class times of one rank's apply in an R-rank source partition
(one GPU), vs 1/R of the single-GPU apply.  usage: rank_profile.py cfg4 8 0"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_02857_b200 import ifgf, inputs  # noqa: E402

name, R, r = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
c = inputs.CONFIGS[name]
pts = torch.from_numpy(c.points()).cuda()
a = torch.from_numpy(c.densities()).cuda()
for ranks, rank in ((1, 0), (R, r)):
    plan = ifgf.Plan(pts, c.k, c.levels, c.Ps, c.Pang, rank=rank, nranks=ranks)
    plan.apply(a)
    torch.cuda.synchronize()
    plan.profile_enable(True)
    plan.profile_read(reset=True)
    for _ in range(2):
        plan.apply(a)
    torch.cuda.synchronize()
    prof = plan.profile_read()
    st = plan.stats()
    scale = 1.0 / R if ranks == 1 else 1.0
    print(f"ranks={ranks} rank={rank}:", {k: round(v[0] / 2 * scale, 2) for k, v in prof.items()},
          "upward_evals", sum(st["upward_evals"].values()) * scale, "cousin", sum(st["cousin_evals"].values()) * scale,
          "nseg", {d: int(v * scale) for d, v in st["nseg"].items() if v}, flush=True)
    del plan
    torch.cuda.empty_cache()
