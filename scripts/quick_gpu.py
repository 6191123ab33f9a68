"""Quick GPU check of one BASELINE config: plan, per-kernel-class times, points/s,
error vs the direct sum at 1000 targets, plus per-level K7 kernel choice."""
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_02857_b200 import ifgf, inputs  # noqa: E402

name = sys.argv[1]
c = inputs.CONFIGS[name]
pts = c.points()
a = c.densities()
dp = torch.from_numpy(pts).cuda()
da = torch.from_numpy(a).cuda()
t = time.time()
plan = ifgf.Plan(dp, c.k, c.levels, c.Ps, c.Pang)
torch.cuda.synchronize()
print(name, "plan s", time.time() - t, flush=True)
st = plan.stats()
print({k: st[k] for k in ("nseg", "upward_evals", "cousin_evals", "upward_kernel", "plan_device_bytes")}, flush=True)
plan.profile_enable(True)
out = plan.apply(da)
torch.cuda.synchronize()
plan.profile_read(reset=True)
ts = []
for i in range(3):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    out = plan.apply(da)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("apply ms", ts, "pts/s", c.n / (min(ts) * 1e-3), flush=True)
prof = plan.profile_read()
print({k: (v[0] / 3, v[1] / 3) for k, v in prof.items()}, flush=True)
tg = inputs.error_targets(c.n, 1000)
ex = ifgf.direct(dp, c.k, da, torch.from_numpy(tg).cuda()).cpu().numpy()
g = out.cpu().numpy()[tg]
print("rel err vs direct", np.sqrt(np.sum(np.abs(g - ex) ** 2) / np.sum(np.abs(ex) ** 2)), flush=True)
