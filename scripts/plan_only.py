"""Plan only (IFGF_PLAN_VERBOSE diagnostics) for any bench config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2010_02857_b200 import ifgf, inputs  # noqa: E402

c = {**inputs.CONFIGS, **inputs.EXTRA_CONFIGS}[sys.argv[1]]
plan = ifgf.Plan(torch.from_numpy(c.points()).cuda(), c.k, c.levels, c.Ps, c.Pang)
torch.cuda.synchronize()
print(plan.stats()["upward_kernel"])
