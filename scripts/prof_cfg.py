"""Plan + 2 applies of any bench config (BASELINE or §8(f) extra), for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2010_02857_b200 import ifgf, inputs  # noqa: E402

c = {**inputs.CONFIGS, **inputs.EXTRA_CONFIGS}[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
pts = torch.from_numpy(c.points()).cuda()
a = torch.from_numpy(c.densities()).cuda()
plan = ifgf.Plan(pts, c.k, c.levels, c.Ps, c.Pang)
for _ in range(2):
    out = plan.apply(a)
torch.cuda.synchronize()
print("ok", c.name, float(out.abs().sum()))
