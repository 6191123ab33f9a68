"""Plan only (IFGF_PLAN_VERBOSE diagnostics, plan wall times) for any bench config."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2010_02857_b200 import ifgf, inputs  # noqa: E402

c = {**inputs.CONFIGS, **inputs.EXTRA_CONFIGS}[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
pts = torch.from_numpy(c.points()).cuda()
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = ifgf.Plan(pts, c.k, c.levels, c.Ps, c.Pang)
    torch.cuda.synchronize()
    print(f"plan {c.name}: {time.perf_counter() - t0:.3f} s", flush=True)
    st = plan.stats()
    del plan
print(st["upward_kernel"])
