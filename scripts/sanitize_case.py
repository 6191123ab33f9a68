#!/usr/bin/env python
"""Small applies for compute-sanitizer (memcheck / racecheck / synccheck):
cfg1 and a 60k-point lambda/4 sphere whose fine levels run the FP64 tensor-core
K7 with quarter-turn orbits, both eager (graph=False) so every kernel launch is
visible to the tool.

    compute-sanitizer --tool memcheck python scripts/sanitize_case.py
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2010_02857_b200 import ifgf, inputs  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    cases = [("cfg1", inputs.CONFIGS["cfg1"].points(), 4 * math.pi, 4),
             ("tc60k", inputs.fibonacci_sphere(60_000), 8 * math.pi, 6)]
    if len(sys.argv) > 1:
        cases = [c for c in cases if c[0] in sys.argv[1:]]
    for name, pts, k, D in cases:
        a = inputs.densities(len(pts))
        plan = ifgf.Plan(torch.from_numpy(pts).to(dev), k, D, 3, 5, graph=False)
        out = plan.apply(torch.from_numpy(a).to(dev))
        torch.cuda.synchronize()
        st = plan.stats()
        print(f"{name}: N={len(pts)} D={D} kernels={st['upward_kernel']} |out|={float(out.abs().sum()):.6e}",
              flush=True)


if __name__ == "__main__":
    main()
