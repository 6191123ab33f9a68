"""Host logic of bench.py (no GPU): the algorithmic work figures of the roofline
 and the config object shared by both arms."""
import math
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2010_02857_b200 import inputs  # noqa: E402


def test_upward_flops_per_unit():
    # "~310 with a precomputed tensor basis ... up to ~460 with per-evaluation geometry"
    assert bench.algorithmic_flops_per_upward_eval(3, 5) == 308.0
    assert bench.algorithmic_flops_per_upward_eval(3, 5, True) == 460.0
    assert bench.algorithmic_flops_per_upward_eval(5, 5) == 4 * 125 + 8


def test_workload_config_names_every_config():
    for name, c in {**inputs.CONFIGS, **inputs.EXTRA_CONFIGS}.items():
        cfg = bench.workload_config(c, 1)
        assert cfg["workload"].startswith(name + ":")
        assert cfg["N"] == c.n and cfg["levels"] == c.levels and cfg["parallelism"] == "1 GPU"
        assert math.isclose(cfg["k"], c.k)
    assert "x8" in bench.workload_config(inputs.CONFIGS["cfg4"], 8)["parallelism"]


def test_oracle_sample_slice():
    """The bounded CPU sample (cpu_baseline / --impl reference): a Morton slice of
    the leaves, its partial apply, and the rate extrapolated by its share of sources."""
    smp = bench.OracleSample(inputs.CONFIGS["cfg2"], bench.CPU_SLICE_REFERENCE)
    assert 0.0 < smp.frac < 0.03
    t = smp.step()
    assert t > 0 and smp.value(t) == smp.frac * smp.c.n / t
    assert "Morton slice" in smp.desc and smp.cores >= 1
