#!/usr/bin/env python
"""IFGF matvec benchmark (BASELINE.json metric: "IFGF matvec points/s (fp64
complex) at 1/2/4/8 B200; rel. error vs direct sum").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = one full IFGF operator application (the whole hot path: permute,
near field, source-to-cone, per-level fit / cousin / upward, un-permute; plus
the in-library NCCL all-reduce of the partial fields when N > 1) on synthetic
inputs resident in HBM.  Prints ONE JSON line on rank 0.

--impl reference times the oracle (oracle/, C++ with its deterministic OpenMP
mode on all host cores) on a bounded sample of the same workload: the partial
apply of a 1/128 Morton slice of the leaves (sources) over all N targets,
extrapolated by the slice's share of the sources (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2010_02857_b200 import inputs  # noqa: E402

ALL_CONFIGS = {**inputs.CONFIGS, **inputs.EXTRA_CONFIGS}
METRIC = "IFGF matvec points/s (fp64 complex) at 1/2/4/8 B200; rel. error vs direct sum"
UNIT = "points/s"

# Bounded CPU sample of the oracle (cpu_baseline and --impl reference): the oracle
# plan of the SAME workload owning a contiguous Morton slice of the leaf boxes
# (source partition); one step = its partial apply over all N
# targets; points/s = (owned sources / N) * N / t, i.e. the full apply's rate if its
# time scaled with the sources.  The slice's coarse ancestors carry whole-box cone
# data, so a slice costs more than its share (a conservative estimate): on cfg4 with
# 16 host cores the full apply measured 495 s (50.8 k points/s,
# profiles/r02/parity_full_cfg4.json).  cpu_baseline: 1/32 of the leaves (one step,
# ~20 s); --impl reference: 1/128 per step, so K + W steps end within minutes.
CPU_SLICE_START = 0.45
CPU_SLICE_BASELINE = 1.0 / 32
CPU_SLICE_REFERENCE = 1.0 / 128


class OracleSample:
    def __init__(self, c, frac_leaves: float):
        import oracle
        oracle.set_threads(0)
        self.cores = oracle.get_threads()
        self.c = c
        pts = c.points()
        self.a = c.densities()
        t0 = time.perf_counter()
        tree = oracle.OraclePlan(pts, c.k, c.levels, c.Ps, c.Pang, owned_morton=(0, 0))  # tree only
        info = tree.level_info(c.levels)
        del tree
        q = np.clip(np.floor((pts - info["x0"]) / info["H"]), 0, 2 ** (c.levels - 1) - 1).astype(np.uint64)
        key = np.zeros(len(pts), dtype=np.uint64)
        for bit in range(21):
            for ax, sh in ((0, 2), (1, 1), (2, 0)):
                key |= ((q[:, ax] >> np.uint64(bit)) & np.uint64(1)) << np.uint64(3 * bit + sh)
        leaves = np.unique(key)
        i0 = int(CPU_SLICE_START * len(leaves))
        i1 = i0 + max(1, int(frac_leaves * len(leaves)))
        lo, hi = int(leaves[i0]), int(leaves[min(i1, len(leaves) - 1)])
        self.frac = float(np.mean((key >= np.uint64(lo)) & (key < np.uint64(hi))))
        self.plan = oracle.OraclePlan(pts, c.k, c.levels, c.Ps, c.Pang, owned_morton=(lo, hi))
        self.setup_s = time.perf_counter() - t0
        self.desc = (f"oracle (C++, deterministic OpenMP on {self.cores} host threads) partial apply of "
                     f"{c.name} over all N={c.n} targets from a Morton slice of {i1 - i0} of {len(leaves)} leaf "
                     f"boxes ({self.frac * 100:.3f}% of the sources); points/s = (slice sources / N) * N / t")

    def step(self) -> float:
        t0 = time.perf_counter()
        self.plan.apply(self.a)
        return time.perf_counter() - t0

    def value(self, t: float) -> float:
        return self.frac * self.c.n / t


def algorithmic_flops_per_upward_eval(Ps: int, Pa: int, per_eval_geometry: bool = False) -> float:
    """SURVEY.md §8(d) "Algorithmic work per unit", upward evaluation (K7) per (parent
    node, child): "~310 with a precomputed tensor basis (P complex x real MACs), up to
    ~460 with per-evaluation geometry".  Grouped levels (the tensor-core kernels share
    one geometry per cell / orbit): every one of the P coefficients enters one
    complex x real MAC (4 flops) plus the recentering complex MAC (8 flops).  Levels
    run by the per-evaluation kernel (k_upward_pe) also compute each evaluation's
    geometry: +152 flops (460 - 308 at P = 75).  Special functions (sqrt, division,
    atan2, sincos) and padding are not counted, so the fraction understates the
    FP64 pipe's real load."""
    return 4.0 * (Ps * Pa * Pa) + 8.0 + (152.0 if per_eval_geometry else 0.0)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines: list[str] = []
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm, smax, power, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


def workload_config(c, world: int, st=None) -> dict:
    """The `config` object of the JSON line (same for both arms)."""
    cfg = {
        "workload": f"{c.name}: {c.geometry} {c.scale}, k={c.k / math.pi:.0f}pi ({c.k / math.pi:.0f} lambda across), "
                    f"N={c.n}, D={c.levels}, (P_s,P_ang)=({c.Ps},{c.Pang}), Fibonacci points, "
                    "splitmix64 densities",
        "N": c.n, "k": c.k, "levels": c.levels, "P_s": c.Ps, "P_ang": c.Pang,
        "parallelism": f"source-partition x{world} (work-weighted Morton leaf ranges) + in-library NCCL "
                       "all-reduce" if world > 1 else "1 GPU",
    }
    if st is not None:
        cfg["l2"] = ("inputs larger than L2: each apply streams "
                     f"{sum(st['segment_bytes'].values()) / 1e9:.1f} GB of cone-segment data")
    return cfg


def run_reference(args, rank: int):
    """Reference arm: the oracle (C++ CPU IFGF, deterministic OpenMP on all host
    cores) as it stands, each step the partial apply of the bounded cfg slice
    (OracleSample); the line carries our arm's config, metric and unit."""
    if rank != 0:
        return
    c = ALL_CONFIGS[args.config]
    smp = OracleSample(c, CPU_SLICE_REFERENCE)
    ts = [smp.step() for _ in range(args.warmup + args.steps)]
    timed = ts[args.warmup:] if len(ts) > args.warmup else ts
    t = sum(timed) / len(timed)
    value = smp.value(t)
    sample = smp.desc + f"; mean of {len(timed)} timed steps after {args.warmup} warm-up"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(c, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": smp.cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    from paper_2010_02857_b200 import ifgf

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    c = ALL_CONFIGS[args.config]

    pts_h = c.points()
    a_h = c.densities()
    pts = torch.from_numpy(pts_h).to(dev)
    a = torch.from_numpy(a_h).to(dev)
    del pts_h

    dfma_flops, _ = ifgf.bench_dfma(20000)  # measured FP64 FMA peak (roofline denominator)

    dist_on = world > 1 or args.dist
    comm = ifgf.NcclComm.from_group(None, local_rank) if dist_on else None
    t0 = time.perf_counter()
    plan = ifgf.Plan(pts, c.k, c.levels, c.Ps, c.Pang, rank=rank, nranks=world, comm=comm)
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - t0
    st = plan.stats()
    out = torch.empty(c.n, dtype=torch.complex128, device=dev)

    for _ in range(args.warmup):
        plan.apply(a, out)
    torch.cuda.synchronize()

    # ---------------- timed region: K applies, inputs resident in HBM.  The apply's
    # kernels replay from the plan's CUDA graph (one launch per step); a second timed
    # region of K applies launches them one by one with CUDA events around each
    # kernel on the apply stream (ifgf_profile_enable), for the per-kernel times and
    # the roofline.  Both regions are inside the clock sampling window.
    clocks = ClockSampler(local_rank)
    clocks.start()
    stream = torch.cuda.current_stream()

    def timed(profiled: bool) -> float:
        if profiled:
            plan.profile_enable(True)
            plan.profile_read(reset=True)
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            plan.apply(a, out)
        e1.record(stream)
        torch.cuda.synchronize()
        if dist_on:
            dist.barrier()
        t_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if dist_on:
            dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        return float(t_ms.item()) / args.steps

    ms_per_step = timed(False)
    ms_per_step_profiled = timed(True)
    clk = clocks.stop()
    prof = plan.profile_read(reset=True)
    plan.profile_enable(False)
    plan.stats()  # raises IfgfError if an apply met an invariant violation
    value = c.n / (ms_per_step * 1e-3)

    # ---------------- end to end: host buffers in, host result out, every step
    a_pin = torch.from_numpy(a_h).pin_memory()
    out_pin = torch.empty(c.n, dtype=torch.complex128).pin_memory()
    plan.apply_host(a_pin, out_pin)  # warm
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        plan.apply_host(a_pin, out_pin)  # C ABI: H2D, apply (+ NCCL all-reduce when N > 1), D2H, sync
    e3.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e2.elapsed_time(e3)], dtype=torch.float64, device=dev)
    if dist_on:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = c.n / (float(te.item()) / args.steps * 1e-3)

    # ---------------- accuracy vs the direct sum (after timing; not in the metric)
    plan.apply(a, out)
    tg = torch.from_numpy(inputs.error_targets(c.n, 1000)).to(dev)
    exact = ifgf.direct(pts, c.k, a, tg)
    got = out[tg]
    rel_err = float(torch.sqrt(torch.sum(torch.abs(got - exact) ** 2) / torch.sum(torch.abs(exact) ** 2)).item())
    st_after = plan.stats()  # raises IfgfError if an apply met an invariant violation

    # ---------------- roofline of the dominant kernel (K7 upward, FP64 pipe)
    up_ms, up_launch = prof["upward"]
    up_evals = sum(st["upward_evals"].values())  # per apply (this rank)
    # per level: kernel 2 (k_upward_pe) computes the geometry per evaluation
    pe_evals = sum(v for d, v in st["upward_evals"].items() if st["upward_kernel"].get(d, -1) == 2)
    flops_apply = ((up_evals - pe_evals) * algorithmic_flops_per_upward_eval(c.Ps, c.Pang)
                   + pe_evals * algorithmic_flops_per_upward_eval(c.Ps, c.Pang, True))
    achieved = flops_apply * args.steps / (up_ms * 1e-3) if up_ms > 0 else 0.0
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"{args.config}:upward_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    launches = sum(v[1] for v in prof.values())
    kernel_ms = {k: v[0] / args.steps for k, v in prof.items()}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            smp = OracleSample(c, CPU_SLICE_BASELINE)
            ts = [smp.step() for _ in range(args.cpu_repeats)]
            cpu = {"value": smp.value(statistics.median(ts)), "unit": UNIT, "cores": smp.cores, "kind": "oracle",
                   "sample": smp.desc + f"; median of {len(ts)} steps ({sum(ts):.1f} s wall, after "
                                        f"{smp.setup_s:.0f} s of oracle plan set-up)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(c, world, st),
            "rel_err_vs_direct": rel_err,
            "plan_ms": plan_s * 1e3,
            "ms_per_step_profiled": ms_per_step_profiled,
            "kernel_ms_per_step": kernel_ms,
            "roofline": {"kernel": "K7 upward (k_upward_tc / k_upward_s / k_upward_pe, all levels)", "bound": "alu", "achieved": achieved / 1e12,
                         "peak": dfma_flops / 1e12, "unit": "TFLOP/s", "frac": achieved / dfma_flops,
                         "traffic": traffic,
                         "peak_source": "FP64 DFMA microbenchmark (ifgf_bench_dfma) measured in this run; "
                                        "nominal 148 SM x 64 FMA/clk x 2 x 1.965 GHz = 37.2 TFLOP/s",
                         "flops_per_unit": {"grouped_geometry": algorithmic_flops_per_upward_eval(c.Ps, c.Pang),
                                            "per_evaluation_geometry":
                                                algorithmic_flops_per_upward_eval(c.Ps, c.Pang, True)},
                         "units_per_step": {"grouped_geometry": up_evals - pe_evals,
                                            "per_evaluation_geometry": pe_evals},
                         "flops_per_step": flops_apply},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 16 * c.n, "d2h_bytes_per_step": 16 * c.n},
            "gpu_launches": launches,
            "graph_applies": st_after["graph_applies"],
            "clocks": clk,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4", choices=sorted(inputs.CONFIGS) + sorted(inputs.EXTRA_CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-repeats", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="take the multi-GPU code path (process group, library NCCL communicator, in-library "
                         "all-reduce) even with one rank: a single-GPU check of that path")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1 or args.dist:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1 or args.dist:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
