"""GPU parity at the BASELINE configs' full sizes and in the bench's launch
configuration (one plan, nranks = 1), plus the paths that only large problems
reach (several K7 L2 tiles, orbit-aware chunk order), against the oracle.

Bar (BASELINE.json north_star): relative l2 <= 1e-11 vs the oracle over all N
targets; error vs the direct sum <= 1.1 x the oracle's own (eq.
errorcomputation); equal relevant-segment sets.  Beside the global
relative l2, every element is bounded: max_l |GPU_l - oracle_l| <= 1e-10 x
rms(oracle) (per-element differences are rounding, ~1e-13 of the rms).

cfg4 (N = 25,165,824, the bench workload) runs the full GPU plan and apply with
densities zeroed outside a 1/64 Morton slice of the leaves; the oracle plan owns
that slice (source partition) and returns exactly the field of
the masked densities (tests/test_oracle_parallel.py), so the comparison covers
all N targets at a bounded oracle cost.  The all-sources cfg4 comparison is
scripts/parity_full.py (profiles/r02/parity_full_cfg4.json).
"""
import math
import os

import numpy as np
import pytest

import oracle
from paper_2010_02857_b200 import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PARITY = 1e-11
ELEMENT = 1e-10


@pytest.fixture(scope="module")
def ifgf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2010_02857_b200 import ifgf as m
    oracle.set_threads(0)  # all host cores (bitwise equal to serial)
    return m


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda:0")


def element_max(got, ref):
    rms = np.sqrt(np.mean(np.abs(ref) ** 2))
    return float(np.max(np.abs(got - ref)) / rms)


def morton(q):
    q = np.asarray(q, dtype=np.uint64)
    r = np.zeros(q.shape[0], dtype=np.uint64)
    for b in range(21):
        for a, sh in ((0, 2), (1, 1), (2, 0)):
            r |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + sh)
    return r


def leaf_keys_of_points(pts, st):
    """Leaf Morton key of every point from the plan's root box (DESIGN.md §3:
    q = clamp(floor((x - x0)/H_D)))."""
    D = st["levels"]
    HD = math.ldexp(st["root_side"], -(D - 1))
    x0 = np.array(st["root_center"]) - st["root_side"] / 2.0
    q = np.clip(np.floor((pts - x0) / HD), 0, 2 ** (D - 1) - 1).astype(np.int64)
    return morton(q)


def box_keys(rows):
    return morton(np.asarray(rows)[:, :3])


def check_level_segments(plan, oplan, D, active_only):
    for d in range(3, D + 1):
        o = oplan.level_segments(d)
        g = plan.level_segments(d)
        if active_only:
            g = g[np.isin(box_keys(g), np.unique(box_keys(o)))]
        key = lambda x: np.sort(box_keys(x) * np.uint64(1 << 24) + x[:, 3].astype(np.uint64))  # noqa: E731
        assert len(o) == len(g), d
        assert np.array_equal(key(o), key(g)), d


def test_cfg3_full_parity(ifgf):
    """cfg3 (oblate (1, 1, 0.25), 32 lambda, N = 1,572,864, D = 7, (P_s, P_ang) = (5, 5))
    against the oracle over all N, in the bench's launch configuration."""
    c = inputs.CONFIGS["cfg3"]
    pts, a = c.points(), c.densities()
    oplan = oracle.OraclePlan(pts, c.k, c.levels, c.Ps, c.Pang)
    ref = oplan.apply(a)
    plan = ifgf.Plan(dev(pts), c.k, c.levels, c.Ps, c.Pang)
    got = plan.apply(dev(a)).cpu().numpy()
    st = plan.stats()
    assert oracle.rel_l2(got, ref) <= PARITY
    assert element_max(got, ref) <= ELEMENT
    for d in range(1, c.levels + 1):
        assert st["nbox"][d] == oplan.level_info(d)["nbox"]
        assert st["nseg"][d] == oplan.level_info(d)["nseg"]
    check_level_segments(plan, oplan, c.levels, active_only=False)
    tg = inputs.error_targets(c.n, 1000)
    exact = ifgf.direct(dev(pts), c.k, dev(a), dev(tg)).cpu().numpy()
    assert oracle.rel_l2(got[tg], exact) <= 1.1 * oracle.rel_l2(ref[tg], exact)


@pytest.mark.parametrize("part", [(0.45, 1 / 64)])
def test_cfg4_bench_config_slice_parity(ifgf, part):
    """cfg4 (128 lambda sphere, N = 25,165,824, D = 10, the bench workload): the GPU
    plan exactly as bench.py builds it (nranks = 1, adaptive L2 tiles, orbit chunk
    order, every K7 kernel the plan picks), applied to densities zeroed outside a
    1/64 Morton slice of the leaves, against the oracle owning that slice: all N
    targets, every level's relevant segments of the slice's boxes, and the error
    against the direct sum of the masked densities."""
    c = inputs.CONFIGS["cfg4"]
    pts, a = c.points(), c.densities()
    plan = ifgf.Plan(dev(pts), c.k, c.levels, c.Ps, c.Pang)
    st = plan.stats()
    assert st["upward_kernel"][c.levels] == 1  # the tensor-core K7 at the finest level
    pk = leaf_keys_of_points(pts, st)
    leaves = np.unique(pk)
    i0 = int(part[0] * len(leaves))
    i1 = i0 + max(1, int(part[1] * len(leaves)))
    lo, hi = int(leaves[i0]), int(leaves[i1])
    mine = (pk >= np.uint64(lo)) & (pk < np.uint64(hi))
    am = np.where(mine, a, 0.0)
    got = plan.apply(dev(am)).cpu().numpy()
    st = plan.stats()  # raises if an apply met an invariant violation
    oplan = oracle.OraclePlan(pts, c.k, c.levels, c.Ps, c.Pang, owned_morton=(lo, hi))
    ref = oplan.apply(a)  # partial field of the owned slice == field of the masked densities
    assert oracle.rel_l2(got, ref) <= PARITY
    assert element_max(got, ref) <= ELEMENT
    check_level_segments(plan, oplan, c.levels, active_only=True)
    tg = inputs.error_targets(c.n, 1000)
    exact = ifgf.direct(dev(pts), c.k, dev(am), dev(tg)).cpu().numpy()
    assert oracle.rel_l2(got[tg], exact) <= 1.1 * oracle.rel_l2(ref[tg], exact)


@pytest.mark.parametrize("env", [
    {"IFGF_TILE_MB": "0.3"},                                           # several fixed tiles, kernels by run length
    {"IFGF_TILE_MB": "1", "IFGF_LEGACY_UPWARD": "5"},                  # TC everywhere, many tiles
    {"IFGF_TILE_MB": "1", "IFGF_LEGACY_UPWARD": "8"},                  # TC2 everywhere, many tiles
    {"IFGF_TILE_TARGET": "4", "IFGF_TILE_MIN_MB": "0.2"},             # adaptive tile shrink path
    {"IFGF_TILE_MB": "0.5", "IFGF_NO_CHUNK_ORDER": "1"},               # tiles without chunk order
])
def test_k7_multi_tile_and_chunk_order(ifgf, env, monkeypatch):
    """The K7 grouping by L2 tiles (consecutive parent boxes), the orbit-aware chunk
    order and the adaptive tile shrink only trigger on large problems by default;
    forcing small tiles exercises them at oracle-checkable size (60k points, D = 6,
    quarter-turn orbits on the tensor-core levels)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    n, k, D = 60_000, 8 * math.pi, 6
    pts = inputs.fibonacci_sphere(n)
    a = inputs.densities(n, seed=31)
    plan = ifgf.Plan(dev(pts), k, D, 3, 5)
    got = plan.apply(dev(a)).cpu().numpy()
    plan.stats()
    ref = oracle.OraclePlan(pts, k, D, 3, 5).apply(a)
    assert oracle.rel_l2(got, ref) <= PARITY
    assert element_max(got, ref) <= ELEMENT


@pytest.mark.parametrize("n,kpi,D", [(24_576, 16, 7), (98_304, 32, 8)])
def test_f3_sweeps_parity(ifgf, n, kpi, D):
    """SURVEY.md §8(f) f3 sweeps at oracle-checkable sizes, leaves lambda/4
    (P:2056-2059): the N sweep at kappa a = 16 pi (Table timings3; its
    first row, N = 24,576, D = 7) and the kappa sweep (Table timings2)
    at kappa a = 32 pi on N = 98,304 (D = 8).  All N targets, per-level segment
    counts, and the error against the direct sum within 1.1x the oracle's."""
    k = kpi * math.pi
    pts, a = inputs.fibonacci_sphere(n), inputs.densities(n)
    oplan = oracle.OraclePlan(pts, k, D, 3, 5)
    ref = oplan.apply(a)
    plan = ifgf.Plan(dev(pts), k, D, 3, 5)
    got = plan.apply(dev(a)).cpu().numpy()
    st = plan.stats()
    assert oracle.rel_l2(got, ref) <= PARITY
    assert element_max(got, ref) <= ELEMENT
    for d in range(3, D + 1):
        assert st["nseg"][d] == oplan.level_info(d)["nseg"]
    tg = inputs.error_targets(n, 1000)
    exact = ifgf.direct(dev(pts), k, dev(a), dev(tg)).cpu().numpy()
    assert oracle.rel_l2(got[tg], exact) <= 1.1 * oracle.rel_l2(ref[tg], exact)
