"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bar (BASELINE.json north_star): relative l2 <= 1e-11 vs the oracle; error vs the
direct sum <= 1.1 x the oracle's own; discrete plan decisions bit-identical.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2010_02857_b200 import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PARITY = 1e-11


@pytest.fixture(scope="module")
def ifgf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2010_02857_b200 import ifgf as m
    return m


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda:0")


def run_gpu(ifgf, pts, a, k, D, Ps=3, Pa=5, **kw):
    plan = ifgf.Plan(dev(pts), k, D, Ps, Pa, **kw)
    out = plan.apply(dev(a)).cpu().numpy()
    st = plan.stats()  # also raises if an apply met an invariant violation
    return plan, out, st


def segs_sorted(x):
    x = np.asarray(x, dtype=np.int64).reshape(-1, 4)
    return x[np.lexsort((x[:, 3], x[:, 2], x[:, 1], x[:, 0]))]


# ------------------------------------------------------------------ cfg1
@pytest.fixture(scope="module")
def cfg1_runs(ifgf):
    c = inputs.CONFIGS["cfg1"]
    pts, a = c.points(), c.densities()
    oplan = oracle.OraclePlan(pts, c.k, c.levels, c.Ps, c.Pang)
    ref = oplan.apply(a)
    plan, got, st = run_gpu(ifgf, pts, a, c.k, c.levels, c.Ps, c.Pang)
    return c, pts, a, oplan, ref, plan, got, st


def test_cfg1_parity_all_points(cfg1_runs):
    c, pts, a, oplan, ref, plan, got, st = cfg1_runs
    assert oracle.rel_l2(got, ref) <= PARITY


def test_cfg1_error_vs_full_direct_sum(cfg1_runs, ifgf):
    """cfg1 is compared to the full O(N^2) direct sum (BASELINE.json configs[0])."""
    c, pts, a, oplan, ref, plan, got, st = cfg1_runs
    tg = np.arange(c.n)
    exact = ifgf.direct(dev(pts), c.k, dev(a), dev(tg)).cpu().numpy()
    sample = inputs.error_targets(c.n, 500)
    np.testing.assert_allclose(exact[sample], oracle.direct(pts, c.k, a, sample), rtol=1e-12, atol=1e-13)
    e_gpu, e_or = oracle.rel_l2(got, exact), oracle.rel_l2(ref, exact)
    assert e_gpu <= 1.1 * e_or


def test_cfg1_plan_diff(cfg1_runs):
    """Per level: relevant boxes and the sorted (box, cell) keys are identical."""
    c, pts, a, oplan, ref, plan, got, st = cfg1_runs
    for d in range(1, c.levels + 1):
        assert st["nbox"][d] == oplan.level_info(d)["nbox"]
        assert st["grid"][d] == (oplan.level_info(d)["ns"], oplan.level_info(d)["nC"])
        np.testing.assert_array_equal(segs_sorted(plan.level_segments(d)), segs_sorted(oplan.level_segments(d)))


def test_plan_flags_by_runs_match_per_node(ifgf, monkeypatch):
    """The plan's relevance flags by runs of parent segments sharing a cell (one
    classification per (cell, node, octant)) give exactly the per-(segment, node)
    flags (IFGF_FLAG_PER_NODE=1): identical segment lists at every level, on a
    rough sphere with long and short runs, and the oracle's lists too."""
    n, k, D = 30000, 8 * math.pi, 6
    pts = inputs.rough_sphere(n)
    monkeypatch.setenv("IFGF_FLAG_PER_NODE", "1")
    per_node = ifgf.Plan(dev(pts), k, D, 3, 5)
    monkeypatch.delenv("IFGF_FLAG_PER_NODE")
    runs = ifgf.Plan(dev(pts), k, D, 3, 5)
    oplan = oracle.OraclePlan(pts, k, D, 3, 5)
    for d in range(3, D + 1):
        a = segs_sorted(runs.level_segments(d))
        np.testing.assert_array_equal(a, segs_sorted(per_node.level_segments(d)))
        np.testing.assert_array_equal(a, segs_sorted(oplan.level_segments(d)))


def test_cfg1_stage_masks(cfg1_runs, ifgf):
    c, pts, a, oplan, ref, plan, got, st = cfg1_runs
    for mask in (ifgf.IFGF_STAGE_NEAR, ifgf.IFGF_STAGE_NEAR | ifgf.IFGF_STAGE_COUSIN, ifgf.IFGF_STAGE_COUSIN):
        _, g, _ = run_gpu(ifgf, pts, a, c.k, c.levels, stage_mask=mask)
        r = oplan.apply(a, stage_mask=mask)
        assert oracle.rel_l2(g, r) <= PARITY, mask


def test_apply_host_and_reuse(cfg1_runs):
    """ifgf_apply_host (host buffers, e2e path) equals ifgf_apply; the plan is reusable."""
    c, pts, a, oplan, ref, plan, got, st = cfg1_runs
    h = plan.apply_host(a).numpy()
    assert np.array_equal(h, got)
    b = inputs.densities(c.n, seed=3)
    assert oracle.rel_l2(plan.apply(dev(b)).cpu().numpy(), oplan.apply(b)) <= PARITY


def test_linearity_and_determinism(cfg1_runs):
    c, pts, a, oplan, ref, plan, got, st = cfg1_runs
    b = inputs.densities(c.n, seed=11)
    al, be = 0.7 + 0.2j, -1.1 + 0.4j
    lhs = plan.apply(dev(al * a + be * b)).cpu().numpy()
    rhs = al * got + be * plan.apply(dev(b)).cpu().numpy()
    assert oracle.rel_l2(lhs, rhs) < 1e-12
    again = plan.apply(dev(a)).cpu().numpy()
    assert np.array_equal(again, got)


# ---------------------------------------------------- ragged / small / edge
@pytest.mark.parametrize("n,D", [(1, 3), (2, 2), (2, 4), (7, 3), (100, 1), (100, 2), (333, 3), (1000, 4),
                                 (4099, 5), (5000, 6)])
def test_small_and_ragged(ifgf, n, D):
    rng = np.random.default_rng(n + D)
    pts = inputs.fibonacci_sphere(n) * rng.uniform(0.5, 2.0)
    a = inputs.densities(n, seed=n)
    k = 9.0
    _, got, _ = run_gpu(ifgf, pts, a, k, D)
    ref = oracle.OraclePlan(pts, k, D, 3, 5).apply(a)
    if n == 1:
        assert np.all(got == 0)
    else:
        assert oracle.rel_l2(got, ref) <= PARITY


@pytest.mark.parametrize("Ps,Pa", [(5, 5), (5, 7), (4, 6), (1, 1), (2, 3), (7, 9)])
def test_orders_generic_and_specialised(ifgf, Ps, Pa):
    """(3,5) and (5,5) run specialised kernels; the rest the runtime-order path."""
    n = 6000
    pts = inputs.fibonacci_sphere(n, (1.0, 1.0, 0.25))
    a = inputs.densities(n)
    k = 20.0
    _, got, _ = run_gpu(ifgf, pts, a, k, 5, Ps, Pa)
    ref = oracle.OraclePlan(pts, k, 5, Ps, Pa).apply(a)
    assert oracle.rel_l2(got, ref) <= PARITY


def test_leaf_grid_and_laplace(ifgf):
    n = 5000
    pts = inputs.rough_sphere(n)
    a = inputs.densities(n)
    for k, ns, nc in [(0.0, 1, 2), (15.0, 2, 3), (15.0, 1, 4)]:
        _, got, _ = run_gpu(ifgf, pts, a, k, 5, leaf_ns=ns, leaf_nc=nc)
        ref = oracle.OraclePlan(pts, k, 5, 3, 5, leaf_ns=ns, leaf_nc=nc).apply(a)
        assert oracle.rel_l2(got, ref) <= PARITY, (k, ns, nc)


def test_centred_source_exact(ifgf):
    """One unit source exactly at a leaf centre, D = 3: the result is exact (no
    interpolation error): GPU equals the direct sum to rounding."""
    rng = np.random.default_rng(4)
    pts = rng.uniform(-1.99, 1.99, (600, 3))
    pts[0] = [0.5, 0.5, -0.5]
    a = np.zeros(len(pts), dtype=complex)
    a[0] = 1.0
    _, got, _ = run_gpu(ifgf, pts, a, 3.0, 3, root=([0.0, 0.0, 0.0], 4.0))
    ref = oracle.direct(pts, 3.0, a, np.arange(len(pts)))
    assert oracle.rel_l2(got, ref) < 1e-14


def test_metamorphic_rotation(ifgf):
    n = 8000
    pts = inputs.fibonacci_sphere(n)
    a = inputs.densities(n)
    _, I, _ = run_gpu(ifgf, pts, a, 25.0, 5)
    rot = np.stack([-pts[:, 1], pts[:, 0], pts[:, 2]], axis=1)
    _, J, _ = run_gpu(ifgf, rot, a, 25.0, 5)
    assert oracle.rel_l2(J, I) < 1e-12


def test_errors(ifgf):
    pts = inputs.fibonacci_sphere(100)
    with pytest.raises(ifgf.IfgfError) as e:
        ifgf.Plan(dev(np.concatenate([pts, pts[:1]])), 1.0, 3, 3, 5)
    assert e.value.code == 2
    with pytest.raises(ifgf.IfgfError) as e:
        ifgf.Plan(dev(np.zeros((4, 3))), 1.0, 3, 3, 5)
    assert e.value.code == 2
    bad = pts.copy()
    bad[5, 1] = np.nan
    with pytest.raises(ifgf.IfgfError) as e:
        ifgf.Plan(dev(bad), 1.0, 3, 3, 5)
    assert e.value.code == 1
    for kw in [dict(k=-1.0), dict(levels=0), dict(levels=23), dict(P_s=0), dict(P_ang=17)]:
        args = dict(k=1.0, levels=3, P_s=3, P_ang=5)
        args.update(kw)
        with pytest.raises(ifgf.IfgfError) as e:
            ifgf.Plan(dev(pts), args["k"], args["levels"], args["P_s"], args["P_ang"])
        assert e.value.code == 1


def test_multirank_emulation_one_gpu(ifgf):
    """Source partition by work-weighted Morton leaf ranges: the per-rank partial
    fields (run sequentially on one GPU) sum to the single-GPU field."""
    c = inputs.CONFIGS["cfg1"]
    pts, a = c.points(), c.densities()
    _, full, _ = run_gpu(ifgf, pts, a, c.k, c.levels)
    for R in (2, 3, 8):
        acc = np.zeros_like(full)
        covered = []
        for r in range(R):
            p, part, st = run_gpu(ifgf, pts, a, c.k, c.levels, rank=r, nranks=R)
            covered.append(st["owned_leaf_range"])
            acc += part
        assert covered[0][0] == 0 and all(covered[i][1] == covered[i + 1][0] for i in range(R - 1))
        assert oracle.rel_l2(acc, full) < 1e-13, R


def test_multirank_emulation_tc_orbits(ifgf):
    """Source partition on a case whose fine levels run the tensor-core K7 with
    quarter-turn orbits: the per-rank partial fields (3 ranks, sequentially on one GPU)
    sum to the single-GPU field."""
    n, k, D = 60000, 8 * math.pi, 6
    pts = inputs.fibonacci_sphere(n)
    a = inputs.densities(n, seed=21)
    _, full, st = run_gpu(ifgf, pts, a, k, D)
    assert st["upward_kernel"][D] == 1
    acc = np.zeros_like(full)
    for r in range(3):
        _, part, _ = run_gpu(ifgf, pts, a, k, D, rank=r, nranks=3)
        acc += part
    assert oracle.rel_l2(acc, full) < 1e-13


@pytest.mark.parametrize("legacy,slots", [("0", None), ("0", "1"), ("0", "0"), ("1", None)])
def test_cousin_kernel_variants(ifgf, legacy, slots, monkeypatch):
    """K6: the warp-staged kernel (default) and the per-lane global-load kernel
    (IFGF_LEGACY_COUSIN=1) both match the oracle.  IFGF_STAGE_SLOTS caps the child
    segments a warp stages (K6 and the per-evaluation K7), so that their
    global-memory fallback is exercised as well."""
    monkeypatch.setenv("IFGF_LEGACY_COUSIN", legacy)
    if slots is not None:
        monkeypatch.setenv("IFGF_STAGE_SLOTS", slots)
        monkeypatch.setenv("IFGF_LEGACY_UPWARD", "7")
    n = 20000
    pts = inputs.rough_sphere(n)
    a = inputs.densities(n, seed=8)
    k = 5 * math.pi
    _, got, _ = run_gpu(ifgf, pts, a, k, 5)
    ref = oracle.OraclePlan(pts, k, 5, 3, 5).apply(a)
    assert oracle.rel_l2(got, ref) <= PARITY


@pytest.mark.parametrize("nosym", ["0", "1"])
def test_default_kernel_choice_tc_and_staged(ifgf, nosym, monkeypatch):
    """At the default settings a lambda/4-leaf sphere uses the FP64 tensor-core
    K7 on its fine levels and a per-evaluation or staged K7 on the coarse ones;
    all match the oracle, with and without the quarter-turn orbit grouping
    (reading R18; IFGF_NO_SYMMETRY=1: cells only), and both groupings give the
    same field up to rounding."""
    monkeypatch.setenv("IFGF_NO_SYMMETRY", nosym)
    n, k, D = 60000, 8 * math.pi, 6
    pts = inputs.fibonacci_sphere(n)
    a = inputs.densities(n, seed=5)
    _, got, st = run_gpu(ifgf, pts, a, k, D)
    kern = st["upward_kernel"]
    assert kern[D] == 1 and all(kern[d] in (0, 1, 2, 3) for d in range(4, D + 1)), kern
    ref = oracle.OraclePlan(pts, k, D, 3, 5).apply(a)
    assert oracle.rel_l2(got, ref) <= PARITY


@pytest.mark.parametrize("scale", [(0.1, 0.1, 1.0), (1.0, 1.0, 0.25)])
def test_spheroids(ifgf, scale):
    """SURVEY.md §8(f) f3 shapes at small size: prolate (0.1, 0.1, 1) and oblate
    (1, 1, 0.25) spheroids (segment counts and load balance differ from the sphere's)."""
    n, k, D = 20000, 8 * math.pi, 6
    pts = inputs.fibonacci_sphere(n, scale)
    a = inputs.densities(n, seed=17)
    _, got, _ = run_gpu(ifgf, pts, a, k, D)
    ref = oracle.OraclePlan(pts, k, D, 3, 5).apply(a)
    assert oracle.rel_l2(got, ref) <= PARITY


@pytest.mark.slow
def test_cfg3_family_oblate_p55(ifgf):
    """cfg3's workload family at 1/16 of its size: oblate (1, 1, 0.25) spheroid, leaves
    lambda/2, (P_s, P_ang) = (5, 5) (the P = 125 specialised kernels), N = 98,304,
    k = 8 pi, D = 5: parity with the oracle, and the error against the direct sum
    within 1.1x the oracle's."""
    n, k, D = 98_304, 8 * math.pi, 5
    pts = inputs.fibonacci_sphere(n, (1.0, 1.0, 0.25))
    a = inputs.densities(n)
    ref = oracle.OraclePlan(pts, k, D, 5, 5).apply(a)
    _, got, _ = run_gpu(ifgf, pts, a, k, D, 5, 5)
    assert oracle.rel_l2(got, ref) <= PARITY
    tg = inputs.error_targets(n, 1000)
    exact = ifgf.direct(dev(pts), k, dev(a), dev(tg)).cpu().numpy()
    assert oracle.rel_l2(got[tg], exact) <= 1.1 * oracle.rel_l2(ref[tg], exact)


def test_classification_fast_path_matches_exact_chain(ifgf, monkeypatch):
    """The certified classification fast path (rsqrt-based s/ds and v_z/r with
    margins) takes the same discrete decisions as the contract's
    exact IEEE chain (IFGF_EXACT_CLASSIFY=1): identical relevant-segment counts,
    fields equal up to value rounding, both at oracle parity."""
    n, k, D = 20000, 6 * math.pi, 5
    pts = inputs.rough_sphere(n)
    a = inputs.densities(n, seed=13)
    monkeypatch.setenv("IFGF_EXACT_CLASSIFY", "1")
    _, exact, st_e = run_gpu(ifgf, pts, a, k, D)
    monkeypatch.setenv("IFGF_EXACT_CLASSIFY", "0")
    _, fast, st_f = run_gpu(ifgf, pts, a, k, D)
    assert st_e["nseg"] == st_f["nseg"] and st_e["cousin_evals"] == st_f["cousin_evals"]
    ref = oracle.OraclePlan(pts, k, D, 3, 5).apply(a)
    assert oracle.rel_l2(exact, ref) <= PARITY and oracle.rel_l2(fast, ref) <= PARITY
    assert oracle.rel_l2(fast, exact) <= 1e-13


@pytest.mark.parametrize("mode,umax,leaf_nc", [("5", None, 2), ("8", None, 2), ("5", "0", 2), ("5", None, 3),
                                               ("8", None, 3)])
def test_symmetry_orbit_grouping(ifgf, mode, umax, leaf_nc, monkeypatch):
    """K7 tensor-core kernels with segments grouped by quarter-turn orbits (one
    geometry for the four rotated parent cells, rotated child octants and cells)
    against the oracle and against the cell-only grouping.  leaf_nc = 3 makes the
    finest level's n_C odd (orbits disabled there, enabled above); umax = 0 sends
    every octant through the per-(segment, node) fallback."""
    monkeypatch.setenv("IFGF_LEGACY_UPWARD", mode)
    if umax is not None:
        monkeypatch.setenv("IFGF_TC_UMAX", umax)
    n, k, D = 20000, 6 * math.pi, 5
    pts = inputs.rough_sphere(n)
    a = inputs.densities(n, seed=11)
    monkeypatch.setenv("IFGF_NO_SYMMETRY", "0")
    _, got, _ = run_gpu(ifgf, pts, a, k, D, leaf_nc=leaf_nc)
    monkeypatch.setenv("IFGF_NO_SYMMETRY", "1")
    _, plain, _ = run_gpu(ifgf, pts, a, k, D, leaf_nc=leaf_nc)
    ref = oracle.OraclePlan(pts, k, D, 3, 5, leaf_nc=leaf_nc).apply(a)
    assert oracle.rel_l2(got, ref) <= PARITY
    assert oracle.rel_l2(got, plain) <= PARITY


# ------------------------------------------------------------ larger configs
@pytest.mark.slow
def test_cfg2_parity(ifgf):
    c = inputs.CONFIGS["cfg2"]
    pts, a = c.points(), c.densities()
    oplan = oracle.OraclePlan(pts, c.k, c.levels, c.Ps, c.Pang)
    ref = oplan.apply(a)
    plan, got, st = run_gpu(ifgf, pts, a, c.k, c.levels, c.Ps, c.Pang)
    assert oracle.rel_l2(got, ref) <= PARITY
    for d in range(3, c.levels + 1):
        assert st["nseg"][d] == oplan.level_info(d)["nseg"]
    tg = inputs.error_targets(c.n, 1000)
    exact = ifgf.direct(dev(pts), c.k, dev(a), dev(tg)).cpu().numpy()
    assert oracle.rel_l2(got[tg], exact) <= 1.1 * oracle.rel_l2(ref[tg], exact)


@pytest.mark.parametrize("mode,umax", [("1", None), ("3", None), ("5", None), ("5", "1"), ("5", "0"), ("7", None),
                                       ("8", None), ("8", "1")])
def test_upward_kernel_variants(ifgf, mode, umax, monkeypatch):
    """Every K7 kernel forced at every level matches the oracle (env
    IFGF_LEGACY_UPWARD: 1 per-evaluation geometry with per-lane global loads,
    3 cell-grouped shared-memory staged DFMA, 5 FP64 tensor-core GEMM on
    64-chunks, 7 warp-staged per-evaluation, 8 register-basis FP64 tensor-core
    GEMM on 32-chunks).  IFGF_TC_UMAX caps the child cells the tensor-core
    kernels stage per octant, so that their per-node fallback (taken near the
    poles) is exercised too.  The default (0) picks per level by segments per
    cell run."""
    monkeypatch.setenv("IFGF_LEGACY_UPWARD", mode)
    if umax is not None:
        monkeypatch.setenv("IFGF_TC_UMAX", umax)
    n = 20000
    pts = inputs.fibonacci_sphere(n, (1.0, 1.0, 0.5))
    a = inputs.densities(n, seed=21)
    k = 6 * math.pi
    _, got, _ = run_gpu(ifgf, pts, a, k, 5)
    ref = oracle.OraclePlan(pts, k, 5, 3, 5).apply(a)
    assert oracle.rel_l2(got, ref) <= PARITY


def lattice_shell(spacing=1.0 / 32, radius=0.8, width=1.0 / 40):
    """Points on the lattice -1 + m * spacing inside a thin spherical shell: with
    root box centre 0 and side 2 (x0 = -1), box faces and centres of every level
    lie on the same lattice, so relative vectors x - c_B hit exact ties of the
    interval rules (R7): poles (v_x = v_y = 0), v_z = 0 (theta = pi/2,
    a boundary of every even n_C), the phi = j pi/2 half-planes and the phi = pi/4
    diagonals (equal cos/sin table entries), and points on box faces."""
    m = np.arange(-int(1 / spacing), int(1 / spacing) + 1)
    g = -1.0 + (m + int(1 / spacing)) * spacing
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    P = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    r = np.linalg.norm(P, axis=1)
    return np.ascontiguousarray(P[np.abs(r - radius) < width])


@pytest.mark.parametrize("k,D", [(12.0, 5), (20.0, 6)])
def test_lattice_boundary_ties(ifgf, k, D):
    """Exact boundary ties of the classification against the oracle: identical
    relevant boxes and segment sets per level (plan-diff) and field parity."""
    pts = lattice_shell()
    root = ([0.0, 0.0, 0.0], 2.0)
    a = inputs.densities(len(pts), seed=41)
    plan, got, st = run_gpu(ifgf, pts, a, k, D, root=root)
    oplan = oracle.OraclePlan(pts, k, D, 3, 5, root=root)
    ref = oplan.apply(a)
    for d in range(1, D + 1):
        assert st["nbox"][d] == oplan.level_info(d)["nbox"]
        np.testing.assert_array_equal(segs_sorted(plan.level_segments(d)), segs_sorted(oplan.level_segments(d)))
    assert oracle.rel_l2(got, ref) <= PARITY
    # ties really occur: cousin points on the poles / on the phi half-planes of some box
    x0 = -1.0
    H = 2.0 / 2 ** (D - 1)
    q = np.floor((pts - x0) / H)
    c = x0 + (q + 0.5) * H
    assert np.any(pts[:, 0] == c[:, 0]) and np.any(pts[:, 2] == c[:, 2])
