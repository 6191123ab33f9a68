"""Algorithm-level pins of the oracle (Algorithm 1) against brute
force, exact special cases, invariants and the paper's printed errors.  CPU only.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2010_02857_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def cfg1():
    c = inputs.CONFIGS["cfg1"]
    pts, a = c.points(), c.densities()
    plan = oracle.OraclePlan(pts, c.k, c.levels, c.Ps, c.Pang)
    return c, pts, a, plan, plan.apply(a)


def small_sphere(n=3000, k=4 * math.pi, D=4, Ps=3, Pa=5, seed=5):
    pts = inputs.fibonacci_sphere(n)
    a = inputs.densities(n, seed)
    return pts, a, oracle.OraclePlan(pts, k, D, Ps, Pa)


# ------------------------------------------------------------ box tree (L2)
def test_tree_partition_and_brute_force_boxes():
    """Relevant boxes: every point in exactly one box per level and
    that box is the one a linear scan over all level-d boxes finds (eq. defbox,
    half-open)."""
    pts, a, p = small_sphere(n=700, D=4)
    for d in range(1, 5):
        info = p.level_info(d)
        boxes = p.level_boxes(d)
        assert boxes[:, 3].sum() == len(pts)
        H, x0 = info["H"], info["x0"]
        nb = 2 ** (d - 1)
        for m in range(0, len(pts), 37):
            hits = []
            for i in range(nb):
                for j in range(nb):
                    for k in range(nb):
                        lo = x0 + np.array([i, j, k]) * H
                        if np.all(pts[m] >= lo) and np.all(pts[m] < lo + H):
                            hits.append((i, j, k))
            assert len(hits) == 1
            assert any((b[0], b[1], b[2]) == hits[0] for b in boxes)


def test_neighbours_cousins_brute_force():
    """N B and M B (eq. defcousinboxes) recomputed here
    from the box multi-indices; symmetry; |M B| <= 189; no cousins
    at levels 1-2."""
    pts, a, p = small_sphere(n=2000, D=5)
    for d in range(1, 6):
        boxes = p.level_boxes(d)
        keys = [tuple(b[:3]) for b in boxes]
        kset = set(keys)
        for bi, kb in enumerate(keys):
            nb = {keys[i] for i in p.box_list(d, bi, "nbrs")}
            ref_nb = {x for x in kset if max(abs(x[t] - kb[t]) for t in range(3)) <= 1}
            assert nb == ref_nb
            co = {keys[i] for i in p.box_list(d, bi, "cousins")}
            par = tuple(v >> 1 for v in kb)
            ref_co = {x for x in kset
                      if max(abs((x[t] >> 1) - par[t]) for t in range(3)) <= 1
                      and max(abs(x[t] - kb[t]) for t in range(3)) >= 2} if d >= 2 else set()
            assert co == ref_co
            assert len(co) <= 189
            if d <= 2:
                assert not co
        for bi in range(len(keys)):
            for ci in p.box_list(d, bi, "cousins"):
                assert bi in set(p.box_list(d, int(ci), "cousins"))


def test_cone_grid_schedule():
    """Readings R5/R6/R8: (n_s,n_C)_D = (1,2), doubling per level while kappa H_{d-1} > 1;
    kappa = 0 keeps the grid constant."""
    pts = inputs.fibonacci_sphere(500)
    p = oracle.OraclePlan(pts, 4 * math.pi, 4, 3, 5)
    assert [(p.level_info(d)["ns"], p.level_info(d)["nC"]) for d in (3, 4)] == [(2, 4), (1, 2)]
    p0 = oracle.OraclePlan(pts, 0.0, 5, 3, 5)
    assert {(p0.level_info(d)["ns"], p0.level_info(d)["nC"]) for d in range(1, 6)} == {(1, 2)}


def test_relevant_segment_counts_cfg1(cfg1):
    """|R_C^d| at cfg1 matches the independent work-structure count of SURVEY.md
    §8(a) (1.3k, 1.9k for levels 3, 4); levels 1-2 have none."""
    c, pts, a, p, I = cfg1
    assert p.level_info(1)["nseg"] == 0 and p.level_info(2)["nseg"] == 0
    assert abs(p.level_info(3)["nseg"] - 1300) < 100
    assert abs(p.level_info(4)["nseg"] - 1900) < 100
    # leaf grid 1 x 2 x 4: at most 8 segments per leaf
    assert p.level_info(4)["nseg"] <= 8 * p.level_info(4)["nbox"]


# ------------------------------------------------------- whole algorithm (L3)
def test_bypass_equals_direct_sum():
    """Interpolation-bypass mode (every Interp F_B replaced by the exact F_B of
    eq. I_k) must equal the direct sum eq. field1: pins level loops, neighbour
    and cousin lists, self-exclusion and 'every pair exactly once'."""
    pts, a, p = small_sphere(n=2500, D=5)
    I = p.apply(a, mode=oracle.MODE_BYPASS)
    ref = oracle.direct(pts, p.k, a, np.arange(len(pts)))
    assert oracle.rel_l2(I, ref) < 1e-13


def test_near_stage_equals_restricted_direct_sum():
    """Stage NEAR = sum over m in U(box of l), m != l, brute force."""
    pts, a, p = small_sphere(n=1200, D=4)
    I = p.apply(a, stage_mask=oracle.ST_NEAR)
    info = p.level_info(4)
    q = np.clip(np.floor((pts - info["x0"]) / info["H"]).astype(np.int64), 0, 7)
    ref = np.zeros(len(pts), dtype=complex)
    for l in range(0, len(pts), 7):
        near = np.max(np.abs(q - q[l]), axis=1) <= 1
        near[l] = False
        r = np.linalg.norm(pts[near] - pts[l], axis=1)
        ref[l] = np.sum(a[near] * np.exp(1j * p.k * r) / (4 * np.pi * r))
    sel = np.arange(0, len(pts), 7)
    assert oracle.rel_l2(I[sel], ref[sel]) < 1e-13


def test_centred_source_exact():
    """Exact pin with no interpolation error: one unit source exactly at a leaf
    centre (g_B(., c_B) = 1), D = 3 (no upward pass): IFGF = G(x, c_B)."""
    rng = np.random.default_rng(4)
    pts = rng.uniform(-1.99, 1.99, (600, 3))
    pts[0] = [0.5, 0.5, -0.5]  # centre of a level-3 box for root centre 0, side 4
    a = np.zeros(len(pts), dtype=complex)
    a[0] = 1.0
    k = 3.0
    p = oracle.OraclePlan(pts, k, 3, 3, 5, root=([0.0, 0.0, 0.0], 4.0))
    I = p.apply(a)
    ref = oracle.direct(pts, k, a, np.arange(len(pts)))
    assert oracle.rel_l2(I, ref) < 1e-14


def test_recentering_exact():
    """Exact-upward check: sum_B F_B(y) G(y,c_B)/G(y,c_Q) = F_Q(y) at every node of
    every relevant parent segment."""
    pts, a, p = small_sphere(n=1500, D=5)
    assert p.recentering_check(a) < 1e-11


def test_error_vs_direct_cfg1_and_convergence(cfg1):
    """IFGF vs the direct sum on 1000 seeded targets (eq. errorcomputation
    P:2022-2028): cfg1 (0.5 lambda leaves) is in the paper's 1e-4..2e-3 band
    (Table timings1); the error decreases as (P_s, P_ang) grows (Theorem
    errorestimatenested P:732-746)."""
    c, pts, a, p, I = cfg1
    tg = inputs.error_targets(c.n, 1000)
    ex = oracle.direct(pts, c.k, a, tg)
    e35 = oracle.rel_l2(I[tg], ex)
    assert 1e-4 < e35 < 5e-3
    p57 = oracle.OraclePlan(pts, c.k, c.levels, 5, 7)
    e57 = oracle.rel_l2(p57.apply(a)[tg], ex)
    assert e57 < e35 / 5


@pytest.mark.slow
def test_paper_anchor_table1_row1():
    """cfg1 points at the paper's leaf size H_D ~ lambda/4 (D = 5):
    eps_1000 within a factor 3 of Table timings1 row 1 (3.57e-4)."""
    with open(os.path.join(GOLD, "paper_errors.json")) as f:
        paper = json.load(f)["table_timings1_sphere_Ps3_Pang5"]["rows"][0]["eps"]
    c = inputs.CONFIGS["cfg1"]
    pts, a = c.points(), c.densities()
    tg = inputs.error_targets(c.n, 1000)
    e = oracle.rel_l2(oracle.OraclePlan(pts, c.k, 5, 3, 5).apply(a)[tg], oracle.direct(pts, c.k, a, tg))
    assert paper / 3 < e < paper * 3


def test_linearity(cfg1):
    """apply(alpha a + beta b) = alpha apply(a) + beta apply(b) (eq. field1 is linear)."""
    c, pts, a, p, I = cfg1
    b = inputs.densities(c.n, seed=99)
    al, be = 0.3 - 1.2j, -2.0 + 0.5j
    lhs = p.apply(al * a + be * b)
    rhs = al * I + be * p.apply(b)
    assert oracle.rel_l2(lhs, rhs) < 1e-12


def test_metamorphic_rotation_and_reflection():
    """Rotation (x,y,z)->(-y,x,z) maps boxes to boxes and phi-sectors to phi-sectors
    (pi/2 is a multiple of pi/n_C); reflection z->-z maps theta-intervals to
    theta-intervals.  Both must leave the field unchanged."""
    pts, a, p = small_sphere(n=2000, D=4, seed=8)
    I = p.apply(a)
    rot = np.stack([-pts[:, 1], pts[:, 0], pts[:, 2]], axis=1)
    ref = np.stack([pts[:, 0], pts[:, 1], -pts[:, 2]], axis=1)
    for q in (rot, ref):
        J = oracle.OraclePlan(q, p.k, 4, 3, 5).apply(a)
        assert oracle.rel_l2(J, I) < 1e-12


def test_laplace_kappa_zero():
    """kappa = 0 (Laplace, reading R4): constant (1,2) grids at every level; the
    error decreases with (P_s, P_ang) and reaches the order of Table
    timingsLaplace (1.5e-5; the paper does not state its Laplace orders)."""
    pts = inputs.fibonacci_sphere(6000)
    a = inputs.densities(6000)
    tg = inputs.error_targets(6000, 500)
    ex = oracle.direct(pts, 0.0, a, tg)
    e35 = oracle.rel_l2(oracle.OraclePlan(pts, 0.0, 5, 3, 5).apply(a)[tg], ex)
    e57 = oracle.rel_l2(oracle.OraclePlan(pts, 0.0, 5, 5, 7).apply(a)[tg], ex)
    assert e35 < 2e-3
    assert e57 < 5e-5


# ------------------------------------------------------------- degenerate cases
def test_degenerate_cases():
    """N = 1 -> 0; N = 2 closed form (eq. field1); D <= 2 -> pure direct sum
    (P:1595-1600); coincident points and zero extent -> EDOMAIN;
    bad arguments -> EINVAL."""
    one = oracle.OraclePlan([[0.3, 0.1, 0.2]], 5.0, 3, 3, 5)
    assert np.all(one.apply(np.array([1 + 1j])) == 0)
    two = np.array([[0.0, 0, 0], [0.7, 0.2, -0.1]])
    a2 = np.array([1 - 2j, 0.5 + 0.25j])
    g = oracle.green(two[0], two[1], 3.0)
    I = oracle.OraclePlan(two, 3.0, 2, 3, 5).apply(a2)  # D = 2: the two leaves are neighbours
    np.testing.assert_allclose(I, [a2[1] * g, a2[0] * g], rtol=1e-15)
    I = oracle.OraclePlan(two, 3.0, 4, 3, 5).apply(a2)  # D = 4: level-3 cousins, interpolated
    np.testing.assert_allclose(I, [a2[1] * g, a2[0] * g], rtol=1e-2)
    pts = inputs.fibonacci_sphere(400)
    a = inputs.densities(400)
    for D in (1, 2):
        I = oracle.OraclePlan(pts, 6.0, D, 3, 5).apply(a)
        assert oracle.rel_l2(I, oracle.direct(pts, 6.0, a, np.arange(400))) < 1e-14
    with pytest.raises(oracle.OracleError) as e:
        oracle.OraclePlan(np.array([[0.0, 0, 0], [1, 1, 1], [0, 0, 0]]), 1.0, 3, 3, 5)
    assert e.value.code == 2
    with pytest.raises(oracle.OracleError) as e:
        oracle.OraclePlan(np.zeros((3, 3)), 1.0, 3, 3, 5)
    assert e.value.code == 2
    for bad in [dict(k=-1.0), dict(k=float("nan")), dict(levels=0), dict(levels=23), dict(Ps=0)]:
        kw = dict(k=1.0, levels=3, Ps=3, Pang=5)
        kw.update(bad)
        with pytest.raises(oracle.OracleError) as e:
            oracle.OraclePlan(pts, **kw)
        assert e.value.code == 1
