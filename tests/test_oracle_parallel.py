"""Pins of the oracle's parallel, target-/parent-segment-major loop order and of
its source partition (SURVEY.md §8(c) "Oracle data layout and cost", §8(e)).
CPU only.

- The OpenMP mode is bitwise equal to the serial mode (one owner per output,
  terms in increasing source-box order; oracle/ifgf_oracle.cpp header).
- The fast classification (bisection for i_theta, atan2 guess verified by the
  defining cross-product condition for i_phi) takes exactly the decisions of the
  literal interval scans of the classification contract (DESIGN.md §3,
  eq. defconedomain), including exact boundary ties.
- A plan owning a Morton range of leaves returns exactly the field of the
  densities zeroed outside those leaves (linearity of eq. field1).
"""
import math

import numpy as np
import pytest

import oracle
from paper_2010_02857_b200 import inputs


def _morton(i, j, k):
    r = 0
    for b in range(21):
        r |= ((i >> b) & 1) << (3 * b + 2) | ((j >> b) & 1) << (3 * b + 1) | ((k >> b) & 1) << (3 * b)
    return r


@pytest.fixture(autouse=True)
def _restore_threads():
    yield
    oracle.set_threads(0)


@pytest.mark.parametrize("case", ["cfg1", "d6"])
def test_parallel_bitwise_equals_serial(case):
    if case == "cfg1":
        c = inputs.CONFIGS["cfg1"]
        pts, a, k, D, Ps, Pa = c.points(), c.densities(), c.k, c.levels, c.Ps, c.Pang
    else:
        n = 12_000
        pts, a, k, D, Ps, Pa = inputs.fibonacci_sphere(n), inputs.densities(n), 8 * math.pi, 6, 3, 5
    res = {}
    for th in (1, 3, 8):
        oracle.set_threads(th)
        plan = oracle.OraclePlan(pts, k, D, Ps, Pa)
        res[th] = (plan.apply(a), [plan.level_segments(d) for d in range(3, D + 1)])
    for th in (3, 8):
        assert np.array_equal(res[th][0].view(np.float64), res[1][0].view(np.float64)), th
        for s1, s in zip(res[1][1], res[th][1]):
            assert np.array_equal(s1, s)


def _tie_vectors(H, ns, nC, rng):
    """Relative vectors on the boundaries of the (s, theta, phi) intervals:
    poles, v_z = 0, phi = j pi/nC rays (incl. the quarter-turn half-planes),
    theta = k pi/nC cones and s on multiples of Delta_s."""
    h = math.sqrt(3) / 2 * H
    eta = math.sqrt(3) / 3
    ds, dth = eta / ns, math.pi / nC
    out = []
    radii = [h / (m * ds) for m in range(1, ns + 1)] + [h / rng.uniform(1e-3, eta) for _ in range(3)]
    for r in radii:
        out += [[0.0, 0.0, r], [0.0, 0.0, -r]]
        for j in range(2 * nC):
            ph = j * dth
            for z in (0.0, 0.3 * r, -0.7 * r):
                rho = math.sqrt(max(r * r - z * z, 0.0))
                out.append([rho * math.cos(ph), rho * math.sin(ph), z])
            out += [[r * math.cos(ph), r * math.sin(ph), 0.0]]
        for kk in range(nC + 1):
            th = kk * dth
            ph = rng.uniform(0, 2 * math.pi)
            out.append([r * math.sin(th) * math.cos(ph), r * math.sin(th) * math.sin(ph), r * math.cos(th)])
    for q in range(4):  # exact quarter-turn half-planes: x = 0 or y = 0
        out += [[0.0, 1.0, 0.5], [1.0, 0.0, -0.5], [0.0, -2.0, 0.1], [-2.0, 0.0, 0.1]]
    return out


@pytest.mark.parametrize("ns,nC", [(1, 2), (2, 4), (4, 8), (16, 32), (128, 256), (3, 5)])
def test_fast_classification_equals_interval_scans(ns, nC):
    rng = np.random.default_rng(ns * 1000 + nC)
    H = 0.75
    vecs = _tie_vectors(H, ns, nC, rng)
    d = rng.normal(size=(3000, 3))
    vecs += list(d * (H * 10 ** rng.uniform(-0.1, 2, size=(3000, 1))))
    for v in vecs:
        cell, _ = oracle.classify(H, ns, nC, v)
        assert cell[0] >= 0, (v, "fast classification differs from the literal scans")
        assert 0 <= cell[1] < nC and 0 <= cell[2] < 2 * nC


def test_partition_equals_masked_densities():
    n, k, D = 20_000, 8 * math.pi, 5
    pts, a = inputs.fibonacci_sphere(n), inputs.densities(n)
    full = oracle.OraclePlan(pts, k, D, 3, 5)
    keys = np.array(sorted(_morton(*map(int, b[:3])) for b in full.level_boxes(D)))
    info = full.level_info(D)
    q = np.clip(np.floor((pts - info["x0"]) / info["H"]).astype(np.int64), 0, 2 ** (D - 1) - 1)
    mk = np.array([_morton(*map(int, x)) for x in q], dtype=np.uint64)
    parts = [0, len(keys) // 4, len(keys) // 2, len(keys)]
    acc = np.zeros(n, dtype=np.complex128)
    for r in range(3):
        lo = int(keys[parts[r]])
        hi = int(keys[parts[r + 1]]) if parts[r + 1] < len(keys) else 2 ** 64 - 1
        mine = (mk >= lo) & (mk < hi)
        part = oracle.OraclePlan(pts, k, D, 3, 5, owned_morton=(lo, hi))
        got = part.apply(a)
        # exact: the skipped boxes contribute exact zeros (equality ignores the sign of zero)
        assert np.array_equal(got, full.apply(np.where(mine, a, 0.0)))
        # the partition's relevant segments are those of its boxes in the full plan
        for d in range(3, D + 1):
            sp = {tuple(s) for s in part.level_segments(d)}
            boxes = {s[:3] for s in sp}
            sf = {tuple(s) for s in full.level_segments(d) if tuple(s[:3]) in boxes}
            assert sp == sf
        acc += got
    assert oracle.rel_l2(acc, full.apply(a)) < 1e-14
