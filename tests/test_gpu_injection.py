"""Exact pins of the K6 and K7 kernels in isolation (SURVEY.md §8(c) "exact pins",
pin 2: polynomial injection), through the C-ABI test hook ifgf_debug_level_pass.

Every relevant segment of a level d gets the node values of f_B p(s, theta, phi),
p a polynomial of degree < P_s in s and < P_ang in theta and phi (random complex
coefficients) and f_B a random complex factor per box.  The tensor Chebyshev
interpolant at first-kind nodes (R1) reproduces such a polynomial
exactly on every segment, so with no interpolation error:
  - K6 must return, for every target x,
        sum over cousin boxes B of x's level-d box of f_B p(s, theta, phi)(x - c_B) G(x, c_B);
  - K7 must produce, at every node y of every relevant parent
    segment, sum over children B of f_B p(...)(y - c_B) G(y, c_B) / G(y, c_Q).
The expected values are computed here with numpy from those formulas (no
classification, no interpolation), independently of both the CUDA path and the
oracle.  Every K6 and K7 kernel variant is forced in turn.
"""
import math

import numpy as np
import pytest

from paper_2010_02857_b200 import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ETA = math.sqrt(3.0) / 3.0


@pytest.fixture(scope="module")
def ifgf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2010_02857_b200 import ifgf as m
    return m


def cheb_nodes(n):
    return np.cos((2 * np.arange(n) + 1) * np.pi / (2 * n))


class Geo:
    def __init__(self, st):
        self.D, self.Ps, self.Pa, self.P, self.k = st["levels"], st["P_s"], st["P_ang"], st["P"], st["k"]
        self.H1 = st["root_side"]
        self.x0 = np.array(st["root_center"]) - self.H1 / 2
        self.grid = st["grid"]

    def H(self, d):
        return math.ldexp(self.H1, -(d - 1))

    def centre(self, d, ijk):
        return self.x0 + (np.asarray(ijk, dtype=np.float64) + 0.5) * self.H(d)

    def sph(self, d, v):
        """(s, theta, phi) of relative vectors v (eq. defparametrizationins)."""
        r = np.linalg.norm(v, axis=-1)
        s = (math.sqrt(3) / 2 * self.H(d)) / r
        th = np.arctan2(np.hypot(v[..., 0], v[..., 1]), v[..., 2])
        ph = np.mod(np.arctan2(v[..., 1], v[..., 0]), 2 * np.pi)
        return s, th, ph, r


class Poly:
    def __init__(self, Ps, Pa, seed):
        rng = np.random.default_rng(seed)
        self.c = rng.normal(size=(Ps, Pa, Pa)) + 1j * rng.normal(size=(Ps, Pa, Pa))

    def __call__(self, s, th, ph):
        Ps, Pa, _ = self.c.shape
        xs, xt, xp = s / ETA, th / np.pi, ph / (2 * np.pi)
        out = np.zeros(np.shape(s), dtype=np.complex128)
        for a in range(Ps):
            for b in range(Pa):
                for c in range(Pa):
                    out += self.c[a, b, c] * xs ** a * xt ** b * xp ** c
        return out


def box_factor(ijk, seed=99):
    """A complex factor per box (detects a read of another box's segment)."""
    i, j, k = (np.asarray(ijk, dtype=np.int64).T)
    h = (i * 73856093) ^ (j * 19349663) ^ (k * 83492791) ^ seed
    return np.exp(1j * (h % 1000) / 1000.0 * 2 * np.pi) * (1.0 + (h % 7) / 7.0)


def node_values(g, d, segs, poly):
    """f_B p(s, theta, phi) at the nodes of every segment (s-fastest layout)."""
    ns, nC = g.grid[d]
    cell = segs[:, 3]
    i_s, i_t, i_p = cell % ns, (cell // ns) % nC, cell // (ns * nC)
    ts, ta = cheb_nodes(g.Ps), cheb_nodes(g.Pa)
    ds, dth = ETA / ns, np.pi / nC
    s = (i_s[:, None] + (1 + ts[None, :]) / 2) * ds          # [seg, Ps]
    th = (i_t[:, None] + (1 + ta[None, :]) / 2) * dth        # [seg, Pa]
    ph = (i_p[:, None] + (1 + ta[None, :]) / 2) * dth        # [seg, Pa]
    S = s[:, None, None, :]
    TH = th[:, None, :, None]
    PH = ph[:, :, None, None]                                # [seg, c, b, a]
    v = poly(np.broadcast_to(S, (len(segs), g.Pa, g.Pa, g.Ps)), np.broadcast_to(TH, (len(segs), g.Pa, g.Pa, g.Ps)),
             np.broadcast_to(PH, (len(segs), g.Pa, g.Pa, g.Ps)))
    return (v * box_factor(segs[:, :3])[:, None, None, None]).reshape(len(segs), -1)


def level_boxes(g, pts, d):
    q = np.clip(np.floor((pts - g.x0) / g.H(d)), 0, 2 ** (d - 1) - 1).astype(np.int64)
    boxes, inv = np.unique(q, axis=0, return_inverse=True)
    return boxes, inv.reshape(-1)


def expected_cousin_field(g, pts, d, poly, have_segs):
    boxes, inv = level_boxes(g, pts, d)
    out = np.zeros(len(pts), dtype=np.complex128)
    par = boxes >> 1
    for t in range(len(boxes)):
        tgt = np.nonzero(inv == t)[0]
        near_par = np.max(np.abs(par - par[t]), axis=1) <= 1
        far = np.max(np.abs(boxes - boxes[t]), axis=1) >= 2
        for b in np.nonzero(near_par & far)[0]:
            key = tuple(boxes[b])
            assert key in have_segs  # every cousin source box has relevant segments
            v = pts[tgt] - g.centre(d, boxes[b])
            s, th, ph, r = g.sph(d, v)
            G = np.exp(1j * g.k * r) / (4 * np.pi * r)
            out[tgt] += box_factor(boxes[b][None, :])[0] * poly(s, th, ph) * G
    return out


def expected_parent_values(g, pts, d, poly, psegs):
    """Node values of level d-1's relevant segments after the upward pass from level d."""
    dp = d - 1
    boxes, _ = level_boxes(g, pts, d)
    nsP, nCP = g.grid[dp]
    ts, ta = cheb_nodes(g.Ps), cheb_nodes(g.Pa)
    dsP, dthP = ETA / nsP, np.pi / nCP
    cell = psegs[:, 3]
    i_s, i_t, i_p = cell % nsP, (cell // nsP) % nCP, cell // (nsP * nCP)
    s = (i_s[:, None, None, None] + (1 + ts[None, None, None, :]) / 2) * dsP
    th = (i_t[:, None, None, None] + (1 + ta[None, None, :, None]) / 2) * dthP
    ph = (i_p[:, None, None, None] + (1 + ta[None, :, None, None]) / 2) * dthP
    s, th, ph = np.broadcast_arrays(s, th, ph)                  # [seg, c, b, a]
    rQ = (math.sqrt(3) / 2 * g.H(dp)) / s
    off = np.stack([rQ * np.sin(th) * np.cos(ph), rQ * np.sin(th) * np.sin(ph), rQ * np.cos(th)], axis=-1)
    cQ = g.centre(dp, psegs[:, :3])[:, None, None, None, :]
    y = cQ + off
    out = np.zeros(s.shape, dtype=np.complex128)
    bkeys = {tuple(b): b for b in boxes}
    for o in range(8):
        oi = np.array([(o >> 2) & 1, (o >> 1) & 1, o & 1])
        child = psegs[:, :3] * 2 + oi
        has = np.array([tuple(c) in bkeys for c in child])
        if not has.any():
            continue
        cB = g.centre(d, child[has])[:, None, None, None, :]
        v = y[has] - cB
        sB, thB, phB, rB = g.sph(d, v)
        rec = (rQ[has] / rB) * np.exp(1j * g.k * (rB - rQ[has]))
        out[has] += box_factor(child[has])[:, None, None, None] * poly(sB, thB, phB) * rec
    return out.reshape(len(psegs), -1)


def coeffs_to_node_values(C, Ps, Pa):
    """Tensor Chebyshev series -> values at the first-kind node grid (s-fastest)."""
    Ts = np.polynomial.chebyshev.chebvander(cheb_nodes(Ps), Ps - 1)  # [node, coef]
    Ta = np.polynomial.chebyshev.chebvander(cheb_nodes(Pa), Pa - 1)
    Cr = C.reshape(-1, Pa, Pa, Ps)                                    # [seg, c, b, a]
    return np.einsum("zcba,ka,jb,ic->zijk", Cr, Ts, Ta, Ta).reshape(len(C), -1)


@pytest.fixture(scope="module")
def case(ifgf):
    n, k, D = 20_000, 6 * math.pi, 5
    pts = inputs.rough_sphere(n)
    return n, k, D, pts


def _plan(ifgf, pts, k, D):
    return ifgf.Plan(torch.from_numpy(pts).to("cuda:0"), k, D, 3, 5)


@pytest.mark.parametrize("legacy", ["0", "1"])
@pytest.mark.parametrize("d", [5, 4, 3])
def test_k6_polynomial_injection(ifgf, case, d, legacy, monkeypatch):
    monkeypatch.setenv("IFGF_LEGACY_COUSIN", legacy)
    n, k, D, pts = case
    plan = _plan(ifgf, pts, k, D)
    g = Geo(plan.stats())
    poly = Poly(g.Ps, g.Pa, seed=d)
    segs = plan.level_segments(d)
    vals = node_values(g, d, segs, poly)
    field, _ = plan.debug_level_pass(d, vals, cousin=True, upward=False)
    have = {tuple(b) for b in segs[:, :3]}
    exp = expected_cousin_field(g, pts, d, poly, have)
    err = np.max(np.abs(field - exp)) / np.max(np.abs(exp))
    assert err <= 1e-12, err


@pytest.mark.parametrize("mode", ["0", "5", "8", "3", "7", "1"])
@pytest.mark.parametrize("d", [5, 4])
def test_k7_polynomial_injection(ifgf, case, d, mode, monkeypatch):
    """Forced K7 variants (IFGF_LEGACY_UPWARD): 0 default per-level choice, 5 FP64
    tensor core (shared-memory basis), 8 tensor core v2 (register basis), 3 staged
    DFMA, 7 warp-staged per-evaluation, 1 per-evaluation with global loads."""
    monkeypatch.setenv("IFGF_LEGACY_UPWARD", mode)
    n, k, D, pts = case
    plan = _plan(ifgf, pts, k, D)
    st = plan.stats()
    g = Geo(st)
    poly = Poly(g.Ps, g.Pa, seed=10 + d)
    vals = node_values(g, d, plan.level_segments(d), poly)
    _, parent = plan.debug_level_pass(d, vals, cousin=False, upward=True)
    psegs = plan.level_segments(d - 1)
    exp = expected_parent_values(g, pts, d, poly, psegs)
    got = coeffs_to_node_values(parent, g.Ps, g.Pa)
    err = np.max(np.abs(got - exp)) / np.max(np.abs(exp))
    assert err <= 1e-12, (err, st["upward_kernel"])
