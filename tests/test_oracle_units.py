"""Pins of the oracle's building blocks against closed forms, textbook identities
and brute force (task rule ③).  CPU only.

Each test names the PAPER.md passage (P:n) the pinned function follows.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- kernel math
def test_green_closed_forms():
    """eq. greensfunction at hand-evaluated points."""
    for e in _gold("closed_forms.json")["green"]:
        g = oracle.green(e["x"], e["y"], e["k"])
        assert abs(g - complex(e["re"], e["im"])) <= 1e-15, e["_cite"]


def test_analytic_factor_closed_forms():
    """eq. factored_f: -(4/3)i example and g(x, c, c) = 1."""
    for e in _gold("closed_forms.json")["analytic_factor"]:
        g = oracle.analytic_factor(e["x"], e["xp"], e["c"], e["k"])
        assert abs(g - complex(e["re"], e["im"])) <= 2e-15, e["_cite"]


def test_factorization_identity():
    """eq. factor: G(x,x') = G(x,x_S) g_S(x,x') for x' in the box and
    x at least H away (pairs in A_eta^H).  G(x,x') is computed by the plain kernel
    (an independent formula), the right-hand side by the two factors."""
    rng = np.random.default_rng(1)
    worst = 0.0
    for _ in range(4000):
        H = 10 ** rng.uniform(-3, 0)
        c = rng.uniform(-1, 1, 3)
        xp = c + rng.uniform(-H / 2, H / 2, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        x = c + d * H * 10 ** rng.uniform(0.2, 3)
        k = 10 ** rng.uniform(-1, 3)
        k = min(k, 2000.0 / np.linalg.norm(x - xp))  # phases up to 2e3 rad (cfg5 scale)
        lhs = oracle.green(x, xp, k)
        rhs = oracle.green(x, c, k) * oracle.analytic_factor(x, xp, c, k)
        worst = max(worst, abs(lhs - rhs) / abs(lhs))
    # the phase k|x-x'| <= 2e3 rad: its rounding (2e3 * 2^-53 per ulp) bounds the agreement
    assert worst < 5e-12


def test_recenter_closed_form_and_identity():
    """Recentering factor G(y,c_B)/G(y,c_Q).
    off=(2,0,0) from c_Q, delta=c_Q-c_B=(-0.5,0,0): r_B=1.5, r_Q=2, kappa=pi ->
    (2/1.5) e^{i pi (1.5-2)} = -(4/3) i."""
    g = oracle.recenter([2.0, 0, 0], [-0.5, 0, 0], math.pi)
    assert abs(g - (-4j / 3)) < 2e-15
    rng = np.random.default_rng(2)
    for _ in range(500):
        cQ = rng.uniform(-1, 1, 3)
        delta = rng.choice([-1.0, 1.0], 3) * 0.125
        off = rng.normal(size=3)
        off *= 10 ** rng.uniform(-0.3, 2) / np.linalg.norm(off)
        k = 10 ** rng.uniform(0, 2.5)
        y = cQ + off
        cB = cQ - delta
        ref = oracle.green(y, cB, k) / oracle.green(y, cQ, k)
        got = oracle.recenter(off, delta, k)
        # reference phase carries k*ulp(|y|) rounding; the tested form does not
        assert abs(got - ref) / abs(ref) < 1e-11


# ------------------------------------------------------------- Chebyshev (L1)
def test_cheb_nodes_closed_form():
    """P:697-698 first-kind nodes."""
    for e in _gold("closed_forms.json")["cheb_nodes"]:
        np.testing.assert_allclose(oracle.cheb_nodes(e["n"]), e["t"], rtol=0, atol=1e-16)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 9])
def test_cheb_node_reproduction_and_exactness(n):
    """The interpolant (reading R1) reproduces node values and every polynomial of
    degree < n (numpy.polynomial evaluates the reference polynomial)."""
    rng = np.random.default_rng(n)
    t = oracle.cheb_nodes(n)
    u = rng.normal(size=n) + 1j * rng.normal(size=n)
    a = oracle.cheb_fit1d(u)
    for k in range(n):
        assert abs(oracle.cheb_eval1d(a, t[k]) - u[k]) < 1e-14
    coef = rng.normal(size=n) + 1j * rng.normal(size=n)  # power-basis coefficients
    a = oracle.cheb_fit1d(np.polynomial.polynomial.polyval(t, coef))
    for x in rng.uniform(-1, 1, 50):
        assert abs(oracle.cheb_eval1d(a, x) - np.polynomial.polynomial.polyval(x, coef)) < 1e-13


def test_cheb_T2_coefficients():
    """u = T_2 sampled at n >= 3 nodes -> coefficient vector e_2 (orthogonality)."""
    n = 5
    t = oracle.cheb_nodes(n)
    a = oracle.cheb_fit1d(2 * t * t - 1)
    np.testing.assert_allclose(a, [0, 0, 1, 0, 0], atol=1e-15)


def test_eq19_bound_exp():
    """eq. errorestimatechebinterpolation for u = e^x, n = 5, [0,1]:
    max error over 10^4 points is below e/(2^9 5!) and not vacuous."""
    n = 5
    t = oracle.cheb_nodes(n)
    a = oracle.cheb_fit1d(np.exp((t + 1) / 2))
    xs = np.linspace(0, 1, 10_001)
    err = max(abs(oracle.cheb_eval1d(a, 2 * x - 1) - math.exp(x)) for x in xs)
    bound = _gold("closed_forms.json")["eq19_bound_exp_n5_on_0_1"]["bound"]
    assert err <= bound
    assert err > bound / 100  # the bound is sharp to within ~1 decade


@pytest.mark.parametrize("Ps,Pa", [(3, 5), (5, 5), (2, 3)])
def test_tensor_monomial_exactness(Ps, Pa):
    """Nested interpolation (Theorem errorestimatenested) reproduces every
    tensor monomial u_s^a u_t^b u_p^c with a < P_s, b,c < P_ang."""
    ts, ta = oracle.cheb_nodes(Ps), oracle.cheb_nodes(Pa)
    rng = np.random.default_rng(7)
    for (ea, eb, ec) in [(0, 0, 0), (Ps - 1, Pa - 1, Pa - 1), (1 % Ps, 0, Pa - 1), (Ps - 1, Pa // 2, 1 % Pa)]:
        V = np.zeros(Ps * Pa * Pa, dtype=complex)
        for jp in range(Pa):
            for it in range(Pa):
                for ks in range(Ps):
                    V[(jp * Pa + it) * Ps + ks] = (1 + 2j) * ts[ks] ** ea * ta[it] ** eb * ta[jp] ** ec
        C = oracle.tensor_fit(Ps, Pa, V)
        for _ in range(20):
            us, ut, up = rng.uniform(-1, 1, 3)
            ref = (1 + 2j) * us ** ea * ut ** eb * up ** ec
            assert abs(oracle.tensor_eval(Ps, Pa, C, us, ut, up) - ref) < 1e-13


def test_tensor_separable_outer_product():
    """Separable data -> coefficient tensor = outer product of 1-D coefficients."""
    Ps, Pa = 3, 5
    rng = np.random.default_rng(3)
    f, g, h = rng.normal(size=Ps), rng.normal(size=Pa), rng.normal(size=Pa) + 1j * rng.normal(size=Pa)
    V = np.einsum("j,i,k->jik", h, g, f).reshape(-1)
    C = oracle.tensor_fit(Ps, Pa, V).reshape(Pa, Pa, Ps)
    ref = np.einsum("j,i,k->jik", oracle.cheb_fit1d(h), oracle.cheb_fit1d(g), oracle.cheb_fit1d(f))
    np.testing.assert_allclose(C, ref, atol=1e-14)


# --------------------------------------------------- cone segments
def _angles(v):
    r = np.linalg.norm(v)
    th = math.atan2(math.hypot(v[0], v[1]), v[2])
    ph = math.atan2(v[1], v[0]) % (2 * math.pi)
    return r, th, ph


def test_classify_brute_force():
    """Segment index = the interval scan of (s, theta, phi) (eqs defconedomain,
    defconesegments); local coordinates lie in [-1,1] and map back to the angle."""
    rng = np.random.default_rng(11)
    eta = math.sqrt(3) / 3
    for (ns, nC) in [(1, 2), (2, 4), (8, 16), (64, 128)]:
        H = 0.37
        h = math.sqrt(3) / 2 * H
        for _ in range(400):
            d = rng.normal(size=3)
            d /= np.linalg.norm(d)
            r = h / rng.uniform(1e-3, eta)
            v = d * r
            (is_, it, ip), loc = oracle.classify(H, ns, nC, v)
            _, th, ph = _angles(v)
            s = h / r
            assert is_ == min(int(s / (eta / ns)), ns - 1)
            assert it == min(int(th / (math.pi / nC)), nC - 1)
            assert ip == min(int(ph / (math.pi / nC)), 2 * nC - 1)
            assert np.all(np.abs(loc[:3]) <= 1 + 1e-9)
            assert abs((it + (1 + loc[1]) / 2) * math.pi / nC - th) < 1e-12
            assert abs((ip + (1 + loc[2]) / 2) * math.pi / nC - ph) < 1e-12


def test_classify_poles_and_axes():
    """Poles get phi := 0 (reading R7); theta = pi closes the last interval."""
    H, ns, nC = 1.0, 2, 4
    (is_, it, ip), _ = oracle.classify(H, ns, nC, [0, 0, 2.0])
    assert (it, ip) == (0, 0)
    (is_, it, ip), _ = oracle.classify(H, ns, nC, [0, 0, -2.0])
    assert (it, ip) == (nC - 1, 0)
    # +x axis: phi = 0 -> sector 0; -x axis: phi = pi -> sector nC (lower-closed)
    assert oracle.classify(H, ns, nC, [3.0, 0, 0])[0][2] == 0
    assert oracle.classify(H, ns, nC, [-3.0, 0, 0])[0][2] == nC
    # s = eta exactly is clamped into the last radial interval
    h = math.sqrt(3) / 2 * H
    (is_, _, _), _ = oracle.classify(H, ns, nC, [1.5 * H, 0, 0])
    assert is_ == ns - 1 and abs(h / (1.5 * H) - math.sqrt(3) / 3) < 1e-15


@pytest.mark.parametrize("ns,nC,Ps,Pa", [(1, 2, 3, 5), (4, 8, 3, 5), (16, 32, 5, 5)])
def test_nodes_lie_in_their_segment(ns, nC, Ps, Pa):
    """Interpolation points (eq. interp_pts) classify into their own
    segment with local coordinates equal to the reference nodes."""
    rng = np.random.default_rng(ns)
    H = 0.25
    ts, ta = oracle.cheb_nodes(Ps), oracle.cheb_nodes(Pa)
    for _ in range(30):
        cell = (int(rng.integers(ns)), int(rng.integers(nC)), int(rng.integers(2 * nC)))
        node = (int(rng.integers(Ps)), int(rng.integers(Pa)), int(rng.integers(Pa)))
        off = oracle.node_offset(H, ns, nC, Ps, Pa, cell, node)
        got, loc = oracle.classify(H, ns, nC, off)
        assert got == cell
        np.testing.assert_allclose(loc[:3], [ts[node[0]], ta[node[1]], ta[node[2]]], atol=1e-12)


@pytest.mark.parametrize("ns,nC,Ps,Pa", [(1, 2, 3, 5), (4, 8, 3, 5), (8, 16, 5, 5), (2, 6, 3, 5)])
def test_quarter_turn_tables(ns, nC, Ps, Pa):
    """Reading R18 (n_C even): node directions come from the first-quadrant sector
    rotated by q quarter turns.  Pins (i) the identity itself: offsets agree with
    the unreduced spherical formula (eq. interp_pts, libm sin/cos of
    the full angle) to rounding; (ii) exact equivariance: the node of sector
    i_phi + n_C/2 is bit for bit (-y, x, z) of the node of sector i_phi, and a
    vector turned by a quarter turn classifies into the sector shifted by n_C/2
    with identical (s, theta) decisions."""
    rng = np.random.default_rng(100 + nC)
    H = 0.5
    h = math.sqrt(3) / 2 * H
    ds, dth = (math.sqrt(3) / 3) / ns, math.pi / nC
    ts, ta = oracle.cheb_nodes(Ps), oracle.cheb_nodes(Pa)
    for _ in range(40):
        cell = [int(rng.integers(ns)), int(rng.integers(nC)), int(rng.integers(2 * nC))]
        node = [int(rng.integers(Ps)), int(rng.integers(Pa)), int(rng.integers(Pa))]
        off = oracle.node_offset(H, ns, nC, Ps, Pa, cell, node)
        s = (cell[0] + (1 + ts[node[0]]) / 2) * ds
        th = (cell[1] + (1 + ta[node[1]]) / 2) * dth
        ph = (cell[2] + (1 + ta[node[2]]) / 2) * dth
        r = h / s
        ref = [r * math.sin(th) * math.cos(ph), r * math.sin(th) * math.sin(ph), r * math.cos(th)]
        np.testing.assert_allclose(off, ref, rtol=0, atol=4e-15 * r)
        if nC % 2 == 0:
            turned = [cell[0], cell[1], (cell[2] + nC // 2) % (2 * nC)]
            off2 = oracle.node_offset(H, ns, nC, Ps, Pa, turned, node)
            assert off2[0] == -off[1] and off2[1] == off[0] and off2[2] == off[2]
    for _ in range(300):
        v = rng.normal(size=3) * H
        c0, _ = oracle.classify(H, ns, nC, v)
        c1, _ = oracle.classify(H, ns, nC, [-v[1], v[0], v[2]])
        if nC % 2 == 0:
            assert c1 == (c0[0], c0[1], (c0[2] + nC // 2) % (2 * nC))
        else:
            assert c1[:2] == c0[:2]
