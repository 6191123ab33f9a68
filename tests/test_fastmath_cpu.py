"""CPU check of the CUDA path's lean FP64 atan2 / sincos (csrc/fastmath.cuh),
compiled as plain C++, against mpmath at 50 digits.  These functions only
produce values (local interpolation coordinates, phases); the bar is a few ulp."""
import math
import os
import subprocess

import mpmath as mp
import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "fastmath_check.cpp")


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("fm") / "fastmath_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", SRC, "-o", exe], check=True)
    return exe


def run(exe, lines):
    r = subprocess.run([exe], input="\n".join(lines) + "\n", capture_output=True, text=True, check=True)
    return r.stdout.split("\n")


def test_atan2(harness):
    mp.mp.dps = 50
    rng = np.random.default_rng(1)
    pts = list(rng.normal(size=(4000, 2)))
    # special directions: axes, diagonals, poles, tiny / huge magnitudes, tan(pi/8) boundary
    for a in [0.0, 1.0, -1.0, 1e-300, 1e300]:
        for b in [0.0, 1.0, -1.0, 0.41421356237309503, 2.414213562373095]:
            if a != 0.0 or b != 0.0:
                pts.append(np.array([a, b]))
                pts.append(np.array([b, a]))
    out = run(harness, [f"a {float(y)!r} {float(x)!r}" for y, x in pts])
    worst = 0.0
    for (y, x), got in zip(pts, out):
        ref = mp.atan2(mp.mpf(float(y)), mp.mpf(float(x)))
        err = abs(mp.mpf(got) - ref) / max(abs(ref), mp.mpf(2.0) ** -1022)
        worst = max(worst, float(err))
        if y == 0.0 and x > 0:
            assert float(got) == 0.0
    assert worst < 4 * 2.0 ** -53, worst


def test_atan2_2pi(harness):
    # phi in [0, 2 pi]: atan2 + 2 pi for y < 0 (reading R13), one rounding
    mp.mp.dps = 50
    rng = np.random.default_rng(3)
    pts = list(rng.normal(size=(4000, 2)))
    for a in [0.0, -0.0, 1.0, -1.0, 1e-300, -1e-300, 1e300, -1e300]:
        for b in [0.0, 1.0, -1.0, 0.41421356237309503, -2.414213562373095]:
            if a != 0.0 or b != 0.0:
                pts.append(np.array([a, b]))
                pts.append(np.array([b, a]))
    out = run(harness, [f"b {float(y)!r} {float(x)!r}" for y, x in pts])
    worst = 0.0
    for (y, x), got in zip(pts, out):
        ref = mp.atan2(mp.mpf(float(y)), mp.mpf(float(x)))
        if ref < 0:
            ref += 2 * mp.pi
        assert 0.0 <= float(got) <= 2 * math.pi
        err = abs(mp.mpf(got) - ref) / max(abs(ref), mp.mpf(2.0) ** -1022)
        if ref > 1e-300:
            worst = max(worst, float(err))
    assert worst < 4 * 2.0 ** -53, worst


def test_sincos(harness):
    mp.mp.dps = 50
    rng = np.random.default_rng(2)
    xs = list(rng.uniform(-10, 10, 2000)) + list(rng.uniform(0, 6000, 2000)) + [0.0, math.pi / 4, math.pi / 2,
                                                                                  -math.pi, 1e10, -3e9, 1e-8]
    out = run(harness, [f"s {float(x)!r}" for x in xs])
    worst = 0.0
    for x, got in zip(xs, out):
        s, c = (mp.mpf(v) for v in got.split())
        worst = max(worst, float(abs(s - mp.sin(mp.mpf(x)))), float(abs(c - mp.cos(mp.mpf(x)))))
    # absolute error: the reduction of x ~ 6e3 contributes ~ulp(x) * eps_pi ~ 1e-16 at most
    assert worst < 4e-16, worst
