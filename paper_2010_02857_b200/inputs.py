"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the IFGF method: it only generates point
clouds, densities and error-target subsets.  It is the one module both the
oracle side (``oracle/``) and the CUDA side may use (task rule ③).

Recipes:

* Points: Fibonacci (golden-spiral) lattice on the unit sphere, BASELINE.json
  configs[0..4].  For i = 0..N-1::

      z_i   = 1 - (2i+1)/N
      rho_i = sqrt(1 - z_i^2)
      phi_i = 2*pi*frac(i*(3-sqrt(5))/2)
      x_i   = (rho_i cos phi_i, rho_i sin phi_i, z_i)

  The paper's meshes are unpublished (§4); this lattice
  stands in for them.  Spheroids (PAPER.md eq. defspheroid) are
  the same lattice scaled per axis (config 3: (1, 1, 0.25)).
* Densities: a_m = (2u-1) + i(2v-1), u, v 53-bit uniforms from the counter-based
  splitmix64 mixer at counters seed^(2m) and seed^(2m+1).
* Error targets: the first M entries of a seeded partial Fisher-Yates shuffle
  (PAPER.md eq. errorcomputation), uniforms from splitmix64 under
  seed+1.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

DEFAULT_SEED = 0x1F6F0C5D

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Standard public splitmix64 finaliser applied elementwise to uint64 counters."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform53(counters: np.ndarray) -> np.ndarray:
    """u = (splitmix64(c) >> 11) * 2^-53 in [0, 1)."""
    z = splitmix64(counters)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def fibonacci_sphere(n: int, scale=(1.0, 1.0, 1.0)) -> np.ndarray:
    """N x 3 float64 Fibonacci-lattice points on the unit sphere, scaled per axis."""
    if n < 1:
        raise ValueError("n must be >= 1")
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / n
    rho = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    golden = (3.0 - math.sqrt(5.0)) / 2.0
    t = i * golden
    phi = 2.0 * math.pi * (t - np.floor(t))
    pts = np.empty((n, 3), dtype=np.float64)
    pts[:, 0] = rho * np.cos(phi) * scale[0]
    pts[:, 1] = rho * np.sin(phi) * scale[1]
    pts[:, 2] = z * scale[2]
    return pts


def rough_sphere(n: int) -> np.ndarray:
    """Fibonacci lattice mapped to the rough sphere r = 1 + 0.05 sin(40 theta) sin(40 phi)
    (PAPER.md eq. defbumpysphere)."""
    p = fibonacci_sphere(n)
    theta = np.arccos(np.clip(p[:, 2], -1.0, 1.0))
    phi = np.arctan2(p[:, 1], p[:, 0])
    r = 1.0 + 0.05 * np.sin(40.0 * theta) * np.sin(40.0 * phi)
    return p * r[:, None]


def densities(n: int, seed: int = DEFAULT_SEED) -> np.ndarray:
    """complex128 densities a_m = (2u-1) + i(2v-1) (uniform on [-1,1]+i[-1,1])."""
    m = np.arange(n, dtype=np.uint64)
    s = np.uint64(seed)
    u = uniform53(s ^ (np.uint64(2) * m))
    v = uniform53(s ^ (np.uint64(2) * m + np.uint64(1)))
    return (2.0 * u - 1.0) + 1j * (2.0 * v - 1.0)


def error_targets(n: int, m: int = 1000, seed: int = DEFAULT_SEED) -> np.ndarray:
    """First min(m, n) entries of a seeded partial Fisher-Yates permutation of 0..n-1."""
    m = min(m, n)
    u = uniform53(np.uint64(seed + 1) ^ np.arange(m, dtype=np.uint64))
    swap: dict[int, int] = {}
    out = np.empty(m, dtype=np.int64)
    for i in range(m):
        j = i + int(u[i] * (n - i))
        if j >= n:
            j = n - 1
        vi = swap.get(i, i)
        vj = swap.get(j, j)
        swap[i], swap[j] = vj, vi
        out[i] = vj
    return out


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config (or a scaled variant used as a parity case)."""
    name: str
    n: int
    k: float
    levels: int
    Ps: int
    Pang: int
    scale: tuple = (1.0, 1.0, 1.0)
    geometry: str = "sphere"
    n_err_targets: int = 1000
    notes: str = ""

    def points(self) -> np.ndarray:
        if self.geometry == "rough":
            return rough_sphere(self.n)
        return fibonacci_sphere(self.n, self.scale)

    def densities(self, seed: int = DEFAULT_SEED) -> np.ndarray:
        return densities(self.n, seed)


# BASELINE.json configs[0..4] ("levels" = D, root = level 1, reading R10).
CONFIGS = {
    "cfg1": Config("cfg1", 24_576, 4 * math.pi, 4, 3, 5, n_err_targets=24_576,
                   notes="sphere 4 lambda; full O(N^2) direct sum"),
    "cfg2": Config("cfg2", 393_216, 16 * math.pi, 6, 3, 5),
    "cfg3": Config("cfg3", 1_572_864, 32 * math.pi, 7, 5, 5, scale=(1.0, 1.0, 0.25),
                   geometry="oblate"),
    "cfg4": Config("cfg4", 25_165_824, 128 * math.pi, 10, 3, 5),
    "cfg5": Config("cfg5", 100_663_296, 512 * math.pi, 12, 3, 5),
}

# SURVEY.md §8(f) workloads beyond BASELINE.json (bench.py --config; not bench defaults):
# f1 Laplace (kappa = 0) on the cfg4 sphere; f3 the paper's 512-lambda prolate spheroid
# (0.1, 0.1, 1) stand-in (N = 25.2 M, leaves lambda/4: D = 12) and a rough sphere at cfg4's
# size and wavenumber.
EXTRA_CONFIGS = {
    "lap4": Config("lap4", 25_165_824, 0.0, 10, 3, 5, notes="f1: Laplace on the cfg4 sphere"),
    "prolate512": Config("prolate512", 25_165_824, 512 * math.pi, 12, 3, 5, scale=(0.1, 0.1, 1.0),
                         geometry="prolate", notes="f3: 512 lambda along z, leaves lambda/4"),
    "rough4": Config("rough4", 25_165_824, 128 * math.pi, 10, 3, 5, geometry="rough",
                     notes="f3: rough sphere r = 1 + 0.05 sin(40 theta) sin(40 phi)"),
    # f3: Table timings2: kappa sweep at fixed N = 393,216 on the sphere,
    # leaves lambda/4 (D = 7, 8, 9 for kappa a = 16, 32, 64 pi)
    "t4_16pi": Config("t4_16pi", 393_216, 16 * math.pi, 7, 3, 5, notes="f3 T4: kappa a = 16 pi, N fixed"),
    "t4_32pi": Config("t4_32pi", 393_216, 32 * math.pi, 8, 3, 5, notes="f3 T4: kappa a = 32 pi, N fixed"),
    "t4_64pi": Config("t4_64pi", 393_216, 64 * math.pi, 9, 3, 5, notes="f3 T4: kappa a = 64 pi, N fixed"),
    # f3: Table timings3: N sweep at fixed kappa a = 16 pi (D = 7, leaves lambda/4)
    "t5_24k": Config("t5_24k", 24_576, 16 * math.pi, 7, 3, 5, notes="f3 T5: N = 24,576 at 16 pi"),
    "t5_98k": Config("t5_98k", 98_304, 16 * math.pi, 7, 3, 5, notes="f3 T5: N = 98,304 at 16 pi"),
    "t5_393k": Config("t5_393k", 393_216, 16 * math.pi, 7, 3, 5, notes="f3 T5: N = 393,216 at 16 pi"),
    "t5_1573k": Config("t5_1573k", 1_572_864, 16 * math.pi, 7, 3, 5, notes="f3 T5: N = 1,572,864 at 16 pi"),
}

