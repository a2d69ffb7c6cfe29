"""Synthetic workload recipe for the reference arm of bench.py -- TEST INFRASTRUCTURE.

The reference arm (``bench.py --impl reference``) must not import the product package, so
the two pieces of the config-2 workload it needs are restated here, independently of
``paper_2306_09427_b200.synth``:

* ``mt19937_64`` -- std::mt19937_64 (the reference tests' generator, tests/oracles.cpp:89-92);
* ``batch_F`` -- the deformation-gradient recipe of tests/test_batch.cpp:149-157:
  F = I; F11 += U(0.01, 0.06); F22 -= U(0, 0.02); F12 += U(0, 0.02) with
  U(lo, hi) = lo + (hi - lo) * ((rng() >> 11) * 2^-53);
* ``CONFIG1_KNN`` -- the config-1 network spec, which the reference arm builds
  with the reference's own generator (``oracle.ref_generate``, netgen.cpp:276-285).

``tests/test_host.py`` checks both restatements give identical F bits.
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1

CONFIG1_KNN = dict(style="knn", nodes=375, fibers=1000, neighbors=10, merge_radius=0.05)
NET_SEED = 1


class mt19937_64:
    """std::mt19937_64 (Matsumoto & Nishimura 64-bit parameters)."""

    def __init__(self, seed: int = 5489):
        self.state = [0] * 312
        self.state[0] = seed & _M64
        for i in range(1, 312):
            prev = self.state[i - 1]
            self.state[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _M64
        self.index = 312

    def _generate(self):
        s = self.state
        for k in range(312):
            y = (s[k] & 0xFFFFFFFF80000000) | (s[(k + 1) % 312] & 0x7FFFFFFF)
            s[k] = s[(k + 156) % 312] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
        self.index = 0

    def next(self) -> int:
        if self.index >= 312:
            self._generate()
        x = self.state[self.index]
        self.index += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _M64


def batch_F(n: int, seed: int = 55) -> np.ndarray:
    """(n, 3, 3) deformation gradients of the test_batch.cpp:149-157 recipe."""
    g = mt19937_64(seed)

    def u(lo, hi):
        return lo + (hi - lo) * (float(g.next() >> 11) * 2.0 ** -53)

    F = np.tile(np.eye(3), (n, 1, 1))
    for p in range(n):
        F[p, 0, 0] += u(0.01, 0.06)
        F[p, 1, 1] -= u(0.0, 0.02)
        F[p, 0, 1] += u(0.0, 0.02)
    return F


CONFIG3_POINTS = 16384


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def config3_spec(p: int):
    """Config-3 RVE p: M = 500 + splitmix64(p) mod 4501 fibers, N = round(M / r)
    nodes with r = 2.67 up to 1,500 fibers and 4 above; knn, neighbors 10, merge 0.05,
    seed p + 1 (advanced by 16,384 on ConfigError)."""
    m = 500 + splitmix64(p) % 4501
    r = 2.67 if m <= 1500 else 4.0
    return dict(style="knn", nodes=int(round(m / r)), fibers=m, neighbors=10,
                merge_radius=0.05), p + 1


def config3_ref_network(p: int):
    """Config-3 RVE p built by the REFERENCE generator (oracle/_ref)."""
    import oracle as O
    spec, seed = config3_spec(p)
    for _ in range(64):
        try:
            return O.ref_generate(seed=seed, **spec), seed
        except O.OracleError:
            seed += CONFIG3_POINTS
    raise RuntimeError(f"config-3 RVE {p}: no valid seed")
