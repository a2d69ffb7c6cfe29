"""Synthetic workload inputs: deformation gradients and networks.

``mt19937_64`` reproduces std::mt19937_64 exactly so the reference tests' recipes can be
re-created bit for bit, e.g. the batch F recipe of test_batch.cpp:149-157:
F = I; F11 += U(0.01, 0.06); F22 -= U(0, 0.02); F12 += U(0, 0.02), with
U(lo, hi) = lo + (hi - lo) * ((rng() >> 11) * 2^-53) (oracles.cpp:89-92).
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1


class mt19937_64:
    NN, MM = 312, 156
    A = 0xB5026F5AA96619E9
    UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        mt = [0] * self.NN
        mt[0] = seed & _M64
        for i in range(1, self.NN):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt, self.i = mt, self.NN

    def _twist(self):
        mt, NN, MM = self.mt, self.NN, self.MM
        for k in range(NN):
            x = (mt[k] & self.UM) | (mt[(k + 1) % NN] & self.LM)
            xa = x >> 1
            if x & 1:
                xa ^= self.A
            mt[k] = mt[(k + MM) % NN] ^ xa
        self.i = 0

    def __call__(self) -> int:
        if self.i >= self.NN:
            self._twist()
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _M64


def uniform(rng: mt19937_64, lo: float, hi: float) -> float:
    u = float(rng() >> 11) * 2.0 ** -53
    return lo + (hi - lo) * u


def batch_F(n: int, seed: int = 55) -> np.ndarray:
    """n deformation gradients from the test_batch.cpp:149-157 recipe, (n, 3, 3)."""
    rng = mt19937_64(seed)
    F = np.tile(np.eye(3), (n, 1, 1))
    for p in range(n):
        F[p, 0, 0] += uniform(rng, 0.01, 0.06)
        F[p, 1, 1] -= uniform(rng, 0.0, 0.02)
        F[p, 0, 1] += uniform(rng, 0.0, 0.02)
    return F


def config1_spec():
    """Config-1 network: knn 375 nodes / 1000 fibers, neighbors 10."""
    from . import NetGenSpec
    return NetGenSpec(style="knn", nodes=375, fibers=1000, neighbors=10, merge_radius=0.05)


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


CONFIG3_POINTS = 16384


def config3_size(p: int):
    """Config-3 RVE p: M = 500 + hash(p) mod 4501 fibers, N = round(M / r) nodes
    with r = 2.67 up to 1,500 fibers and 4 above (denser networks pass the reference's
    attachment check at 5k fibers)."""
    m = 500 + splitmix64(p) % 4501
    r = 2.67 if m <= 1500 else 4.0
    return m, int(round(m / r))


def config3_network(p: int):
    """knn network of config-3 RVE p, seed p + 1; on ConfigError the seed advances by the
    batch size."""
    from . import ConfigError, NetGenSpec, generate_network
    m, n = config3_size(p)
    seed = p + 1
    for _ in range(64):
        try:
            return generate_network(NetGenSpec(style="knn", nodes=n, fibers=m, neighbors=10,
                                               merge_radius=0.05), seed)
        except ConfigError:
            seed += CONFIG3_POINTS
    raise ConfigError(f"config-3 RVE {p}: no valid seed")


def config4_network(p: int):
    """Config-4 RVE p: a ~50k-fiber jittered lattice (23^3 nodes), seed p + 1 (the reference
    knn generator cannot build this size)."""
    from . import generate_lattice_network
    return generate_lattice_network(23, 50000, p + 1)


def parallel_networks(make, points, threads=None):
    """Build networks for `points` with `make` on a thread pool (the C generator releases
    the GIL through ctypes)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 1) as ex:
        return list(ex.map(make, points))
