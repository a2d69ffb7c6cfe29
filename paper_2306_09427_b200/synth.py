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
