"""Shared test helpers (numpy side)."""
import numpy as np

from oracle.pyoracle import Config


class SplitMix64:
    """Python twin of the reference RNG (rng.hpp:16-40) for test-case generation."""
    M = (1 << 64) - 1

    def __init__(self, seed):
        self.s = seed & self.M

    def next(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def below(self, n):
        return self.next() % n

    def unit(self):
        return (self.next() >> 11) * 2.0 ** -53


def random_config(rng: SplitMix64, allow_shared=True) -> Config:
    """Same shape distribution as proj/tests/support.hpp:154-167."""
    E = 1 + rng.below(16)
    K = 1 + rng.below(min(4, E))
    D = 1 + rng.below(64)
    N = 1 + rng.below(128)
    S = 0
    if allow_shared and rng.below(2) == 0:
        S = 1 + rng.below(32)
    renorm = rng.below(2) == 0
    return Config(E, K, D, N, S, renorm)


def max_rel_diff(a, b):
    """proj/tests/support.hpp:32-42"""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1.0, np.max(np.abs(b))))
