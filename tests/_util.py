"""Shared comparison helpers for the parity tests."""
import numpy as np


def bits(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.view(np.uint64)


def assert_bitwise(a, b, what=""):
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    assert a.shape == b.shape, f"{what}: shape {a.shape} vs {b.shape}"
    # +0.0 and -0.0 compare equal here on purpose only through the scaled check;
    # bitwise means identical IEEE bit patterns
    diff = np.nonzero(bits(a) != bits(b))[0]
    assert diff.size == 0, (f"{what}: {diff.size} of {a.size} values differ bitwise; first at "
                            f"{diff[:5]}: {a[diff[:5]]} vs {b[diff[:5]]}")


def assert_scaled_close(v, ref, rel=1e-12, floor=1e-14, what=""):
    """|v - ref| <= rel*|ref| + floor*max|ref| for every entry."""
    v = np.asarray(v, dtype=np.float64).reshape(-1)
    ref = np.asarray(ref, dtype=np.float64).reshape(-1)
    assert v.shape == ref.shape
    s = np.max(np.abs(ref)) if ref.size else 0.0
    err = np.abs(v - ref)
    bad = err > rel * np.abs(ref) + floor * s
    assert not bad.any(), (f"{what}: {bad.sum()} entries outside tolerance; max err "
                           f"{err.max():.3e} (scale {s:.3e})")


class MT64:
    """std::mt19937_64, to reproduce the reference tests' seeded inputs."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def __call__(self):
        if self.i >= 312:
            for k in range(312):
                y = (self.mt[k] & 0xFFFFFFFF80000000) | (self.mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = self.mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                self.mt[k] = v
            self.i = 0
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & 0xFFFFFFFFFFFFFFFF

    def uniform(self, n):
        """acceptance.cpp:47: (rng() >> 11) * 2^-53"""
        return np.array([(self() >> 11) * 2.0 ** -53 for _ in range(n)])
