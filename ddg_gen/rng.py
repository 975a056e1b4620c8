"""Counter-based random numbers shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic: it
only turns (seed, counter) into numbers, so that both sides of a parity test
see bit-identical inputs.

SplitMix64 (Steele, Lea & Flood 2014) on the 64-bit word (seed << 32) ^ idx,
top 53 bits scaled to [0, 1).  Everything is vectorised numpy uint64 math,
exact and platform independent.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """One SplitMix64 output per uint64 input word (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """u[i] in [0,1), i = offset .. offset+n-1, for stream `seed` (< 2**31)."""
    if not (0 <= seed < 2**31):
        raise ValueError("seed must be in [0, 2**31)")
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    words = (np.uint64(seed) << np.uint64(32)) ^ idx
    bits = splitmix64(words) >> np.uint64(11)
    return bits.astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform_pm1(seed: int, n: int) -> np.ndarray:
    """f ~ U(-1, 1) per entry (BASELINE.json configs)."""
    return 2.0 * uniform01(seed, n) - 1.0


def normal(seed: int, n: int) -> np.ndarray:
    """g ~ N(0, 1) by Box-Muller on the host (c15: host only, so libm decides once)."""
    u1 = uniform01(seed, n, 0)
    u2 = uniform01(seed, n, n)
    r = np.sqrt(-2.0 * np.log1p(-u1))      # 1 - u1 in (0, 1]
    return r * np.cos(2.0 * np.pi * u2)
