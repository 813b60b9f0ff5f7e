"""Seeded synthetic inputs shared by the oracle-side tests and the product-side bench.

This module holds NONE of the method's arithmetic: it only draws the SpMV input vector
(BASELINE configs[0]: "SpMV on a seeded uniform[-1,1] fp64 vector").  Reading C7
(DESIGN.md §3): x_i = 2*u_i - 1, u_i = (z_i >> 11) * 2^-53, z_i = SplitMix64 output
number i+1 for `seed`, i.e. the SplitMix64 finaliser of seed + (i+1)*0x9E3779B97F4A7C15
(mod 2^64).  Every step is exact, so the vector is bit-identical wherever it is drawn.
"""
from __future__ import annotations

import numpy as np

GOLDEN_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
DEFAULT_SEED = 12345


def splitmix64(seed: int, idx: np.ndarray) -> np.ndarray:
    """Raw 64-bit outputs z_i for counter indices idx (0-based: output number idx+1)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed % (1 << 64)) + (idx + np.uint64(1)) * GOLDEN_GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1(n: int, seed: int = DEFAULT_SEED, idx: np.ndarray | None = None) -> np.ndarray:
    """Seeded uniform[-1, 1) fp64 vector of length n (or at the given indices)."""
    if idx is None:
        idx = np.arange(n, dtype=np.uint64)
    z = splitmix64(seed, idx)
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return 2.0 * u - 1.0
