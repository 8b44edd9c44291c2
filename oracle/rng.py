"""splitmix64 mixer and the SyntheticApp value (TEST INFRASTRUCTURE, see oracle/__init__.py).

Restates /root/reference/pkg/src/allpairs/rng.py:15-25 and apps.py:201-208.
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def mix64(*values: int) -> int:
    """rng.py:15-25 -- one splitmix64 round per value."""
    x = GOLDEN
    for v in values:
        x = (x + (v & M64) + GOLDEN) & M64
        x ^= x >> 30
        x = (x * 0xBF58476D1CE4E5B9) & M64
        x ^= x >> 27
        x = (x * 0x94D049BB133111EB) & M64
        x ^= x >> 31
    return x


def synthetic_value(seed: int, i: int, j: int) -> float:
    """apps.py:207: mix64(seed, 0xC0403A3E, i, j) / 2**64."""
    return mix64(seed, 0xC0403A3E, i, j) / float(1 << 64)


def _round_np(x: np.ndarray, v: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + v + np.uint64(GOLDEN)
        x ^= x >> np.uint64(30)
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x = x * np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def mix64_np(*values) -> np.ndarray:
    """Vectorised mix64 over broadcastable uint64 arrays."""
    arrs = [np.asarray(v).astype(np.uint64) if not isinstance(v, int) else np.uint64(v & M64) for v in values]
    shape = np.broadcast_shapes(*[np.shape(a) for a in arrs])
    x = np.full(shape, GOLDEN, dtype=np.uint64)
    for a in arrs:
        x = _round_np(x, a)
    return x
