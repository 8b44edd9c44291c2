"""Zero-lag normalised cross-correlation, float64 numpy (TEST INFRASTRUCTURE, see oracle/__init__.py).

Parity UNPINNED by the reference (no NCC code; the paper's forensics compare is
NCC).  Standard definition:
  ncc(x, y) = sum (x - mean x)(y - mean y) / (||x - mean x|| * ||y - mean y||)
Pinned by known answers: ncc(x, x) = 1, ncc(x, -x) = -1, scale/offset invariance,
|ncc| ~ 1/sqrt(D) for independent noise.
"""

from __future__ import annotations

import numpy as np


def preprocess(x: np.ndarray) -> np.ndarray:
    v = np.asarray(x, dtype=np.float64).ravel()
    v = v - v.mean()
    return v / np.linalg.norm(v)


def compare(a: np.ndarray, b: np.ndarray) -> float:
    return float(np.dot(a, b))


def all_pairs(items: np.ndarray) -> np.ndarray:
    n = items.shape[0]
    z = np.stack([preprocess(items[k]) for k in range(n)])
    g = z @ z.T
    iu = np.triu_indices(n, k=1)
    return g[iu]
