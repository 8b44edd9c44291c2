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


def all_pairs_chunked(items: np.ndarray, chunk: int = 1 << 16) -> np.ndarray:
    """``all_pairs`` for items[n, ...] too large to hold as one float64 matrix:
    means and norms in float64, then the Gram accumulated in float64 over column
    chunks of D (same definition, summation split into chunks)."""
    n = items.shape[0]
    x = items.reshape(n, -1)
    d = x.shape[1]
    mean = np.zeros(n)
    sq = np.zeros(n)
    for c0 in range(0, d, chunk):
        mean += x[:, c0:c0 + chunk].astype(np.float64).sum(axis=1)
    mean /= d
    g = np.zeros((n, n))
    for c0 in range(0, d, chunk):
        z = x[:, c0:c0 + chunk].astype(np.float64) - mean[:, None]
        sq += np.einsum("ij,ij->i", z, z)
        g += z @ z.T
    inv = 1.0 / np.sqrt(sq)
    g = g * inv[:, None] * inv[None, :]
    iu = np.triu_indices(n, k=1)
    return g[iu]
