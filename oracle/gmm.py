"""Particle-registration (GMM / Bhattacharyya) cost, float64 numpy (TEST INFRASTRUCTURE,
see oracle/__init__.py).

Parity UNPINNED by the reference (no microscopy code; PAPER.md:557-566 describes
the GMM-L2 / Bhattacharyya registration of Heydarian et al.).  Fixed-grid,
deterministic form used by paper_2009_04755_b200/csrc/gmm.cu:
  p_a = (x_a, y_a) - centroid_i, q_b = (x_b, y_b) - centroid_j
  E_k = sum_a sum_b exp(-|R(2 pi k / K) p_a - q_b|^2 / (s_a^2 + s_b^2 + s0))
  value = max_k E_k / (m_i m_j)
"""

from __future__ import annotations

import numpy as np

from .rng import mix64


def particle(key: int, seed: int = 0, sites: int = 8, radius: float = 30.0) -> np.ndarray:
    """Deterministic synthetic particle: (m, 3) float32 rows (x, y, sigma) in nm."""
    rng = np.random.default_rng(mix64(seed, 0x474D4D, key))
    m = int(rng.integers(250, 351))
    ang = rng.uniform(0.0, 2.0 * np.pi)
    shift = rng.uniform(-50.0, 50.0, size=2)
    site_ang = 2.0 * np.pi * np.arange(sites) / sites
    sx, sy = radius * np.cos(site_ang), radius * np.sin(site_ang)
    which = rng.integers(0, sites, size=m)
    sigma = rng.uniform(3.0, 6.0, size=m)
    x = sx[which] + rng.normal(0.0, 1.0, size=m) * sigma
    y = sy[which] + rng.normal(0.0, 1.0, size=m) * sigma
    c, s = np.cos(ang), np.sin(ang)
    out = np.stack([c * x - s * y + shift[0], s * x + c * y + shift[1], sigma], axis=1)
    return out.astype(np.float32)


def compare(a: np.ndarray, b: np.ndarray, angles: int = 36, s0: float = 0.0) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    p = a[:, :2] - a[:, :2].mean(axis=0)
    q = b[:, :2] - b[:, :2].mean(axis=0)
    sa = a[:, 2] ** 2
    sb = b[:, 2] ** 2 + s0
    denom = sa[:, None] + sb[None, :]
    best = -1.0
    for k in range(angles):
        t = 2.0 * np.pi * k / angles
        c, s = np.cos(t), np.sin(t)
        rx = c * p[:, 0] - s * p[:, 1]
        ry = s * p[:, 0] + c * p[:, 1]
        d2 = (rx[:, None] - q[None, :, 0]) ** 2 + (ry[:, None] - q[None, :, 1]) ** 2
        best = max(best, float(np.exp(-d2 / denom).sum()))
    return best / (len(a) * len(b))
