"""Deterministic synthetic workloads of the north_star configs (host-side generators).

Item values are functions of (seed, key) only, via the reference's mix64
(rng.py:15-25), so every rank, run and test sees the same data.
"""

from __future__ import annotations

import numpy as np

from .rng import mix64


def particle(key: int, seed: int = 0, sites: int = 8, radius: float = 30.0) -> np.ndarray:
    """Localization-microscopy particle (config 4): ~300 localizations (x, y, sigma) in nm.

    A ring of ``sites`` binding sites, each localization drawn around a site
    with its own precision sigma in [3, 6] nm, m ~ U[250, 350], under a random
    rigid transform."""
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


def skewed_sequence(key: int, seed: int = 0, min_len: int = 2_000, max_len: int = 200_000) -> str:
    """Bioinformatics item (config 5): a DNA string with log-normally skewed length."""
    rng = np.random.default_rng(mix64(seed, 0x5E9, key))
    length = int(np.clip(rng.lognormal(mean=np.log(12_000), sigma=1.0), min_len, max_len))
    family = key % 7
    base = np.random.default_rng(mix64(seed, 0xFA3, family)).integers(0, 4, size=max_len)
    seq = base[:length].copy()
    mut = rng.random(length) < 0.15
    seq[mut] = rng.integers(0, 4, size=int(mut.sum()))
    return "".join("ACGT"[v] for v in seq)
