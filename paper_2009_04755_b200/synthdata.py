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


def gmm_parsed(n: int, seed: int = 0, max_points: int = 400):
    """Config 4 items in the GMM parsed layout (u32 m | u32 pad | m x (x, y, sigma) f32).

    Returns (uint8 array [n, 8 + 12 * max_points], localization counts)."""
    stride = 8 + 12 * max_points
    host = np.zeros((n, stride), dtype=np.uint8)
    m = np.zeros(n, dtype=np.int64)
    for k in range(n):
        p = particle(k, seed)
        m[k] = len(p)
        host[k, :8] = np.frombuffer(np.array([len(p), 0], dtype="<u4").tobytes(), dtype=np.uint8)
        host[k, 8:8 + 12 * len(p)] = np.frombuffer(p.astype("<f4").tobytes(), dtype=np.uint8)
    return host, m


def cv_nnz(n: int, mean_nnz: float, seed: int) -> np.ndarray:
    """Config 5 item sizes: log-normally skewed nnz clipped to [1e5, 1.8e6]."""
    rng = np.random.default_rng(seed)
    return np.clip(rng.lognormal(np.log(mean_nnz), 0.6, size=n), 1e5, 1.8e6).astype(np.int64)


def cv_parsed_device(n: int, mean_nnz: float, seed: int, vocab_bits: int = 26):
    """Config 5 items in the reference's parsed byte format (<I dim> + dim x <Q token><I count>),
    generated on the current CUDA device (torch) straight into one parsed buffer.

    Items of a family (k % 16) share half their tokens, so cosines are non-trivial.
    Returns (uint8 device tensor [n * stride], stride, capacity, actual nnz)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    nnz = cv_nnz(n, mean_nnz, seed)
    cap = int(nnz.max())
    stride = (4 + 12 * cap + 15) // 16 * 16
    buf = torch.zeros(n * stride, dtype=torch.uint8, device="cuda")
    pools = {}
    for k in range(n):
        fam = k % 16
        if fam not in pools:
            pools[fam] = torch.randint(0, 1 << vocab_bits, (2_000_000,), generator=g, device="cuda")
        m = int(nnz[k])
        shared = pools[fam][torch.randint(0, 2_000_000, (m // 2,), generator=g, device="cuda")]
        own = torch.randint(0, 1 << vocab_bits, (m - m // 2,), generator=g, device="cuda")
        tok = torch.unique(torch.cat([shared, own]))          # sorted, unique
        cnt = torch.randint(1, 50, (tok.numel(),), generator=g, device="cuda", dtype=torch.int32)
        rec = torch.cat([tok.view(torch.uint8).view(-1, 8), cnt.view(torch.uint8).view(-1, 4)], dim=1).reshape(-1)
        base = k * stride
        buf[base:base + 4] = torch.tensor([tok.numel()], dtype=torch.int32, device="cuda").view(torch.uint8)
        buf[base + 4:base + 4 + rec.numel()] = rec
        nnz[k] = tok.numel()
    torch.cuda.synchronize()
    return buf, stride, cap, nnz


def cv_parsed_host(nnz_list, seed: int, vocab_bits: int = 26) -> list:
    """Host (numpy) items of the given sizes in the parsed byte format, for CPU timing samples."""
    out = []
    for k, m in enumerate(nnz_list):
        rng = np.random.default_rng(mix64(seed, 0xC5, k))
        fam = np.random.default_rng(mix64(seed, 0xC6, k % 16)).integers(0, 1 << vocab_bits, size=2_000_000)
        tok = np.unique(np.concatenate([fam[rng.integers(0, 2_000_000, size=int(m) // 2)],
                                        rng.integers(0, 1 << vocab_bits, size=int(m) - int(m) // 2)]))
        rec = np.zeros(len(tok), dtype=[("t", "<u8"), ("c", "<u4")])
        rec["t"], rec["c"] = tok.astype(np.uint64), rng.integers(1, 50, size=len(tok))
        out.append(np.array([len(tok)], dtype="<u4").tobytes() + rec.tobytes())
    return out
