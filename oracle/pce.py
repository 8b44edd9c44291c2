"""PRNU peak-to-correlation-energy, float64 numpy (TEST INFRASTRUCTURE, see oracle/__init__.py).

Parity UNPINNED by the reference: /root/reference has no PCE code (SURVEY.md
section 8(c); the paper names the forensics comparison at PAPER.md:512-529).
The definitions below are the standard ones (Goljan et al.), with every
choice that matters for parity fixed here and mirrored by
paper_2009_04755_b200/csrc/pce.cu:

  preprocess   x <- x - mean(x);  S = rfft2(x)
  compare      C = irfft2(S_i * conj(S_j))             circular cross-correlation
               p* = argmax C  (signed max; first index in row-major order on ties)
               A  = 11 x 11 wrap-around neighbourhood of p*
               PCE = C[p*] * |C[p*]| / ( sum_{s not in A} C[s]^2 / (H*W - 121) )
  postprocess  match = PCE >= threshold

PCE is invariant to any positive scaling of C, so FFT normalisation
conventions do not affect it.
"""

from __future__ import annotations

import numpy as np

from .rng import mix64_np

WIN = 11
PRNU_GAIN = 0.2


def preprocess(x: np.ndarray) -> np.ndarray:
    x64 = np.asarray(x, dtype=np.float64)
    x64 = x64 - x64.mean()
    return np.fft.rfft2(x64)


def correlation(si: np.ndarray, sj: np.ndarray, h: int, w: int) -> np.ndarray:
    return np.fft.irfft2(si * np.conj(sj), s=(h, w))


def pce_from_plane(c: np.ndarray) -> tuple[float, float, int]:
    """Returns (pce, peak, flat peak index)."""
    h, w = c.shape
    p = int(np.argmax(c))
    peak = float(c.flat[p])
    r, q = divmod(p, w)
    rows = np.arange(r - WIN // 2, r + WIN // 2 + 1) % h
    cols = np.arange(q - WIN // 2, q + WIN // 2 + 1) % w
    win = c[np.ix_(rows, cols)]
    energy = (float(np.sum(c * c)) - float(np.sum(win * win))) / (h * w - WIN * WIN)
    return peak * abs(peak) / energy, peak, p


def compare(si: np.ndarray, sj: np.ndarray, h: int, w: int) -> float:
    return pce_from_plane(correlation(si, sj, h, w))[0]


def all_pairs(items: np.ndarray) -> np.ndarray:
    """Packed upper triangle (pair_id order) of PCE over items[n, h, w]."""
    n, h, w = items.shape
    spectra = [preprocess(items[k]) for k in range(n)]
    out = np.empty(n * (n - 1) // 2, dtype=np.float64)
    pid = 0
    for i in range(n):
        for j in range(i + 1, n):
            out[pid] = compare(spectra[i], spectra[j], h, w)
            pid += 1
    return out


def _normal_from_hash(hv: np.ndarray) -> np.ndarray:
    u1 = ((hv >> np.uint64(40)).astype(np.float64) + 0.5) * 2.0 ** -24
    u2 = (((hv >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.float64) + 0.5) * 2.0 ** -24
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def prnu_patterns(h: int, w: int, first_key: int, n_items: int, cameras: int, seed: int) -> np.ndarray:
    """float64 restatement of rk_synth_prnu: item k = 0.2*K[k % cameras] + N(0,1).

    Agrees with the device generator to float32 rounding (the device evaluates
    Box-Muller in fp32); parity tests feed both paths the device's own bytes.
    """
    pix = np.arange(h * w, dtype=np.uint64)
    out = np.empty((n_items, h, w), dtype=np.float32)
    for t in range(n_items):
        key = first_key + t
        cam = key % cameras
        k = _normal_from_hash(mix64_np(seed, 0x50524E55, np.uint64(cam), pix))
        e = _normal_from_hash(mix64_np(seed, 0x4E4F4953, np.uint64(key), pix))
        out[t] = (PRNU_GAIN * k + e).reshape(h, w).astype(np.float32)
    return out


def pairs_batched(items: np.ndarray, pairs, batch: int = 16, workers: int = -1):
    """PCE of the listed (i, j) pairs over items[n, h, w] -- the same definition as
    ``compare`` (float64 throughout), with the inverse FFTs batched through
    scipy.fft on all host threads so parity tests can check thousands of 1024^2
    pairs in seconds.  Spectra are computed once per distinct key."""
    import scipy.fft as sfft
    n, h, w = items.shape
    keys = sorted({k for p in pairs for k in p})
    spec = {}
    for k in keys:
        x = np.asarray(items[k], dtype=np.float64)
        spec[k] = sfft.rfft2(x - x.mean(), workers=workers)
    out = np.empty(len(pairs), dtype=np.float64)
    for b0 in range(0, len(pairs), batch):
        chunk = pairs[b0:b0 + batch]
        prod = np.stack([spec[i] * np.conj(spec[j]) for i, j in chunk])
        planes = sfft.irfft2(prod, s=(h, w), workers=workers)
        for q in range(len(chunk)):
            out[b0 + q] = pce_from_plane(planes[q])[0]
    return out
