"""Composition-vector (sparse k-mer cosine) oracle (TEST INFRASTRUCTURE, see oracle/__init__.py).

Restates /root/reference/pkg/src/allpairs/apps.py:
  kmer_counts            :237-248
  CompositionVectorApp.parse       :286-302  (byte layout <I dim> + dim x <Q token><I count>)
  CompositionVectorApp.preprocess  :304-318  (freq = count / total, <Q token><d freq>)
  CompositionVectorApp.compare     :331-354  (sorted merge; cosine; 0 if a norm is 0)
and the dense-vector oracle of the reference tests (test_apps.py:23-39).
Pinned against tests/golden/cv.json (generated from the reference).
"""

from __future__ import annotations

import math
import struct
from collections import Counter

_HEAD = struct.Struct("<I")
_COUNT = struct.Struct("<QI")
_FREQ = struct.Struct("<Qd")


def kmer_counts(text: str, k: int) -> dict[int, int]:
    cleaned = "".join(text.split()).upper()
    counts: dict[int, int] = {}
    for pos in range(len(cleaned) - k + 1):
        token = int.from_bytes(cleaned[pos:pos + k].encode("utf-8"), "big")
        counts[token] = counts.get(token, 0) + 1
    return counts


def parse(text: str, k: int) -> bytes:
    counts = kmer_counts(text, k)
    if not counts:
        raise ValueError("no k-mers")
    out = bytearray(_HEAD.pack(len(counts)))
    for token in sorted(counts):
        out += _COUNT.pack(token, counts[token])
    return bytes(out)


def preprocess(parsed: bytes) -> list[tuple[int, float]]:
    (dim,) = _HEAD.unpack_from(parsed, 0)
    entries = [_COUNT.unpack_from(parsed, 4 + 12 * i) for i in range(dim)]
    total = sum(c for _, c in entries)
    return [(t, c / total) for t, c in entries]


def preprocessed_bytes(vec: list[tuple[int, float]]) -> bytes:
    out = bytearray(_HEAD.pack(len(vec)))
    for t, f in vec:
        out += _FREQ.pack(t, f)
    return bytes(out)


def compare(va: list[tuple[int, float]], vb: list[tuple[int, float]]) -> float:
    dot = 0.0
    ia = ib = 0
    while ia < len(va) and ib < len(vb):
        ta, fa = va[ia]
        tb, fb = vb[ib]
        if ta == tb:
            dot += fa * fb
            ia += 1
            ib += 1
        elif ta < tb:
            ia += 1
        else:
            ib += 1
    na = math.sqrt(sum(f * f for _, f in va))
    nb = math.sqrt(sum(f * f for _, f in vb))
    return dot / (na * nb) if na > 0 and nb > 0 else 0.0


def dense_cosine(text_a: str, text_b: str, k: int) -> float:
    """Brute-force dense-vector cosine (the reference tests' independent oracle)."""
    def freqs(text):
        cleaned = "".join(text.split()).upper()
        tokens = [cleaned[i:i + k] for i in range(len(cleaned) - k + 1)]
        counts = Counter(tokens)
        total = sum(counts.values())
        return {t: c / total for t, c in counts.items()}

    fa, fb = freqs(text_a), freqs(text_b)
    vocab = sorted(set(fa) | set(fb))
    va = [fa.get(t, 0.0) for t in vocab]
    vb = [fb.get(t, 0.0) for t in vocab]
    dot = sum(x * y for x, y in zip(va, vb))
    na = math.sqrt(sum(x * x for x in va))
    nb = math.sqrt(sum(x * x for x in vb))
    return dot / (na * nb) if na and nb else 0.0
