"""Quadtree decomposition and pair indexing (TEST INFRASTRUCTURE, see oracle/__init__.py).

Restates /root/reference/pkg/src/allpairs/scheduler.py:
  Region.pair_count :33-43, Region.pairs :45-48, is_leaf :53-54, split :56-68,
  iter_leaves :78-86, PairLedger.pair_id :228-231.
"""

from __future__ import annotations


def region_pairs(r0: int, r1: int, c0: int, c1: int) -> int:
    full_rows = max(0, min(r1, c0) - r0)
    total = full_rows * (c1 - c0)
    a = max(r0, c0)
    b = min(r1, c1 - 1)
    if b > a:
        total += (c1 - 1 - a + c1 - b) * (b - a) // 2
    return total


def region_iter_pairs(r0: int, r1: int, c0: int, c1: int):
    for i in range(r0, r1):
        for j in range(max(c0, i + 1), c1):
            yield i, j


def leaves(n: int, leaf_block: int) -> list[tuple[int, int, int, int]]:
    """Depth-first leaves, children in (TL, TR, BL, BR) order, empty quadrants dropped."""
    out: list[tuple[int, int, int, int]] = []

    def rec(r0, r1, c0, c1):
        if region_pairs(r0, r1, c0, c1) == 0:
            return
        if r1 - r0 <= leaf_block and c1 - c0 <= leaf_block:
            out.append((r0, r1, c0, c1))
            return
        rm, cm = (r0 + r1) // 2, (c0 + c1) // 2
        for q in ((r0, rm, c0, cm), (r0, rm, cm, c1), (rm, r1, c0, cm), (rm, r1, cm, c1)):
            rec(*q)

    if n >= 2:
        rec(0, n, 0, n)
    return out


def pair_id(n: int, i: int, j: int) -> int:
    if not 0 <= i < j < n:
        raise ValueError(f"invalid pair ({i}, {j}) for n={n}")
    return i * (2 * n - i - 1) // 2 + (j - i - 1)


def pair_count(n: int) -> int:
    return n * (n - 1) // 2


def pair_from_id(n: int, pid: int) -> tuple[int, int]:
    """Inverse of ``pair_id`` (row i holds n-1-i consecutive ids)."""
    if not 0 <= pid < pair_count(n):
        raise ValueError(f"pair id {pid} out of range for n={n}")
    i = 0
    while pid >= n - 1 - i:
        pid -= n - 1 - i
        i += 1
    return i, i + 1 + pid
