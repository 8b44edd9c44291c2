"""librocket on the CPU: the C ABI loads and exports every declared symbol, and the
host-side runtime structures (pair index, quadtree leaves, rank shares, slot tier)
match the reference -- no device calls."""

import ctypes as C
import json
import os
import re

import pytest

from paper_2009_04755_b200 import _lib
from paper_2009_04755_b200.errors import NoEvictableSlot

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
lib = _lib.lib


def declared_functions():
    text = open(os.path.join(ROOT, "include", "rocket.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rk_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound():
    names = declared_functions()
    assert len(names) >= 25
    raw = C.CDLL(_lib.LIB_PATH)
    bound = {s[0] for s in _lib.SIGNATURES}
    for name in names:
        assert hasattr(raw, name), f"{name} declared in rocket.h but not exported"
        assert name in bound, f"{name} not bound in _lib.SIGNATURES"


def test_abi_version_and_status_names():
    assert lib.rk_abi_version() == 1
    assert lib.rk_status_name(_lib.RK_ERR_SLOT_OVERFLOW) == b"RK_ERR_SLOT_OVERFLOW"


def test_pair_id_roundtrip():
    g = json.load(open(os.path.join(GOLD, "scheduler.json")))
    for n, rows in g["pair_id"].items():
        for i, j, pid in rows:
            assert lib.rk_pair_id(int(n), i, j) == pid
            ii, jj = C.c_int64(), C.c_int64()
            _lib.check(lib.rk_pair_from_id(int(n), pid, C.byref(ii), C.byref(jj)))
            assert (ii.value, jj.value) == (i, j)
    assert lib.rk_pair_id(5, 3, 3) == -1
    assert lib.rk_pair_id(5, 4, 2) == -1
    n = 16384
    for pid in (0, 1, n - 2, n - 1, n * (n - 1) // 2 - 1):
        ii, jj = C.c_int64(), C.c_int64()
        _lib.check(lib.rk_pair_from_id(n, pid, C.byref(ii), C.byref(jj)))
        assert lib.rk_pair_id(n, ii.value, jj.value) == pid
    with pytest.raises(ValueError):
        _lib.check(lib.rk_pair_from_id(10, 45, C.byref(ii), C.byref(jj)))


def leaves(n, lb, rank=0, world=1):
    cnt = lib.rk_leaves(n, lb, rank, world, None, 0)
    buf = (C.c_int32 * max(1, 4 * cnt))()
    got = lib.rk_leaves(n, lb, rank, world, buf, cnt)
    assert got == cnt
    return [list(buf[4 * k:4 * k + 4]) for k in range(cnt)]


def test_quadtree_leaves_match_reference():
    g = json.load(open(os.path.join(GOLD, "scheduler.json")))
    for key, want in g["leaves"].items():
        n, lb = map(int, key.split("/"))
        assert leaves(n, lb) == want, key


@pytest.mark.parametrize("world", [2, 3, 8])
def test_rank_shares_partition_the_pairs(world):
    n, lb = 100, 8
    all_leaves = leaves(n, lb)
    pairs = []
    per_rank = []
    for r in range(world):
        mine = leaves(n, lb, r, world)
        per_rank.append(sum(
            sum(1 for i in range(r0, r1) for j in range(max(c0, i + 1), c1)) for r0, r1, c0, c1 in mine))
        for r0, r1, c0, c1 in mine:
            pairs.extend((i, j) for i in range(r0, r1) for j in range(max(c0, i + 1), c1))
    assert len(pairs) == len(set(pairs)) == n * (n - 1) // 2
    # contiguous DFS blocks in leaf order, balanced by pair count
    concat = [l for r in range(world) for l in leaves(n, lb, r, world)]
    assert concat == all_leaves
    assert max(per_rank) - min(per_rank) <= 2 * lb * lb


def test_slot_tier_replays_reference_trace():
    g = json.load(open(os.path.join(GOLD, "slotcache.json")))
    t = C.c_void_p()
    _lib.check(lib.rk_tier_create(g["capacity"], C.byref(t)))
    kinds = {0: "hit", 1: "wait", 2: "miss"}
    try:
        for op, key, arg, slot in g["ops"]:
            if op == "acquire":
                kind, s = C.c_int32(), C.c_int32()
                st = lib.rk_tier_acquire(t, key, C.byref(kind), C.byref(s))
                if arg == "noslot":
                    assert st == _lib.RK_ERR_NO_EVICTABLE
                    with pytest.raises(NoEvictableSlot):
                        _lib.check(st)
                else:
                    _lib.check(st)
                    assert (kinds[kind.value], s.value) == (arg, slot), (op, key)
            elif op == "publish":
                _lib.check(lib.rk_tier_publish(t, slot, arg))
            elif op == "abort":
                _lib.check(lib.rk_tier_abort(t, slot))
            else:
                _lib.check(lib.rk_tier_release(t, slot))
        stats = (C.c_int64 * 5)()
        _lib.check(lib.rk_tier_stats(t, stats))
        f = g["final"]
        assert list(stats) == [f["hits"], f["misses"], f["waits"], f["evictions"], f["occupancy"]]
        keys = [lib.rk_tier_slot_key(t, s) for s in range(g["capacity"])]
        assert keys == [-1 if k is None else k for k in g["final_keys"]]
    finally:
        lib.rk_tier_destroy(t)


def test_slot_tier_rejects_misuse():
    t = C.c_void_p()
    _lib.check(lib.rk_tier_create(2, C.byref(t)))
    try:
        with pytest.raises(ValueError):
            _lib.check(lib.rk_tier_release(t, 0))     # nothing published
        kind, s = C.c_int32(), C.c_int32()
        _lib.check(lib.rk_tier_acquire(t, 5, C.byref(kind), C.byref(s)))
        assert kind.value == 2 and s.value == 0       # free list hands out slot 0 first
        _lib.check(lib.rk_tier_publish(t, 0, 1))
        _lib.check(lib.rk_tier_release(t, 0))
        with pytest.raises(ValueError):
            _lib.check(lib.rk_tier_release(t, 0))     # double release
    finally:
        lib.rk_tier_destroy(t)
    with pytest.raises(ValueError):
        _lib.check(lib.rk_tier_create(0, C.byref(t)))
