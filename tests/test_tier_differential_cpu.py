"""Differential test of the slot tier: random operation sequences applied to the
reference's own CacheTier (slotcache.py:139-282, imported from the staged
oracle/_ref or /root/reference) and to librocket's SlotTier (rk_tier_*) must
give the same Hit / MustWait / Miss kinds, the same slots, the same
NoEvictableSlot refusals, the same counters and the same final key placement.
(The golden 4,000-op trace in test_clib_cpu.py pins one sequence; this explores
many.)"""

import ctypes as C
import os
import sys

import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = next((p for p in (os.path.join(HERE, "oracle", "_ref"), "/root/reference/pkg/src")
            if os.path.isdir(os.path.join(p, "allpairs"))), None)


def _ref_modules():
    if REF is None:
        pytest.skip("reference package not present")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from allpairs import slotcache
    from allpairs.apps import ItemData, Stage
    from allpairs.errors import NoEvictableSlot
    return slotcache, ItemData, Stage, NoEvictableSlot


ops = st.lists(st.tuples(st.sampled_from(["acquire", "publish", "publish_keep", "abort", "release"]),
                         st.integers(0, 9)), min_size=1, max_size=80)


@settings(max_examples=150, deadline=None)
@given(capacity=st.integers(1, 5), seq=ops)
def test_tier_matches_reference_cache_tier(capacity, seq):
    slotcache, ItemData, Stage, NoEvictableSlot = _ref_modules()
    from paper_2009_04755_b200 import _lib
    from paper_2009_04755_b200._lib import lib
    ref = slotcache.CacheTier("dev", capacity, slot_size=64)
    t = C.c_void_p()
    _lib.check(lib.rk_tier_create(capacity, C.byref(t)))
    tickets, leases = [], []            # reference handles, each with our slot index
    try:
        for op, k in seq:
            if op == "acquire":
                kind, slot = C.c_int32(), C.c_int32()
                stat = lib.rk_tier_acquire(t, k, C.byref(kind), C.byref(slot))
                try:
                    res = ref.acquire(k)
                except NoEvictableSlot:
                    assert stat == _lib.RK_ERR_NO_EVICTABLE
                    continue
                assert stat == _lib.RK_OK
                name = type(res).__name__
                assert {0: "Hit", 1: "MustWait", 2: "Miss"}[kind.value] == name
                if name == "Hit":
                    assert res.lease.slot.index == slot.value
                    leases.append((res.lease, slot.value))
                elif name == "Miss":
                    assert res.ticket.slot.index == slot.value
                    tickets.append((res.ticket, slot.value))
            elif op in ("publish", "publish_keep", "abort") and tickets:
                ticket, slot = tickets.pop(k % len(tickets))
                if op == "abort":
                    ref.abort(ticket)
                    _lib.check(lib.rk_tier_abort(t, slot))
                else:
                    keep = op == "publish_keep"
                    lease = ref.publish(ticket, ItemData(Stage.PREPROCESSED, b"x"), retain=keep)
                    _lib.check(lib.rk_tier_publish(t, slot, int(keep)))
                    if keep:
                        leases.append((lease, slot))
            elif op == "release" and leases:
                lease, slot = leases.pop(k % len(leases))
                lease.release()
                _lib.check(lib.rk_tier_release(t, slot))
        stats = (C.c_int64 * 5)()
        _lib.check(lib.rk_tier_stats(t, stats))
        snap = ref.snapshot_stats()
        assert list(stats[:4]) == [snap["hits"], snap["misses"], snap["waits"], snap["evictions"]]
        want = [s.key if s.key is not None else -1 for s in ref.slots]
        assert [lib.rk_tier_slot_key(t, s) for s in range(capacity)] == want
    finally:
        lib.rk_tier_destroy(t)


@settings(max_examples=60, deadline=None)
@given(n=st.integers(0, 700), leaf=st.integers(1, 40))
def test_quadtree_leaves_match_reference(n, leaf):
    """librocket's depth-first leaves (rk_leaves, world 1) are the reference's
    iter_leaves(root_region(n), leaf) in order, for random n and leaf sizes."""
    _ref_modules()
    from allpairs.scheduler import iter_leaves, root_region
    from paper_2009_04755_b200.engine import rank_leaves
    want = [r.as_tuple() for r in iter_leaves(root_region(n), leaf)] if n > 1 else []
    assert rank_leaves(n, leaf) == want


@settings(max_examples=200, deadline=None)
@given(n=st.integers(2, 5000), data=st.data())
def test_pair_id_matches_reference_ledger(n, data):
    """rk_pair_id (the result-matrix index every kernel writes) is PairLedger.pair_id."""
    _ref_modules()
    from allpairs.scheduler import PairLedger
    from paper_2009_04755_b200._lib import lib
    i = data.draw(st.integers(0, n - 2))
    j = data.draw(st.integers(i + 1, n - 1))
    assert lib.rk_pair_id(n, i, j) == PairLedger(n).pair_id(i, j)


@settings(max_examples=100, deadline=None)
@given(n=st.integers(1, 100000), r=st.floats(1.0, 50.0), p=st.integers(1, 64),
       costs=st.tuples(*[st.floats(0.0, 1e-2)] * 4), mfb=st.floats(0.0, 1e8), bw=st.floats(1e6, 1e11),
       t=st.floats(1e-3, 1e5))
def test_perf_model_matches_reference(n, r, p, costs, mfb, bw, t):
    """The perf model the bench reports (T_min, efficiency, per-resource bounds)
    equals the reference's perfmodel.py on random inputs."""
    _ref_modules()
    from allpairs import perfmodel as ref
    from paper_2009_04755_b200 import perfmodel as ours
    kw = dict(t_parse=costs[0], t_preprocess=costs[1], t_comparison=costs[2], t_postprocess=costs[3],
              mean_file_bytes=mfb, io_bandwidth=bw)
    rc, oc = ref.StageCosts(**kw), ours.StageCosts(**kw)
    assert ours.t_min(n, oc) == ref.t_min(n, rc)
    assert ours.t_gpu(n, r, oc) == ref.t_gpu(n, r, rc)
    assert ours.t_cpu(n, r, oc) == ref.t_cpu(n, r, rc)
    assert ours.t_io(n, r, oc) == ref.t_io(n, r, rc)
    tm = ours.t_min(n, oc)
    if tm > 0:
        assert ours.efficiency(tm, p, t) == ref.efficiency(tm, p, t)
