"""PCE parity: librocket's CUDA path vs the float64 numpy oracle (oracle/pce.py).

Tolerance: 1e-4 relative on PCE scores (north_star; fp32 FFTs vs float64).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import pce as opce  # noqa: E402
from oracle import scheduler as osched  # noqa: E402

pytestmark = pytest.mark.gpu

RTOL = 1e-4


def _lib():
    from paper_2009_04755_b200 import _lib, device
    return _lib, device


def make_items(n, side, cameras=2, seed=11, first_key=0):
    _, device = _lib()
    buf = torch.empty(n * side * side, dtype=torch.float32, device="cuda")
    device.synth_prnu(side, side, first_key, n, cameras, seed, buf)
    torch.cuda.synchronize()
    return buf


def unpack_slot(slot_bytes: np.ndarray, n: int) -> np.ndarray:
    """Device slot layout -> numpy rfft2 layout (n x (n/2+1)).

    256/1024: [col][row]; 2048: [row parity][col][row >> 1] (csrc/pce2k.cu header).
    """
    if n == 2048:
        zp = slot_bytes.view(np.complex64).reshape(2, n // 2, n // 2).astype(np.complex128)
        z = np.empty((n // 2, n), dtype=np.complex128)
        z[:, 0::2] = zp[0]
        z[:, 1::2] = zp[1]
    else:
        z = slot_bytes.view(np.complex64).reshape(n // 2, n).astype(np.complex128)  # [col][row]
    s = np.zeros((n, n // 2 + 1), dtype=np.complex128)
    s[:, 1:n // 2] = z[1:].T
    p = z[0]
    pr = np.conj(p[(-np.arange(n)) % n])
    s[:, 0] = 0.5 * (p + pr)
    s[:, n // 2] = (p - pr) / 2j
    return s


@pytest.mark.parametrize("side", [256, 1024, 2048])
def test_preprocess_spectrum_layout(side):
    _l, device = _lib()
    n = 3
    items = make_items(n, side)
    app = device.DeviceApp(_l.app_params(_l.APP_PCE, n, height=side, width=side))
    slots = app.alloc_slots(n)
    app.preprocess(items, side * side * 4, n, slots, [2, 0, 1])
    torch.cuda.synchronize()
    host = items.cpu().numpy().reshape(n, side, side)
    raw = slots.cpu().numpy()
    for k, slot in zip(range(n), [2, 0, 1]):
        got = unpack_slot(raw[slot * app.slot_stride: slot * app.slot_stride + app.slot_bytes], side)
        want = opce.preprocess(host[k]) / side
        err = np.abs(got - want).max() / np.abs(want).max()
        assert err < 1e-5, (side, k, err)   # fp32 FFT vs float64


@pytest.mark.parametrize("side,n", [(256, 7), (1024, 4), (2048, 4)])
def test_allpairs_matches_oracle(side, n):
    _l, device = _lib()
    items = make_items(n, side, cameras=2)
    app = device.DeviceApp(_l.app_params(_l.APP_PCE, n, height=side, width=side, threshold=60.0))
    slots = app.alloc_slots(n)
    app.preprocess(items, side * side * 4, n, slots, list(range(n)))
    total = n * (n - 1) // 2
    out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    flags = torch.zeros(total, dtype=torch.uint8, device="cuda")
    app.compare_tile(slots, 0, n, 0, n, list(range(n)), out, flags)
    torch.cuda.synchronize()
    want = opce.all_pairs(items.cpu().numpy().reshape(n, side, side))
    got = out.cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=RTOL)
    f = flags.cpu().numpy()
    assert set(np.unique(f)).issubset({1, 3})
    assert np.array_equal(f == 3, got >= 60.0)
    # same-camera pairs separate from different-camera pairs
    for i in range(n):
        for j in range(i + 1, n):
            v = got[osched.pair_id(n, i, j)]
            assert (v > 60.0) == (i % 2 == j % 2), (i, j, v)


@pytest.mark.parametrize("side,shift", [(256, (5, -9)), (2048, (5, -9)), (2048, (0, 3)), (2048, (-1029, 1500)),
                                        (1024, (1, -517))])
def test_shifted_copy_peak(side, shift):
    """Peak at the shift, including wrap-around windows (row 0 / last row block) and
    peaks in the second half of a 2048 line (the radix-2 step's X[k + 1024] outputs)."""
    _l, device = _lib()
    base = make_items(1, side, cameras=1, seed=3).view(side, side)
    shifted = torch.roll(base, shifts=shift, dims=(0, 1))
    items = torch.stack([base, shifted]).contiguous().view(-1)
    app = device.DeviceApp(_l.app_params(_l.APP_PCE, 2, height=side, width=side))
    slots = app.alloc_slots(2)
    app.preprocess(items, side * side * 4, 2, slots, [0, 1])
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    app.compare_pairs(slots, [(0, 1, 0, 1)], out)
    torch.cuda.synchronize()
    host = items.cpu().numpy().reshape(2, side, side)
    s0, s1 = opce.preprocess(host[0]), opce.preprocess(host[1])
    want, _, idx = opce.pce_from_plane(opce.correlation(s0, s1, side, side))
    assert divmod(idx, side) == ((-shift[0]) % side, (-shift[1]) % side)
    assert out.item() == pytest.approx(want, rel=RTOL)
    assert out.item() > 1e4


def test_compare_rejects_unordered_pair():
    _l, device = _lib()
    app = device.DeviceApp(_l.app_params(_l.APP_PCE, 4, height=256, width=256))
    slots = app.alloc_slots(2)
    out = torch.zeros(6, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        app.compare_pairs(slots, [(2, 1, 0, 1)], out)
    with pytest.raises(ValueError):
        app.compare_pairs(slots, [(1, 1, 0, 1)], out)


@pytest.mark.parametrize("device_slots,leaf", [(64, 4), (9, 3)])
def test_engine_matches_oracle(device_slots, leaf):
    _l, device = _lib()
    side, n = 256, 13
    items = make_items(n, side, cameras=3, seed=5)
    eng = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side), leaf_block=leaf,
                              device_slots=device_slots)
    total = n * (n - 1) // 2
    out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    eng.run(out, device_items=items, parsed_stride=side * side * 4)
    st = eng.stats()
    want = opce.all_pairs(items.cpu().numpy().reshape(n, side, side))
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=RTOL)
    assert st["pairs_done"] == total
    assert st["pinned_at_end"] == 0 and st["writing_at_end"] == 0     # lease hygiene (test_engine.py:124-133)
    if device_slots >= n:
        assert st["loads"] == n and st["evictions"] == 0   # R = 1 at capacity >= n
    else:
        assert st["loads"] > n and st["evictions"] > 0


@pytest.mark.parametrize("device_slots", [None, 5])
def test_engine_host_items_matches_device_items(device_slots):
    """Host (H2D on the load stream) and device inputs agree bit-for-bit, also when
    loads into evicted slots must wait for the compares still reading them."""
    _l, device = _lib()
    side, n = 256, 9
    items = make_items(n, side, cameras=2, seed=9)
    host = items.cpu().pin_memory()
    total = n * (n - 1) // 2
    outs = []
    for kw in ({"device_items": items}, {"host_items": host}):
        eng = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side), leaf_block=4,
                                  **({} if device_slots is None else {"device_slots": device_slots}))
        out = torch.zeros(total, dtype=torch.float64, device="cuda")
        eng.run(out, parsed_stride=side * side * 4, **kw)
        outs.append(out.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])


def test_engine_2048_with_evictions():
    """C3 item shape through the engine with a slot tier smaller than n (reloads)."""
    _l, device = _lib()
    side, n = 2048, 5
    items = make_items(n, side, cameras=2, seed=21)
    eng = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side, threshold=60.0), leaf_block=2,
                              device_slots=3)
    total = n * (n - 1) // 2
    out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    flags = torch.zeros(total, dtype=torch.uint8, device="cuda")
    eng.run(out, flags, device_items=items, parsed_stride=side * side * 4)
    want = opce.all_pairs(items.cpu().numpy().reshape(n, side, side))
    got = out.cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=RTOL)
    assert np.array_equal(flags.cpu().numpy() == 3, got >= 60.0)
    st = eng.stats()
    assert st["pairs_done"] == total and st["evictions"] > 0


def test_engine_trace_events_and_metrics(tmp_path):
    """Trace events (reference TraceEvent schema) cover every compare batch and load
    group; the RunMetrics document reports R, hit rate and the perf-model efficiency."""
    from paper_2009_04755_b200 import metrics, perfmodel
    from paper_2009_04755_b200.apps import PCEApp
    from paper_2009_04755_b200.engine import AllPairsEngine
    app = PCEApp(20, side=256, cameras=3, seed=4)
    eng = AllPairsEngine(app, leaf_block=4, device_slots=8, trace_events=4096)
    res = eng.run()
    ev = res.trace
    comp = [e for e in ev if e["label"] == "compare"]
    loads = [e for e in ev if e["label"] == "preprocess"]
    assert sum(e["count"] for e in comp) == res.pairs == res.stats["pairs_done"]
    assert sum(e["count"] for e in loads) == res.stats["loads"]
    assert all(e["lane"] == "gpu0" for e in comp) and all(e["lane"] == "up0" for e in loads)
    assert all(0 <= e["start_ns"] <= e["end_ns"] for e in ev)
    starts = [e["start_ns"] for e in comp]
    assert starts == sorted(starts)                     # one stream: batches in order
    path = tmp_path / "trace.jsonl"
    metrics.write_trace(str(path), ev)
    assert len(metrics.read_trace(str(path))) == len(ev)
    doc = eng.metrics(res, costs=perfmodel.StageCosts(t_preprocess=1e-5, t_comparison=1e-5))
    assert doc["R"] == res.r_factor and doc["pairs"] == res.pairs
    assert doc["per_node"][0]["comparisons"] == res.pairs and doc["efficiency"] > 0
    eng.close()


@pytest.mark.parametrize("n", [1, 2, 3])
def test_engine_tiny_jobs(n):
    """Degenerate job sizes: n = 1 has no pairs (nothing written, no launch needed),
    n = 2 and 3 one partial leaf."""
    _l, device = _lib()
    side = 256
    items = make_items(max(n, 1), side, cameras=1, seed=2)
    eng = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side), leaf_block=8)
    total = n * (n - 1) // 2
    out = torch.full((max(total, 1),), float("nan"), dtype=torch.float64, device="cuda")
    eng.run(out, device_items=items, parsed_stride=side * side * 4)
    st = eng.stats()
    assert st["pairs_done"] == total
    got = out.cpu().numpy()
    if total == 0:
        assert np.isnan(got[0])
    else:
        want = opce.all_pairs(items.cpu().numpy().reshape(n, side, side))
        np.testing.assert_allclose(got[:total], want, rtol=RTOL)


def test_engine_tight_tier_completes():
    """Two device slots with 8-item leaves: leaves are split until their items fit
    (the reference's tight-tier completion, test_engine.py:88-93); results exact."""
    _l, device = _lib()
    side, n = 256, 9
    items = make_items(n, side, cameras=2, seed=13)
    eng = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side), leaf_block=8,
                              device_slots=2)
    total = n * (n - 1) // 2
    out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    eng.run(out, device_items=items, parsed_stride=side * side * 4)
    want = opce.all_pairs(items.cpu().numpy().reshape(n, side, side))
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=RTOL)
    st = eng.stats()
    assert st["pairs_done"] == total and st["pinned_at_end"] == 0 and st["evictions"] > 0


@pytest.mark.parametrize("side,n,cams", [(1024, 64, 8), (256, 72, 6)])
def test_engine_bench_path_many_pairs_per_cta(side, n, cams):
    """The exact path bench.py times, checked pair by pair against the oracle.

    Engine, leaf 8, all items resident, device inputs -- as bench.py -- with n
    large enough that a compare launch carries a whole number of rounds of the
    persistent grid (1,924 pairs = 13 per CTA at 1024^2 on 148 SMs).  Every CTA
    therefore runs several pairs back to back: carried mbarrier phases, T-slot
    reuse and the staging-buffer refills are all on this path.  Every pair of the
    job is compared with the float64 oracle (scipy-batched inverse FFTs)."""
    _l, device = _lib()
    items = make_items(n, side, cameras=cams, seed=17)
    eng = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side, threshold=60.0),
                              leaf_block=8, device_slots=n)
    eng.set_profiling(every=1, max_samples=256)
    total = n * (n - 1) // 2
    out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    flags = torch.zeros(total, dtype=torch.uint8, device="cuda")
    eng.run(out, flags, device_items=items, parsed_stride=side * side * 4)
    _, launches, launched_pairs = eng.kernel_time()
    assert launched_pairs == total
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    # pairs per launch exceed the number of persistent CTAs several times over
    assert total / launches >= 4 * sms, (total, launches, sms)
    host = items.cpu().numpy().reshape(n, side, side)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    want = opce.pairs_batched(host, pairs)
    got = out.cpu().numpy()
    np.testing.assert_allclose(got, want, rtol=RTOL)
    f = flags.cpu().numpy()
    assert np.array_equal(f == 3, got >= 60.0) and np.all((f == 1) | (f == 3))
    st = eng.stats()
    assert st["pairs_done"] == total and st["loads"] == n


def test_2048_many_pairs_per_cta_sampled():
    """C3 item shape, 780 pairs in one launch (> 5 per persistent CTA), through the
    engine as bench.py --side 2048 (and its C3 mode) runs it; 96 sampled pairs
    (first and last pairs of the launch included) against the float64 oracle."""
    _l, device = _lib()
    side, n = 2048, 40
    items = make_items(n, side, cameras=4, seed=23)
    eng = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side, threshold=60.0),
                              leaf_block=8, device_slots=n)
    eng.set_profiling(every=1, max_samples=64)
    total = n * (n - 1) // 2
    out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    flags = torch.zeros(total, dtype=torch.uint8, device="cuda")
    eng.run(out, flags, device_items=items, parsed_stride=side * side * 4)
    _, launches, launched_pairs = eng.kernel_time()
    assert launched_pairs == total and launches == 1
    got = out.cpu().numpy()
    assert np.all(np.isfinite(got))
    rng = np.random.default_rng(5)
    pids = sorted(set([0, 1, total - 2, total - 1] + rng.choice(total, 92, replace=False).tolist()))
    from oracle import scheduler as osch
    pairs = [osch.pair_from_id(n, int(p)) for p in pids]
    host = items.cpu().numpy().reshape(n, side, side)
    want = opce.pairs_batched(host, pairs, batch=4)
    np.testing.assert_allclose(got[pids], want, rtol=RTOL)
    f = flags.cpu().numpy()
    assert np.array_equal(f == 3, got >= 60.0) and np.all((f == 1) | (f == 3))


@pytest.mark.parametrize("host_slots", [0, 8, 24])
def test_engine_host_tier_write_through(host_slots):
    """Host (L2) tier of preprocessed items (engine.py:375-394, write-through
    :482-508): with a device tier far smaller than n, device misses are served from
    pinned host slots instead of re-preprocessing; with host_slots >= n every item
    is preprocessed exactly once (R = 1), smaller host tiers evict (LRU) and reload.
    Results are bit-identical to the run without a host tier."""
    _l, device = _lib()
    side, n = 256, 24
    items = make_items(n, side, cameras=3, seed=31)
    total = n * (n - 1) // 2
    eng = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side), leaf_block=4,
                              device_slots=6, host_slots=host_slots)
    out = torch.zeros(total, dtype=torch.float64, device="cuda")
    host = items.cpu().pin_memory()
    eng.run(out, host_items=host, parsed_stride=side * side * 4)
    st = eng.stats()
    got = out.cpu().numpy()
    ref = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side), leaf_block=4, device_slots=n)
    want = torch.zeros(total, dtype=torch.float64, device="cuda")
    ref.run(want, device_items=items, parsed_stride=side * side * 4)
    np.testing.assert_array_equal(got, want.cpu().numpy())
    assert st["evictions"] > 0 and st["pinned_at_end"] == 0 and st["ledger_marked"] == total
    if host_slots == 0:
        assert st["loads"] > n and st["host_hits"] == 0
    else:
        assert st["host_hits"] > 0 and st["host_hits"] + st["host_misses"] == st["misses"]
        assert st["loads"] == st["host_misses"]                       # a load is a fresh preprocess
        assert st["d2h_bytes"] == st["host_misses"] * side * side * 4  # written through once per load
        if host_slots >= n:
            assert st["loads"] == n and st["host_evictions"] == 0     # R = 1
        else:
            assert st["loads"] > n and st["host_evictions"] > 0


@pytest.mark.parametrize("side,n,runs", [(256, 72, 4), (1024, 40, 2)])
def test_compare_is_deterministic_run_to_run(side, n, runs):
    """The same job, run repeatedly with many pairs per persistent CTA, is
    bit-identical: no staging buffer is refilled (TMA, async proxy) while another
    thread's generic loads of it may still be in flight (tools/pce_determinism.py
    found 2-3 of 2,556 values differing before the refill proxy fences)."""
    _l, device = _lib()
    items = make_items(n, side, cameras=6, seed=17)
    total = n * (n - 1) // 2
    outs = []
    for _ in range(runs):
        eng = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side), leaf_block=8,
                                  device_slots=n)
        out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
        eng.run(out, device_items=items, parsed_stride=side * side * 4)
        outs.append(out.cpu().numpy())
        eng.close()
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])


@pytest.mark.parametrize("side,n", [(1024, 40), (2048, 24)])
def test_round_barrier_and_l2_hints_do_not_change_results(side, n, monkeypatch):
    """The compare grid's round barrier (RK_PCE_LOCKSTEP) and L2 hints
    (RK_PCE_L2OPTS) only change timing: with them on (the defaults) and off, the
    same job gives bit-identical PCE values, including a launch whose last round
    is partial (n = 40: 780 pairs = 5 rounds of 148 + 40); the defaults match the
    float64 oracle on a sample."""
    _l, device = _lib()
    items = make_items(n, side, cameras=6, seed=23)
    total = n * (n - 1) // 2
    outs = {}
    for lock, l2 in (("1", None), ("0", "0"), ("1", "3")):
        monkeypatch.setenv("RK_PCE_LOCKSTEP", lock)
        if l2 is None:
            monkeypatch.delenv("RK_PCE_L2OPTS", raising=False)
        else:
            monkeypatch.setenv("RK_PCE_L2OPTS", l2)
        eng = device.DeviceEngine(_l.app_params(_l.APP_PCE, n, height=side, width=side), leaf_block=8,
                                  device_slots=n)
        out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
        eng.run(out, device_items=items, parsed_stride=side * side * 4)
        outs[(lock, l2)] = out.cpu().numpy()
        eng.close()
    base = outs[("1", None)]
    assert np.isfinite(base).all()
    for o in outs.values():
        np.testing.assert_array_equal(o, base)
    host = items.cpu().numpy().reshape(n, side, side)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    pick = np.random.default_rng(5).choice(total, size=8, replace=False)
    want = opce.pairs_batched(host, [pairs[p] for p in pick])
    np.testing.assert_allclose(base[pick], want, rtol=RTOL)


def test_synthetic_patterns_match_the_oracle_generator():
    """rk_synth_prnu (the bench's storage stage) against its float64 restatement
    (oracle/pce.py prnu_patterns) to fp32 rounding, and bit-identical whether items
    are generated in one call or one at a time at any key offset."""
    _l, device = _lib()
    side, n = 256, 5
    one = make_items(n, side, cameras=3, seed=7)
    each = torch.empty_like(one)
    for k in range(n):
        device.synth_prnu(side, side, k, 1, 3, 7, each[k * side * side:(k + 1) * side * side])
    torch.cuda.synchronize()
    assert torch.equal(one, each)
    want = opce.prnu_patterns(side, side, 0, n, 3, 7)
    np.testing.assert_allclose(one.cpu().numpy().reshape(n, side, side), want, rtol=1e-4, atol=1e-4)
