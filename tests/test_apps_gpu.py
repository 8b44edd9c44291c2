"""The reference's two built-in applications on the CUDA path, against golden vectors
generated from the reference itself, plus the Application-contract per-pair path."""

import json
import os
import struct

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def _mods():
    from paper_2009_04755_b200 import _lib, device
    return _lib, device


@pytest.mark.parametrize("leaf,slots", [(8, 0), (3, 7)])
def test_synthetic_engine_bit_exact(leaf, slots):
    _l, device = _mods()
    for case in load("synthetic.json")["cases"]:
        n, seed = case["n"], case["seed"]
        eng = device.DeviceEngine(_l.app_params(_l.APP_SYNTHETIC, n, seed=seed), leaf_block=leaf,
                                  device_slots=slots or n)
        out = torch.full((n * (n - 1) // 2,), float("nan"), dtype=torch.float64, device="cuda")
        flags = torch.full_like(out, 255, dtype=torch.uint8)
        eng.run(out, flags)
        got = [float(v).hex() for v in out.cpu().numpy()]
        assert got == case["values"], seed
        assert int(flags.cpu().max()) == 0          # match is None (apps.py:210-212)
        eng.close()


def test_synthetic_pairs_batch_bit_exact():
    _l, device = _mods()
    case = load("synthetic.json")["cases"][3]
    n, seed = case["n"], case["seed"]
    app = device.DeviceApp(_l.app_params(_l.APP_SYNTHETIC, n, seed=seed))
    out = torch.zeros(n * (n - 1) // 2, dtype=torch.float64, device="cuda")
    pairs = [(i, j, 0, 0) for i in range(n) for j in range(i + 1, n)][::-1]
    app.compare_pairs(out, pairs, out)
    assert [float(v).hex() for v in out.cpu().numpy()] == case["values"]


def pack_parsed(parsed_hex, stride):
    buf = np.zeros((len(parsed_hex), stride), dtype=np.uint8)
    for k, h in enumerate(parsed_hex):
        b = bytes.fromhex(h)
        buf[k, :len(b)] = np.frombuffer(b, dtype=np.uint8)
    return torch.from_numpy(buf.reshape(-1))


@pytest.mark.parametrize("name", ["five_docs_k2", "engine_seed0_k3", "acceptance_c04b05_k3", "mixed_k4"])
def test_cv_kernels_match_reference(name):
    _l, device = _mods()
    g = load("cv.json")[name]
    n = len(g["parsed"])
    app = device.DeviceApp(_l.app_params(_l.APP_CV, n, max_entries=512, threshold=0.5))
    parsed = pack_parsed(g["parsed"], app.parsed_bytes).cuda()
    slots = app.alloc_slots(n)
    app.preprocess(parsed, app.parsed_bytes, n, slots, list(range(n)))
    out = torch.zeros(n * (n - 1) // 2, dtype=torch.float64, device="cuda")
    flags = torch.zeros_like(out, dtype=torch.uint8)
    app.compare_tile(slots, 0, n, 0, n, list(range(n)), out, flags)
    want = np.array([float.fromhex(v) for v in g["values"]])
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-12, atol=1e-15)
    match = [None if m is None else bool(m) for m in g["match"]]
    got = [(f & 1) and bool(f & 2) for f in flags.cpu().numpy().tolist()]
    assert got == match
    # frequencies and norms in the slot layout: u32 dim | pad | f64 norm | u64 tok[cap] | f64 freq[cap]
    raw = slots.cpu().numpy()
    for k, pre_hex in enumerate(g["preprocessed"]):
        pre = bytes.fromhex(pre_hex)
        dim = struct.unpack_from("<I", pre)[0]
        base = k * app.slot_stride
        assert struct.unpack_from("<I", raw[base:base + 4].tobytes())[0] == dim
        toks = raw[base + 16: base + 16 + 8 * dim].view(np.uint64)
        freqs = raw[base + 16 + 8 * 512: base + 16 + 8 * 512 + 8 * dim].view(np.float64)
        ref = [struct.unpack_from("<Qd", pre, 4 + 16 * e) for e in range(dim)]
        assert [int(t) for t in toks] == [t for t, _ in ref]
        assert [float(f).hex() for f in freqs] == [f.hex() for _, f in ref]   # count/total bit-exact


@pytest.mark.parametrize("host_slots", [0, 16])
def test_cv_engine_with_eviction_matches_reference(host_slots):
    """Tight device tier (7 slots for 16 items); with a 16-slot host tier every
    document is preprocessed once (R = 1) and device misses are host hits."""
    _l, device = _mods()
    g = load("cv.json")["acceptance_c04b05_k3"]
    n = len(g["parsed"])
    eng = device.DeviceEngine(_l.app_params(_l.APP_CV, n, max_entries=256, threshold=0.5), leaf_block=3,
                              device_slots=7, host_slots=host_slots)
    app = device.DeviceApp(_l.app_params(_l.APP_CV, n, max_entries=256))
    host = pack_parsed(g["parsed"], app.parsed_bytes).pin_memory()
    out = torch.zeros(n * (n - 1) // 2, dtype=torch.float64, device="cuda")
    eng.run(out, host_items=host, parsed_stride=app.parsed_bytes)
    want = np.array([float.fromhex(v) for v in g["values"]])
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-12, atol=1e-15)
    st = eng.stats()
    assert st["pairs_done"] == 120 and st["evictions"] > 0 and st["ledger_marked"] == 120
    if host_slots:
        assert st["loads"] == n and st["host_hits"] > 0
    else:
        assert st["loads"] > n


def test_cv_slot_overflow_and_malformed():
    _l, device = _mods()
    from paper_2009_04755_b200.errors import MalformedInput, SlotOverflow
    g = load("cv.json")["engine_seed0_k3"]
    app = device.DeviceApp(_l.app_params(_l.APP_CV, 2, max_entries=8))
    parsed = pack_parsed(g["parsed"][:1], 4 + 12 * 64)[: app.parsed_bytes].cuda()
    slots = app.alloc_slots(1)
    with pytest.raises(SlotOverflow):
        app.preprocess(parsed, app.parsed_bytes, 1, slots, [0])
    empty = torch.zeros(app.parsed_bytes, dtype=torch.uint8, device="cuda")
    with pytest.raises(MalformedInput):
        app.preprocess(empty, app.parsed_bytes, 1, slots, [0])


def test_application_contract_per_pair(tmp_path):
    """The reference-facing per-pair path: fetch_raw -> parse -> preprocess -> compare -> postprocess."""
    from paper_2009_04755_b200.apps import CompositionVectorApp, ItemData, PCEApp, Stage, SyntheticApp
    from oracle import cv as ocv
    from oracle import pce as opce
    from oracle import rng as orng

    g = load("cv.json")["five_docs_k2"]
    for idx, text in enumerate(g["texts"]):
        (tmp_path / f"d{idx}.txt").write_text(text)
    cv = CompositionVectorApp(str(tmp_path), k=2)
    items = {}
    for key in range(cv.n):
        raw = ItemData(Stage.RAW_FILE, cv.fetch_raw(cv.path_for_key(key)))
        parsed = cv.parse(key, raw)
        assert parsed.payload.hex() == g["parsed"][key]
        items[key] = cv.preprocess(key, parsed)
    k = 0
    for i in range(cv.n):
        for j in range(i + 1, cv.n):
            res = cv.postprocess((i, j), cv.compare((i, items[i]), (j, items[j])))
            assert res.value == pytest.approx(float.fromhex(g["values"][k]), abs=1e-12)
            assert res.match == g["match"][k]
            k += 1
    with pytest.raises(ValueError):
        cv.compare((1, items[1]), (0, items[0]))
    with pytest.raises(ValueError):
        cv.compare((0, ItemData(Stage.PARSED, b"x")), (1, items[1]))

    syn = SyntheticApp(n=5, seed=5)
    pre = {k: syn.preprocess(k, syn.parse(k, ItemData(Stage.RAW_FILE, syn.fetch_raw(syn.path_for_key(k)))))
           for k in range(5)}
    raw = syn.compare((1, pre[1]), (3, pre[3]))
    assert struct.unpack("<d", raw)[0] == orng.synthetic_value(5, 1, 3)
    assert syn.postprocess((1, 3), raw).match is None

    pce = PCEApp(3, side=256, cameras=1, seed=4)
    pre = {}
    for key in range(3):
        raw = ItemData(Stage.RAW_FILE, pce.fetch_raw(pce.path_for_key(key)))
        pre[key] = pce.preprocess(key, pce.parse(key, raw))
    pats = np.stack([np.frombuffer(pce.fetch_raw(pce.path_for_key(key)), dtype=np.float32).reshape(256, 256)
                     for key in range(3)])
    want = opce.all_pairs(pats)
    got = [pce.postprocess((i, j), pce.compare((i, pre[i]), (j, pre[j]))) for i in range(3) for j in range(i + 1, 3)]
    np.testing.assert_allclose([r.value for r in got], want, rtol=1e-4)
    assert all(r.match for r in got)        # one camera: every pair matches at PCE >= 60
    assert pce.stage_cost("compare", 0, 1) == 0.0


def test_allpairs_engine_public_api(tmp_path):
    from paper_2009_04755_b200.apps import PCEApp
    from paper_2009_04755_b200.engine import AllPairsEngine
    from oracle import pce as opce
    app = PCEApp(10, side=256, cameras=3, seed=2)
    eng = AllPairsEngine(app, leaf_block=4, device_slots=6)
    res = eng.run()
    pats = np.stack([np.frombuffer(app.fetch_raw(app.path_for_key(k)), dtype=np.float32).reshape(256, 256)
                     for k in range(10)])
    np.testing.assert_allclose(res.values, opce.all_pairs(pats), rtol=1e-4)
    assert res.stats["pairs_done"] == 45 and res.r_factor > 1.0     # 6 slots < 10 items: reloads
    r = res.result(2, 5)
    assert r.left == 2 and r.right == 5 and r.match == (2 % 3 == 5 % 3)
    assert len(res.results()) == 45
    eng.close()


def test_cv_large_skewed_items_match_oracle():
    """Windowed merge over long, skewed token lists: sizes 1 .. 60k, identical,
    disjoint, nested and heavily overlapping items, matches straddling the warp
    partitions; against the oracle's sequential merge (oracle/cv.py) at 1e-12."""
    from oracle import cv as ocv
    _l, device = _mods()
    rng = np.random.default_rng(5)
    pool = np.unique(rng.integers(1, 1 << 40, size=200_000).astype(np.uint64))
    sizes = [1, 2, 31, 33, 1000, 60_000, 60_000, 45_000, 5_000, 20_000, 7]
    toks = []
    for k, m in enumerate(sizes):
        if k == 6:
            t = toks[5]                                   # identical to item 5
        elif k == 7:
            t = np.sort(rng.choice(toks[5], size=m, replace=False))   # nested in item 5
        elif k == 8:
            t = np.unique(rng.integers(1 << 41, 1 << 42, size=m).astype(np.uint64))   # disjoint range
        else:
            t = np.sort(rng.choice(pool, size=m, replace=False))
        toks.append(t)
    n, cap = len(toks), max(len(t) for t in toks)
    stride = 4 + 12 * cap
    buf = np.zeros((n, stride), dtype=np.uint8)
    vecs = []
    counts = []
    for k, t in enumerate(toks):
        cnt = counts[5] if k == 6 else rng.integers(1, 9, size=len(t)).astype(np.uint32)
        counts.append(cnt)
        rec = np.zeros(len(t), dtype=[("t", "<u8"), ("c", "<u4")])
        rec["t"], rec["c"] = t, cnt
        blob = struct.pack("<I", len(t)) + rec.tobytes()
        buf[k, :len(blob)] = np.frombuffer(blob, dtype=np.uint8)
        vecs.append(ocv.preprocess(blob))
    app = device.DeviceApp(_l.app_params(_l.APP_CV, n, max_entries=cap, threshold=0.5))
    slots = app.alloc_slots(n)
    app.preprocess(torch.from_numpy(buf.reshape(-1)).cuda(), stride, n, slots, list(range(n)))
    out = torch.zeros(n * (n - 1) // 2, dtype=torch.float64, device="cuda")
    app.compare_tile(slots, 0, n, 0, n, list(range(n)), out)
    got = out.cpu().numpy()
    pid = 0
    for i in range(n):
        for j in range(i + 1, n):
            want = ocv.compare(vecs[i], vecs[j])
            assert abs(got[pid] - want) <= 1e-12 * max(1.0, abs(want)), (i, j, got[pid], want)
            pid += 1
    assert got[5 * (2 * n - 5 - 1) // 2 + 0] == pytest.approx(1.0, abs=1e-12)   # identical items 5, 6


def test_exactly_once_over_random_runs():
    """The reference's release criterion "every pair exactly once" over randomized
    runs (test_acceptance.py:56-86): random n, leaf size, tier capacity and rank
    count; the ranks' static shares together write each pair id once, and the
    synthetic values are bit-exact with the reference's mix64 (oracle/rng.py)."""
    from oracle import rng as orng
    _l, device = _mods()
    r = np.random.default_rng(2024)
    for _ in range(40):
        n = int(r.integers(2, 90))
        leaf = int(r.integers(1, 12))
        world = int(r.integers(1, 4))
        seed = int(r.integers(0, 2**63))
        total = n * (n - 1) // 2
        cover = torch.zeros(total, dtype=torch.int32, device="cuda")
        vals = torch.zeros(total, dtype=torch.float64, device="cuda")
        for rank in range(world):
            eng = device.DeviceEngine(_l.app_params(_l.APP_SYNTHETIC, n, seed=seed), leaf_block=leaf,
                                      device_slots=int(r.integers(2, n + 2)), rank=rank, world=world)
            out = torch.zeros(total, dtype=torch.float64, device="cuda")
            flags = torch.full((total,), 255, dtype=torch.uint8, device="cuda")
            eng.run(out, flags)
            touched = flags != 255
            cover += touched.to(torch.int32)
            vals += torch.where(touched, out, torch.zeros_like(out))
            eng.close()
        assert bool((cover == 1).all()), (n, leaf, world)
        want = np.array([orng.synthetic_value(seed, i, j) for i in range(n) for j in range(i + 1, n)])
        assert np.array_equal(vals.cpu().numpy(), want), (n, leaf, world, seed)
