"""NCC: the tcgen05 Gram path and the per-pair path vs the float64 oracle.

Stated bounds: TF32 Gram |error| <= 2e-4 (10-bit operand mantissa, normalised
items); fp32 per-pair path |error| <= 1e-5."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ncc as oncc  # noqa: E402


def _mods():
    from paper_2009_04755_b200 import _lib, device
    return _lib, device


def make_items(n, side, seed=3, cameras=4):
    _, device = _mods()
    buf = torch.empty(n * side * side, dtype=torch.float32, device="cuda")
    device.synth_prnu(side, side, 0, n, cameras, seed, buf)
    return buf


@pytest.mark.parametrize("n", [37, 200, 600])
def test_gram_matches_oracle(n):
    """37: single-CTA 128x128 kernel; 200, 600: CTA-pair 256x256 kernel (one tile
    with zero-filled rows beyond n; six tiles)."""
    _l, device = _mods()
    side = 256
    items = make_items(n, side)
    eng = device.DeviceEngine(_l.app_params(_l.APP_NCC, n, height=side, width=side, threshold=0.02),
                              device_slots=n)
    total = n * (n - 1) // 2
    out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    flags = torch.zeros(total, dtype=torch.uint8, device="cuda")
    eng.run(out, flags, device_items=items, parsed_stride=side * side * 4)
    want = oncc.all_pairs(items.cpu().numpy().reshape(n, side, side).astype(np.float64))
    got = out.cpu().numpy()
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - want)) <= 2e-4
    # same-camera items correlate at ~0.2^2/(1+0.2^2) = 0.038, others at ~1/sqrt(D)
    assert np.array_equal(flags.cpu().numpy() == 3, got >= 0.02)
    st = eng.stats()
    assert st["pairs_done"] == total and st["loads"] == n


def test_gram_sharded_across_ranks_covers_all_pairs():
    _l, device = _mods()
    n, side = 300, 128
    items = make_items(n, side, seed=8)
    total = n * (n - 1) // 2
    acc = torch.zeros(total, dtype=torch.float64, device="cuda")
    done = 0
    for rank in range(3):
        eng = device.DeviceEngine(_l.app_params(_l.APP_NCC, n, height=side, width=side), device_slots=n,
                                  rank=rank, world=3)
        out = torch.zeros(total, dtype=torch.float64, device="cuda")
        eng.run(out, device_items=items, parsed_stride=side * side * 4)
        acc += out
        done += eng.stats()["pairs_done"]
    assert done == total
    want = oncc.all_pairs_chunked(items.cpu().numpy().reshape(n, side, side))
    assert np.max(np.abs(acc.cpu().numpy() - want)) <= 2e-4


def test_pairs_path_and_known_answers():
    _l, device = _mods()
    side = 256
    base = make_items(2, side, seed=11).view(2, side, side)
    items = torch.stack([base[0], base[0] * 3.0 + 1.5, -base[0], base[1]]).contiguous().view(-1)
    app = device.DeviceApp(_l.app_params(_l.APP_NCC, 4, height=side, width=side))
    slots = app.alloc_slots(4)
    app.preprocess(items, side * side * 4, 4, slots, [0, 1, 2, 3])
    out = torch.zeros(6, dtype=torch.float64, device="cuda")
    app.compare_tile(slots, 0, 4, 0, 4, [0, 1, 2, 3], out)
    got = out.cpu().numpy()
    want = oncc.all_pairs(items.cpu().numpy().reshape(4, side, side).astype(np.float64))
    np.testing.assert_allclose(got, want, atol=1e-5)
    assert got[0] == pytest.approx(1.0, abs=1e-5)       # scale/offset invariance
    assert got[1] == pytest.approx(-1.0, abs=1e-5)      # x vs -x
    assert abs(got[2]) < 0.05


def test_constant_item_is_malformed():
    _l, device = _mods()
    from paper_2009_04755_b200.errors import MalformedInput
    app = device.DeviceApp(_l.app_params(_l.APP_NCC, 2, height=64, width=64))
    slots = app.alloc_slots(1)
    flat = torch.ones(64 * 64, dtype=torch.float32, device="cuda")
    with pytest.raises(MalformedInput):
        app.preprocess(flat, 64 * 64 * 4, 1, slots, [0])


def test_gram_blocks_over_a_partial_arena():
    """C3-style NCC: items split into key blocks placed anywhere in the arena (slot
    groups of 128); the triangle of each block plus the rectangle between them
    covers every pair exactly once and matches the oracle."""
    _l, device = _mods()
    n, side = 600, 256
    d = side * side
    items = make_items(n, side, seed=12)
    app = device.DeviceApp(_l.app_params(_l.APP_NCC, n, height=side, width=side, threshold=0.02))
    arena_rows = 768
    slots = app.alloc_slots(arena_rows)
    a_key0, a_cnt, a_row0 = 0, 256, 384          # keys 0..255 at slots 384..639
    b_key0, b_cnt, b_row0 = 256, 344, 0          # keys 256..599 at slots 0..343
    app.preprocess(items, d * 4, a_cnt, slots, list(range(a_row0, a_row0 + a_cnt)))
    app.preprocess(items[b_key0 * d:], d * 4, b_cnt, slots, list(range(b_row0, b_row0 + b_cnt)))
    total = n * (n - 1) // 2
    out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    flags = torch.zeros(total, dtype=torch.uint8, device="cuda")
    device.ncc_gram_block(app, slots, arena_rows, a_row0, a_key0, a_cnt, a_row0, a_key0, a_cnt, out, flags)
    device.ncc_gram_block(app, slots, arena_rows, b_row0, b_key0, b_cnt, b_row0, b_key0, b_cnt, out, flags)
    # the rectangle, passed B-first: the ABI orders the blocks so that i < j
    device.ncc_gram_block(app, slots, arena_rows, b_row0, b_key0, b_cnt, a_row0, a_key0, a_cnt, out, flags)
    torch.cuda.synchronize()
    want = oncc.all_pairs(items.cpu().numpy().reshape(n, side, side).astype(np.float64))
    got = out.cpu().numpy()
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - want)) <= 2e-4
    f = flags.cpu().numpy()
    assert np.all((f == 1) | (f == 3)) and np.array_equal(f == 3, got >= 0.02)
    with pytest.raises(ValueError):   # overlapping key ranges are not a valid block pair
        device.ncc_gram_block(app, slots, arena_rows, 0, 0, 256, 384, 128, 256, out)


@pytest.mark.parametrize("world,side", [(1, 128), (2, 128), (1, 512)])
def test_engine_blocked_gram_when_items_exceed_slots(world, side):
    """device_slots < n: the engine runs the Gram over key blocks that fit (half the
    arena each), loading blocks as needed; ranks take block pairs round-robin.
    side 512: D = 262,144 = two K chunks, so every block triangle and rectangle
    also goes through the chunk-accumulate epilogue."""
    _l, device = _mods()
    n = 600
    items = make_items(n, side, seed=14)
    total = n * (n - 1) // 2
    acc = torch.zeros(total, dtype=torch.float64, device="cuda")
    fl = torch.zeros(total, dtype=torch.int32, device="cuda")
    done = loads = 0
    for rank in range(world):
        eng = device.DeviceEngine(_l.app_params(_l.APP_NCC, n, height=side, width=side, threshold=0.02),
                                  device_slots=512, rank=rank, world=world)
        out = torch.zeros(total, dtype=torch.float64, device="cuda")
        flags = torch.zeros(total, dtype=torch.uint8, device="cuda")
        eng.run(out, flags, device_items=items, parsed_stride=side * side * 4)
        acc += out
        fl += flags.to(torch.int32)
        st = eng.stats()
        done += st["pairs_done"]
        loads += st["loads"]
    assert done == total and loads > n            # blocks reloaded: R > 1
    f = fl.cpu().numpy()
    assert np.all((f == 1) | (f == 3))             # every pair exactly once
    want = oncc.all_pairs_chunked(items.cpu().numpy().reshape(n, side, side))
    assert np.max(np.abs(acc.cpu().numpy() - want)) <= 2e-4


@pytest.mark.parametrize("side", [512, 1024])
def test_gram_multi_k_chunk_matches_oracle(side):
    """BASELINE item sizes take the K-chunked Gram: D = side^2 is streamed in chunks
    of 131,072 elements, one launch each; chunk 0 stores, later chunks add into
    out[pid] in fp64 and the last one writes the flags (ncc.cu).  512^2 = 2 chunks,
    1024^2 = 8 chunks (the C2/C3 item size class).  n = 300 runs the CTA-pair
    256 x 256 kernel with a ragged last tile.  Bound: |error| <= 2e-4 (TF32)."""
    _l, device = _mods()
    n = 300
    items = make_items(n, side, seed=19, cameras=6)
    eng = device.DeviceEngine(_l.app_params(_l.APP_NCC, n, height=side, width=side, threshold=0.02),
                              device_slots=n)
    total = n * (n - 1) // 2
    out = torch.full((total,), float("nan"), dtype=torch.float64, device="cuda")
    flags = torch.zeros(total, dtype=torch.uint8, device="cuda")
    eng.run(out, flags, device_items=items, parsed_stride=side * side * 4)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    want = oncc.all_pairs_chunked(items.cpu().numpy().reshape(n, side * side))
    assert np.all(np.isfinite(got))
    err = np.max(np.abs(got - want))
    assert err <= 2e-4, err
    f = flags.cpu().numpy()
    assert np.all((f == 1) | (f == 3)) and np.array_equal(f == 3, got >= 0.02)
    st = eng.stats()
    assert st["pairs_done"] == total and st["loads"] == n
