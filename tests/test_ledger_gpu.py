"""Exactly-once ledger on the device (PairLedger, scheduler.py:218-246).

Every compare epilogue sets its pair's bit with a system-scope atomicOr; a bit
that was already set is a duplicate completion, which the reference treats as
a scheduling bug (AssertionError "pair (i, j) completed twice",
scheduler.py:233-241) -- the analogue of test_scheduler.py:183-211."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _mods():
    from paper_2009_04755_b200 import _lib, device
    return _lib, device


@pytest.mark.parametrize("kind", ["pce", "synthetic", "ncc"])
def test_engine_run_fills_the_ledger_exactly_once(kind):
    _l, device = _mods()
    n, side = 40, 256
    if kind == "pce":
        params = _l.app_params(_l.APP_PCE, n, height=side, width=side, threshold=60.0)
    elif kind == "ncc":
        n = 300
        params = _l.app_params(_l.APP_NCC, n, height=side, width=side, threshold=0.02)
    else:
        params = _l.app_params(_l.APP_SYNTHETIC, n, seed=3, threshold=0.5)
    items = torch.empty(n * side * side, dtype=torch.float32, device="cuda")
    device.synth_prnu(side, side, 0, n, 4, 5, items)
    eng = device.DeviceEngine(params, leaf_block=8, device_slots=n)
    total = n * (n - 1) // 2
    out = torch.zeros(total, dtype=torch.float64, device="cuda")
    for _ in range(2):   # the ledger is cleared at the start of every run
        eng.run(out, device_items=items if kind != "synthetic" else None, parsed_stride=side * side * 4)
        st = eng.stats()
        assert st["ledger_marked"] == total and st["dup_marks"] == 0
        led = eng.check_ledger()
        assert led["total"] == total and led["completed"] == total and led["full"] == 1
    eng.close()


def test_duplicate_completion_is_an_assertion():
    """Two runs of the same job into one shared ledger without a reset: every pair
    is marked twice; the ledger counts the duplicates and the check raises the
    reference's AssertionError naming the first pair."""
    _l, device = _mods()
    n, side = 12, 256
    items = torch.empty(n * side * side, dtype=torch.float32, device="cuda")
    device.synth_prnu(side, side, 0, n, 2, 8, items)
    params = _l.app_params(_l.APP_PCE, n, height=side, width=side)
    owner = device.DeviceEngine(params, leaf_block=4, device_slots=n)
    other = device.DeviceEngine(params, leaf_block=4, device_slots=n)
    other.use_ledger(owner.ledger_region_ptr())     # marks go to the owner's ledger, like rank r > 0
    owner.use_ledger(owner.ledger_region_ptr())     # the owner's ledger is now the shared one
    owner.ledger_reset()
    total = n * (n - 1) // 2
    out = torch.zeros(total, dtype=torch.float64, device="cuda")
    other.run(out, device_items=items, parsed_stride=side * side * 4)
    assert owner.check_ledger()["full"] == 1
    owner.run(out, device_items=items, parsed_stride=side * side * 4)   # the same pairs again
    led = owner.ledger()
    assert led["dup_marks"] == total and led["completed"] == total and led["full"] == 0
    assert led["first_dup_pid"] >= 0
    with pytest.raises(AssertionError, match="completed twice"):
        owner.check_ledger()
    owner.ledger_reset()
    assert owner.ledger()["completed"] == 0


def test_private_ledger_duplicate_fails_the_call():
    """Per-pair API with a caller-owned ledger: a pair compared twice is counted."""
    _l, device = _mods()
    n, side = 4, 256
    items = torch.empty(n * side * side, dtype=torch.float32, device="cuda")
    device.synth_prnu(side, side, 0, n, 2, 9, items)
    app = device.DeviceApp(_l.app_params(_l.APP_PCE, n, height=side, width=side))
    slots = app.alloc_slots(n)
    app.preprocess(items, side * side * 4, n, slots, list(range(n)))
    region = app.ledger_region()
    app.set_ledger(region)
    out = torch.zeros(6, dtype=torch.float64, device="cuda")
    app.compare_pairs(slots, [(0, 1, 0, 1), (2, 3, 2, 3)], out)
    led = app.ledger(region)
    assert led["completed"] == 2 and led["dup_marks"] == 0
    app.compare_pairs(slots, [(2, 3, 2, 3)], out)
    led = app.ledger(region)
    assert led["completed"] == 2 and led["dup_marks"] == 1 and led["first_dup_pid"] == 5
    app.set_ledger(None)
    app.compare_pairs(slots, [(2, 3, 2, 3)], out)                 # ledger off: not counted
    assert app.ledger(region)["dup_marks"] == 1
