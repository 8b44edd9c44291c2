"""Drop-in proof: the UNMODIFIED reference RealEngine (realrun.py:28-176) runs the
librocket-backed Application classes of integration/allpairs_b200.py.

The reference package is the one oracle/Makefile staged into oracle/_ref (an
offline pip install of /root/reference/pkg; it travels to the GPU box with the
snapshot).  Parity:
  * PCE: the master's results against the float64 oracle (oracle/pce.py) at 1e-4;
  * CV: the master's results against the reference's own CompositionVectorApp run
    through the same RealEngine on the same corpus (apps.py:331-354) at 1e-12.
Both runs must leave the reference's PairLedger full (engine.py:571-582)."""

import importlib.util
import os
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(HERE, "oracle", "_ref")


def _reference():
    if not os.path.isdir(os.path.join(REF, "allpairs")):
        pytest.fail("oracle/_ref is missing: run `make -C oracle` (or __graft_entry__.build()) where "
                    "/root/reference exists, before shipping the snapshot")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    spec = importlib.util.spec_from_file_location("allpairs_b200", os.path.join(HERE, "integration",
                                                                                  "allpairs_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _config(devices=1, device_slots=8, host_slots=16, leaf=4):
    from allpairs.config import NodeShape, RunConfig
    return RunConfig(app={"kind": "drop-in"}, mode="real", seed=0, leaf_block=leaf,
                     nodes=[NodeShape(device_speeds=[1.0] * devices, device_slots=device_slots,
                                      host_slots=host_slots, cpu_width=4)])


@pytest.mark.parametrize("devices", [1, 2])
def test_realengine_runs_b200_pce(devices):
    """devices = 2: two gpu lane threads call the binding concurrently (its lock)."""
    mod = _reference()
    from allpairs.apps import ItemData, Stage
    from allpairs.realrun import RealEngine
    from oracle import pce as opce

    n, side = 24, 256
    pats = opce.prnu_patterns(side, side, 0, n, 3, 29)

    class SyntheticPRNU(mod.B200PCEApp):
        def path_for_key(self, key):
            return f"prnu/{key:05d}.f32"

        def fetch_raw(self, path):
            return pats[int(path[5:10])].tobytes()

        def parse(self, key, raw):
            return ItemData(Stage.PARSED, raw.payload)

    app = SyntheticPRNU(n, side=side, threshold=60.0)
    master = RealEngine(_config(devices=devices), app, run_timeout=600).run()
    assert master.ledger.full and master.ledger.completed == n * (n - 1) // 2
    want = opce.all_pairs(pats)
    pid = 0
    for i in range(n):
        for j in range(i + 1, n):
            r = master.results[(i, j)]
            assert r.value == pytest.approx(want[pid], rel=1e-4), (i, j)
            assert r.match == (want[pid] >= 60.0)
            pid += 1
    # the reference's cache accounting ran over the binding's items: every item loaded
    assert master.metrics.loads >= n


def _write_corpus(tmp_path, count=16, seed=0xC04B05, length=160):
    """The reference acceptance corpus shape (test_acceptance.py:273-321): mix64 DNA text."""
    from allpairs.rng import mix64
    for idx in range(count):
        state = mix64(seed, idx)
        chars = []
        for pos in range(length):
            state = mix64(state, pos)
            chars.append("ACGT"[state % 4])
        (tmp_path / f"doc{idx:02d}.txt").write_text("".join(chars))
    return str(tmp_path)


def test_realengine_runs_b200_cv_against_reference_cv(tmp_path):
    mod = _reference()
    from allpairs.apps import CompositionVectorApp
    from allpairs.realrun import RealEngine
    corpus = _write_corpus(tmp_path)
    ref = RealEngine(_config(), CompositionVectorApp(corpus, k=3)).run()
    got = RealEngine(_config(), mod.B200CompositionVectorApp(corpus, k=3)).run()
    assert got.ledger.full and ref.ledger.full
    assert set(got.results) == set(ref.results) and len(got.results) == 16 * 15 // 2
    for key, r in ref.results.items():
        g = got.results[key]
        assert g.value == pytest.approx(r.value, rel=1e-12, abs=1e-15), key
        assert g.match == r.match


def test_cv_dropin_slot_overflow_matches_reference(tmp_path):
    """A document with more distinct k-mers than the slot holds raises the
    reference's SlotOverflow from the B200 preprocess (apps.py:128-132)."""
    mod = _reference()
    from allpairs.errors import SlotOverflow
    corpus = _write_corpus(tmp_path, count=3, length=4000)
    app = mod.B200CompositionVectorApp(corpus, k=8, slot_size=16 + 16 * 64)
    from allpairs.apps import ItemData, Stage
    raw = ItemData(Stage.RAW_FILE, app.fetch_raw(app.path_for_key(0)))
    with pytest.raises(SlotOverflow):
        app.preprocess(0, app.parse(0, raw))
