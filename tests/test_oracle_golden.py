"""The oracle restatements against golden vectors generated from the reference itself
(tests/golden/make_golden.py) and against the reference tests' known answers."""

import json
import os

import numpy as np
import pytest

from oracle import cv as ocv
from oracle import pce as opce
from oracle import rng as orng
from oracle import scheduler as osched

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def test_mix64_golden():
    g = load("synthetic.json")
    for args, want in g["mix64"]:
        assert orng.mix64(*args) == want


def test_synthetic_values_bit_exact():
    for case in load("synthetic.json")["cases"]:
        n, seed = case["n"], case["seed"]
        got = [orng.synthetic_value(seed, i, j).hex() for i in range(n) for j in range(i + 1, n)]
        assert got == case["values"]


def test_mix64_vectorised_matches_scalar():
    keys = np.arange(50, dtype=np.uint64)
    v = orng.mix64_np(7, 0xC0403A3E, 3, keys)
    assert [int(x) for x in v] == [orng.mix64(7, 0xC0403A3E, 3, int(k)) for k in range(50)]


def test_leaves_golden():
    g = load("scheduler.json")
    for key, leaves in g["leaves"].items():
        n, lb = map(int, key.split("/"))
        assert [list(l) for l in osched.leaves(n, lb)] == leaves, key


def test_leaves_cover_pairs_exactly_once():
    for n in range(2, 41):
        for lb in (1, 3, 8):
            seen = set()
            for leaf in osched.leaves(n, lb):
                for p in osched.region_iter_pairs(*leaf):
                    assert p not in seen
                    seen.add(p)
            assert len(seen) == n * (n - 1) // 2


def test_pair_id_golden_and_counts():
    g = load("scheduler.json")
    for n, rows in g["pair_id"].items():
        for i, j, pid in rows:
            assert osched.pair_id(int(n), i, j) == pid
    for n, cnt in g["pair_count"].items():
        assert osched.region_pairs(0, int(n), 0, int(n)) == cnt
    assert g["pair_count"]["4980"] == 12_397_710 and g["pair_count"]["512"] == 130_816
    with pytest.raises(ValueError):
        osched.pair_id(5, 3, 3)


@pytest.mark.parametrize("name", ["five_docs_k2", "engine_seed0_k3", "acceptance_c04b05_k3", "mixed_k4"])
def test_cv_oracle_golden(name):
    g = load("cv.json")[name]
    k = g["k"]
    vecs = []
    for text, parsed_hex, pre_hex in zip(g["texts"], g["parsed"], g["preprocessed"]):
        parsed = ocv.parse(text, k)
        assert parsed.hex() == parsed_hex
        vec = ocv.preprocess(parsed)
        assert ocv.preprocessed_bytes(vec).hex() == pre_hex      # frequencies bit-exact
        vecs.append(vec)
    n = len(vecs)
    vals = [ocv.compare(vecs[i], vecs[j]) for i in range(n) for j in range(i + 1, n)]
    assert [v.hex() for v in vals] == g["values"]              # same summation order: bit-exact
    dense = [ocv.dense_cosine(g["texts"][i], g["texts"][j], k) for i in range(n) for j in range(i + 1, n)]
    np.testing.assert_allclose(vals, dense, atol=1e-9)         # test_apps.py:197-207


def test_cv_known_answers():
    a = ocv.preprocess(ocv.parse("ACGTACGTAAAC", 2))
    assert ocv.compare(a, a) == pytest.approx(1.0, abs=1e-9)
    x = ocv.preprocess(ocv.parse("AAAA", 2))
    y = ocv.preprocess(ocv.parse("TTTT", 2))
    assert ocv.compare(x, y) == 0.0
    with pytest.raises(ValueError):
        ocv.parse("AB", 3)


# -- PCE oracle: parity unpinned by the reference; pinned by known answers ----

def test_pce_shift_known_answer():
    x = opce.prnu_patterns(64, 64, 0, 1, 1, 3)[0]
    y = np.roll(x, (7, -11), axis=(0, 1))
    pce, peak, idx = opce.pce_from_plane(opce.correlation(opce.preprocess(y), opce.preprocess(x), 64, 64))
    assert divmod(idx, 64) == (7, (-11) % 64)
    assert pce > 1e3


def test_pce_matches_scipy_direct_correlation():
    scipy_fft = pytest.importorskip("scipy.fft")
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((2, 32, 32))
    c = opce.correlation(opce.preprocess(a), opce.preprocess(b), 32, 32)
    a0, b0 = a - a.mean(), b - b.mean()
    direct = np.zeros((32, 32))
    for s in range(32):
        for t in range(32):
            direct[s, t] = np.sum(np.roll(a0, (-s, -t), axis=(0, 1)) * b0)
    np.testing.assert_allclose(c, direct, atol=1e-10)
    c2 = scipy_fft.irfft2(scipy_fft.rfft2(a0) * np.conj(scipy_fft.rfft2(b0)), s=(32, 32))
    np.testing.assert_allclose(c, c2, atol=1e-10)


def test_pce_energy_excludes_11x11_window():
    c = np.zeros((32, 32))
    c[3, 4] = 10.0
    c[3 + 5, 4 + 5] = 1.0    # inside the window: excluded
    c[20, 20] = 2.0          # outside: counted
    pce, peak, idx = opce.pce_from_plane(c)
    assert idx == 3 * 32 + 4 and peak == 10.0
    assert pce == pytest.approx(100.0 / (4.0 / (32 * 32 - 121)))


def test_pce_camera_separation():
    x = opce.prnu_patterns(256, 256, 0, 4, 2, 5)
    s = [opce.preprocess(v) for v in x]
    same = opce.compare(s[0], s[2], 256, 256)
    diff = opce.compare(s[0], s[1], 256, 256)
    assert same > 60.0 > diff
