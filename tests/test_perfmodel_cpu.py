"""perfmodel restatement vs the reference's values (golden perfmodel.json)."""

import json
import math
import os

import pytest

from paper_2009_04755_b200 import perfmodel

GOLD = os.path.join(os.path.dirname(__file__), "golden", "perfmodel.json")


def test_report_matches_reference():
    g = json.load(open(GOLD))
    costs = perfmodel.StageCosts(**g["costs"])
    rep = perfmodel.report(g["n"], g["R"], costs, p=g["p"], t_measured=g["t_measured"])
    for key, want in g["report"].items():
        assert rep[key] == pytest.approx(want, rel=1e-12), key


def test_model_validation():
    with pytest.raises(ValueError):
        perfmodel.StageCosts(t_parse=-1.0)
    with pytest.raises(ValueError):
        perfmodel.t_gpu(10, 0.5, perfmodel.StageCosts())
    with pytest.raises(ValueError):
        perfmodel.efficiency(1.0, 0, 1.0)
    assert perfmodel.t_io(10, 1.0, perfmodel.StageCosts(mean_file_bytes=1.0)) == 0.0
    assert perfmodel.pair_count(4096) == 8_386_560
    assert math.isclose(perfmodel.efficiency(10.0, 2, 5.0), 1.0)
