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


def test_trace_and_metrics_schema_match_reference(tmp_path):
    """Trace lines carry exactly the reference's TraceEvent keys (metrics.py:14-29)
    and the metrics document the RunMetrics.as_dict keys (metrics.py:139-155)."""
    from paper_2009_04755_b200 import metrics, perfmodel
    ev = [{"node": 0, "lane": "gpu0", "label": "compare", "start_ns": 10, "end_ns": 30, "i": 0, "j": 1,
           "count": 4},
          {"node": 0, "lane": "up0", "label": "preprocess", "start_ns": 0, "end_ns": 10, "i": 0, "j": -1,
           "count": 2}]
    path = tmp_path / "trace.jsonl"
    metrics.write_trace(str(path), ev)
    rows = metrics.read_trace(str(path))
    assert [set(r) for r in rows] == [{"node", "lane", "label", "start_ns", "end_ns", "i", "j"}] * 2
    stats = {"loads": 5, "pairs_done": 10, "hits": 20, "misses": 5, "evictions": 0, "h2d_bytes": 100,
             "peer_fetches": 0, "steals": 0}
    nm = metrics.node_metrics(0, stats, 2.0, 8, ev)
    assert nm["lane_busy"] == {"gpu0": 2e-8, "up0": 1e-8}
    assert set(nm) == {"node", "loads", "parses", "preprocesses", "comparisons", "io_bytes", "submitted",
                       "steals_local", "steals_remote", "steal_requests_failed", "messages_sent", "cache",
                       "remote_requests", "remote_hits_by_hop", "remote_failures", "remote_timeouts",
                       "load_counts", "lane_busy", "noslot_retries", "finish_time"}
    costs = perfmodel.StageCosts(t_preprocess=0.01, t_comparison=0.1)
    doc = metrics.run_metrics({"app": "pce"}, 5, [nm], 2.0, costs=costs)
    assert set(doc) == {"config", "n", "pairs", "makespan_s", "total_loads", "R", "t_min_s", "efficiency",
                        "efficiency_r_adjusted", "io_bytes", "io_rate_Bps", "wall_time_s", "cache", "remote",
                        "messages", "per_node"}
    assert doc["R"] == 1.0 and doc["pairs"] == 10
    assert doc["t_min_s"] == pytest.approx(5 * 0.01 + 10 * 0.1)
    assert doc["efficiency"] == pytest.approx(1.05 / 2.0)
    assert doc["cache"]["device"]["hits"] == 20
