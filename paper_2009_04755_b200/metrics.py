"""Trace and run-metrics emission in the reference's schemas (metrics.py:14-159).

* trace: newline-delimited JSON, one object per executed stage with integer-ns
  start/end (``TraceEvent``: node, lane, label, start_ns, end_ns, i, j), so the
  reference's ``read_trace`` and Gantt frontend read B200 runs.  The engine
  records one event per compare batch (lane ``gpu<d>``, label ``compare``, the
  batch's first pair) and per load / peer-fetch group (lane ``up<d>``, labels
  ``preprocess`` / ``fetch``, first key, j = -1); device timestamps from the
  start of the run.
* metrics: the ``RunMetrics.as_dict`` document -- config, n, pairs, makespan,
  R = loads / n (runner.py:41), T_min / efficiency (perfmodel.py:99-114),
  per-tier cache totals, remote (peer-tier) totals and ``NodeMetrics`` per rank.
"""

from __future__ import annotations

import json
from typing import Optional

from . import perfmodel


def write_trace(path: str, events: list[dict]) -> None:
    """metrics.py:write_trace -- compact JSON per line, the reference's keys only."""
    keys = ("node", "lane", "label", "start_ns", "end_ns", "i", "j")
    with open(path, "w") as fh:
        for ev in events:
            fh.write(json.dumps({k: ev[k] for k in keys}, separators=(",", ":")) + "\n")


def read_trace(path: str) -> list[dict]:
    with open(path) as fh:
        return [json.loads(line) for line in fh if line.strip()]


def node_metrics(node: int, stats: dict, seconds: float, device_slots: int, events: Optional[list] = None) -> dict:
    """NodeMetrics.as_dict (metrics.py:48-86) of one rank's engine run."""
    busy: dict = {}
    for ev in events or []:
        busy[ev["lane"]] = busy.get(ev["lane"], 0.0) + (ev["end_ns"] - ev["start_ns"]) / 1e9
    return {
        "node": node,
        "loads": stats.get("loads", 0),
        "parses": stats.get("loads", 0),
        "preprocesses": stats.get("loads", 0),
        "comparisons": stats.get("pairs_done", 0),
        "io_bytes": stats.get("h2d_bytes", 0),
        "submitted": stats.get("pairs_done", 0),
        "steals_local": 0,
        "steals_remote": stats.get("steals", 0),
        "steal_requests_failed": 0,
        "messages_sent": {},
        "cache": dict({"dev0": {"hits": stats.get("hits", 0), "misses": stats.get("misses", 0), "waits": 0,
                                "evictions": stats.get("evictions", 0), "occupancy": device_slots}},
                      **({"host": {"hits": stats["host_hits"], "misses": stats["host_misses"], "waits": 0,
                                   "evictions": stats["host_evictions"], "occupancy": stats["host_misses"]}}
                         if stats.get("host_hits", 0) + stats.get("host_misses", 0) else {})),
        "remote_requests": stats.get("peer_fetches", 0),
        "remote_hits_by_hop": {"1": stats.get("peer_fetches", 0)} if stats.get("peer_fetches", 0) else {},
        "remote_failures": 0,
        "remote_timeouts": 0,
        "load_counts": {},
        "lane_busy": busy,
        "noslot_retries": 0,
        "finish_time": seconds,
    }


def run_metrics(config: dict, n: int, per_node: list[dict], makespan: float,
                costs: Optional[perfmodel.StageCosts] = None, wall_time: float = 0.0) -> dict:
    """RunMetrics.as_dict (metrics.py:89-159) over the ranks' NodeMetrics."""
    total_loads = sum(nm["loads"] for nm in per_node)
    r = total_loads / n if n else 0.0
    t_min = perfmodel.t_min(n, costs) if costs is not None else None
    p = max(1, len(per_node))
    eff = perfmodel.efficiency(t_min, p, makespan) if t_min is not None and makespan > 0 else None
    eff_r = None
    if costs is not None and makespan > 0 and r >= 1.0:
        eff_r = (perfmodel.t_gpu(n, r, costs) / p) / makespan
    cache: dict = {}
    for nm in per_node:
        for tier, st in nm["cache"].items():
            agg = cache.setdefault("device" if tier.startswith("dev") else "host", {})
            for k, v in st.items():
                agg[k] = agg.get(k, 0) + v
    hits_by_hop: dict = {}
    for nm in per_node:
        for hop, c in nm["remote_hits_by_hop"].items():
            hits_by_hop[hop] = hits_by_hop.get(hop, 0) + c
    io_bytes = sum(nm["io_bytes"] for nm in per_node)
    return {
        "config": config,
        "n": n,
        "pairs": perfmodel.pair_count(n),
        "makespan_s": makespan,
        "total_loads": total_loads,
        "R": r,
        "t_min_s": t_min,
        "efficiency": eff,
        "efficiency_r_adjusted": eff_r,
        "io_bytes": io_bytes,
        "io_rate_Bps": io_bytes / makespan if makespan > 0 else 0.0,
        "wall_time_s": wall_time,
        "cache": cache,
        "remote": {"requests": sum(nm["remote_requests"] for nm in per_node), "failures": 0, "timeouts": 0,
                   "hits_by_hop": hits_by_hop},
        "messages": {},
        "per_node": per_node,
    }


def write_metrics(path: str, doc: dict) -> None:
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=2, sort_keys=True)
        fh.write("\n")
