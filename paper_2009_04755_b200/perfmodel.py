"""Rocket performance model (paper Eqs. 1-5) and run metrics.

Restates /root/reference/pkg/src/allpairs/perfmodel.py:79-131 and the metric
formulas of runner.assemble_metrics (runner.py:36-66): the modeled lower bound
T_min = n*t_pre + C(n,2)*t_cmp (perfect reuse, free I/O), the system efficiency
(T_min / p) / T, and the reuse factor R = loads / n.  The B200 engine feeds it
with t_preprocess / t_comparison measured in isolation on one GPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


def pair_count(n: int) -> int:
    if n < 0:
        raise ValueError(f"item count must be non-negative, got {n}")
    return n * (n - 1) // 2


@dataclass(frozen=True)
class StageCosts:
    t_parse: float = 0.0
    t_preprocess: float = 0.0
    t_comparison: float = 0.0
    t_postprocess: float = 0.0
    mean_file_bytes: float = 0.0
    io_bandwidth: float = math.inf

    def __post_init__(self) -> None:
        for name in ("t_parse", "t_preprocess", "t_comparison", "t_postprocess", "mean_file_bytes"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be non-negative")
        if self.io_bandwidth <= 0:
            raise ValueError("io_bandwidth must be positive")


def _check(n: int, r_factor: float) -> None:
    if n < 0:
        raise ValueError("item count must be non-negative")
    if r_factor < 1.0 and n > 0:
        raise ValueError("reuse factor R must be >= 1")


def t_gpu(n: int, r_factor: float, costs: StageCosts) -> float:
    _check(n, r_factor)
    return r_factor * n * costs.t_preprocess + pair_count(n) * costs.t_comparison


def t_cpu(n: int, r_factor: float, costs: StageCosts) -> float:
    _check(n, r_factor)
    return r_factor * n * costs.t_parse + pair_count(n) * costs.t_postprocess


def t_io(n: int, r_factor: float, costs: StageCosts) -> float:
    _check(n, r_factor)
    if math.isinf(costs.io_bandwidth):
        return 0.0
    return r_factor * n * costs.mean_file_bytes / costs.io_bandwidth


def t_min(n: int, costs: StageCosts) -> float:
    return t_gpu(n, 1.0, costs)


def efficiency(t_lower_bound: float, p: int, t_measured: float) -> float:
    if p < 1:
        raise ValueError("node count must be >= 1")
    if t_measured <= 0:
        raise ValueError("measured time must be positive")
    return (t_lower_bound / p) / t_measured


def report(n: int, r_factor: float, costs: StageCosts, p: int = 1, t_measured: float | None = None) -> dict:
    out = {"n": n, "R": r_factor, "T_gpu_s": t_gpu(n, r_factor, costs), "T_cpu_s": t_cpu(n, r_factor, costs),
           "T_io_s": t_io(n, r_factor, costs), "T_min_s": t_min(n, costs)}
    if t_measured is not None:
        out["efficiency"] = efficiency(t_min(n, costs), p, t_measured)
    return out
