"""Public all-pairs API: run every pair of an Application's items on B200s.

The runtime under it is the C++ engine of librocket (csrc/engine.cpp): the
quadtree leaves of the pair triangle (scheduler.py:20-117) are this rank's
work; items are acquired per leaf in ascending key order through the device
slot tier (slotcache.py:159-282), loaded on a miss from the pinned host tier
(H2D + device preprocess, engine.py:436-508) and compared in batches by the
app's fused kernels.  Results land in the packed upper triangle indexed by
PairLedger.pair_id (scheduler.py:228-231).

Multi-GPU: one process per GPU (torchrun).  Each rank starts on a contiguous,
pair-balanced block of the depth-first leaves and takes it in chunks from a
work-queue word in its device memory; a rank that runs dry steals the back
half of the fullest peer's remaining range with system-scope atomics over
NVLink (hierarchical stealing, engine.py:274-309).  Items live on their home
GPU (k mod world) and are fetched peer-to-peer (peer tier).  The disjoint
result triangles are combined on rank 0 with one NCCL reduce -- the only
collective, as in the reference's completion gather to node 0
(engine.py:550-577).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import perfmodel
from .apps import B200Application, ItemData, PairResult, Stage, match_from_flag
from .device import DeviceEngine


@dataclass
class RunResult:
    n: int
    values: np.ndarray                 # float64 [C(n,2)] in pair_id order
    flags: np.ndarray                  # uint8   [C(n,2)] wire-encoded match
    stats: dict = field(default_factory=dict)
    seconds: float = 0.0
    trace: list = field(default_factory=list)      # metrics.py TraceEvent dicts (when tracing)
    node: dict = field(default_factory=dict)       # this rank's NodeMetrics dict
    ledger: dict = field(default_factory=dict)     # exactly-once ledger of the job (rank 0): completed, full

    @property
    def pairs(self) -> int:
        return self.n * (self.n - 1) // 2

    @property
    def r_factor(self) -> float:
        """R = loads / n (runner.py:41)."""
        return self.stats.get("loads", 0) / self.n if self.n else 0.0

    @property
    def device_hit_rate(self) -> float:
        h, m = self.stats.get("hits", 0), self.stats.get("misses", 0)
        return h / (h + m) if h + m else 0.0

    def result(self, i: int, j: int) -> PairResult:
        pid = i * (2 * self.n - i - 1) // 2 + (j - i - 1)
        return PairResult(i, j, float(self.values[pid]), match_from_flag(int(self.flags[pid])))

    def results(self) -> dict:
        out = {}
        pid = 0
        for i in range(self.n):
            for j in range(i + 1, self.n):
                out[(i, j)] = PairResult(i, j, float(self.values[pid]), match_from_flag(int(self.flags[pid])))
                pid += 1
        return out

    def efficiency(self, costs: perfmodel.StageCosts, p: int = 1) -> float:
        """(T_min / p) / T with T_min from measured single-GPU stage costs (perfmodel.py:99-114)."""
        return perfmodel.efficiency(perfmodel.t_min(self.n, costs), p, self.seconds)


def rank_leaves(n: int, leaf_block: int, rank: int = 0, world: int = 1) -> list:
    """This rank's depth-first quadtree leaves (r0, r1, c0, c1), as the C++ engine schedules them."""
    import ctypes as C
    from ._lib import lib
    cnt = lib.rk_leaves(n, leaf_block, rank, world, None, 0)
    if cnt < 0:
        raise ValueError(f"bad leaf_block/rank/world ({leaf_block}, {rank}, {world})")
    buf = (C.c_int32 * max(1, 4 * cnt))()
    lib.rk_leaves(n, leaf_block, rank, world, buf, cnt)
    return [tuple(buf[4 * k:4 * k + 4]) for k in range(cnt)]


def gather_triangle(values: torch.Tensor, flags: Optional[torch.Tensor] = None, dst: int = 0) -> None:
    """Combine the ranks' disjoint result triangles onto ``dst`` (NCCL on GPUs, gloo on CPU).

    Every pair id is written by exactly one rank and is zero elsewhere, so a
    sum-reduce is an exact gather -- the single collective of a multi-GPU job.
    """
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return
    dist.reduce(values, dst=dst, op=dist.ReduceOp.SUM)
    if flags is not None:
        dist.reduce(flags, dst=dst, op=dist.ReduceOp.SUM)


class AllPairsEngine:
    """All pairs of ``app``'s items on one GPU (this rank's share of a multi-GPU job)."""

    def __init__(self, app: B200Application, *, leaf_block: int = 16, device_slots: Optional[int] = None,
                 rank: int = 0, world: int = 1, peer_tier: bool = True, steal: bool = True,
                 steal_chunk: int = 0, trace_events: int = 0, host_slots: int = 0):
        self.app = app
        self.rank = rank
        self.world = world
        torch.cuda.set_device(app.device)
        slots = device_slots if device_slots is not None else app.n
        # NCC: with every item resident (slots >= n) each rank takes its round-robin
        # share of the Gram tiles; with fewer slots the Gram runs over home
        # sub-blocks and peer-fetched partners (the peer tier)
        ncc_resident = app.kind == 3 and slots >= app.n
        self._eng = DeviceEngine(app.app_params(), leaf_block=leaf_block, device_slots=max(2, slots),
                                 rank=rank, world=world, device=app.device,
                                 peer_tier=peer_tier and world > 1 and app.kind != 0 and not ncc_resident,
                                 steal=steal and world > 1 and app.kind != 3, steal_chunk=steal_chunk,
                                 host_slots=host_slots)
        self._peers_connected = False
        self._slots = max(2, slots)
        if trace_events:
            self._eng.set_trace(trace_events)
        self._trace_on = bool(trace_events)
        self._out = torch.empty(app.n * (app.n - 1) // 2, dtype=torch.float64, device=f"cuda:{app.device}")
        self._flags = torch.empty_like(self._out, dtype=torch.uint8)

    def close(self) -> None:
        self._eng.close()

    def load_items(self, pin: bool = True) -> torch.Tensor:
        """Run fetch_raw + parse for every key into one host buffer at the parsed stride."""
        stride = self.app.parsed_bytes()
        host = torch.empty(self.app.n * stride, dtype=torch.uint8, pin_memory=pin)
        view = host.numpy().reshape(self.app.n, stride)
        for key in range(self.app.n):
            raw = ItemData(Stage.RAW_FILE, self.app.fetch_raw(self.app.path_for_key(key)))
            view[key] = self.app.parsed_array(self.app.parse(key, raw))
        return host

    def run(self, host_items: Optional[torch.Tensor] = None, device_items: Optional[torch.Tensor] = None,
            gather: bool = True, home_chunks=None, chunk: int = 256) -> RunResult:
        """One full all-pairs job; returns the packed triangle (on rank 0 when world > 1).

        Items come from ``host_items`` / ``device_items`` (all n at the parsed
        stride), from the app's own fetch_raw + parse, or -- with the peer tier, for
        jobs whose items exist on no single GPU or host (C3) -- from
        ``home_chunks(m0, count)``, which returns this rank's home items m0 ..
        m0 + count - 1 (keys rank + m * world) as one host or device tensor at the
        parsed stride; they are preprocessed ``chunk`` at a time into the home region.
        """
        if home_chunks is not None and not self._eng.peer_tier:
            raise ValueError("home_chunks needs the peer tier (world > 1)")
        if host_items is None and device_items is None and home_chunks is None and self.app.kind != 0:
            host_items = self.load_items()
        self._out.zero_()
        self._flags.zero_()
        self._eng.reset_stats()
        t0 = time.perf_counter()
        stride = self.app.parsed_bytes()
        # world > 1: the ranks share rank 0's exactly-once ledger over IPC (and, with the
        # peer tier / stealing, each other's home regions and queue words)
        shared = self.world > 1
        if home_chunks is not None:
            n_home = len(range(self.rank, self.app.n, self.world))
            for m0 in range(0, n_home, chunk):
                cnt = min(chunk, n_home - m0)
                part = home_chunks(m0, cnt)
                kw = {"device_items": part} if part.is_cuda else {"host_items": part}
                self._eng.load_home_range(m0, cnt, parsed_stride=stride, **kw)
        elif self._eng.peer_tier:
            # home items first (k % world == rank), then the IPC-mapped peer homes
            # home item m = key rank + m*world: a strided view of the full item array
            off = self.rank * stride

            class _At:
                def __init__(self, t):
                    self.t = t

                def data_ptr(self):
                    return self.t.data_ptr() + off

            self._eng.load_home(host_items=None if host_items is None else _At(host_items),
                                device_items=None if device_items is None else _At(device_items),
                                parsed_stride=self.world * stride)
        if shared:
            import torch.distributed as dist
            if not self._peers_connected:
                self._eng.connect_peers()
                self._peers_connected = True
            if self._eng.steal:
                self._eng.queue_reset()
            self._eng.ledger_reset()   # rank 0 clears the job's ledger
            dist.barrier()   # home regions complete, queue words and ledger reset before anyone uses them
        self._eng.run(self._out, self._flags, host_items=host_items, device_items=device_items,
                      parsed_stride=stride)
        if shared:
            dist.barrier()   # peers are done reading our home region and queue word, all marks landed
        ledger = self._eng.check_ledger() if self.rank == 0 else {}   # AssertionError on a duplicate
        if self.world > 1 and gather:
            gather_triangle(self._out, self._flags)
        values = self._out.cpu().numpy()
        flags = self._flags.cpu().numpy()
        seconds = time.perf_counter() - t0
        stats = self._eng.stats()
        events = self._eng.trace(node=self.rank) if self._trace_on else []
        from .metrics import node_metrics
        return RunResult(self.app.n, values, flags, stats, seconds, events,
                         node_metrics(self.rank, stats, seconds, self._slots, events), ledger)

    def metrics(self, result: RunResult, config: Optional[dict] = None,
                costs: Optional[perfmodel.StageCosts] = None) -> dict:
        """RunMetrics document (metrics.py:89-159) of a run, NodeMetrics of every rank."""
        from .metrics import run_metrics
        per_node = [result.node]
        makespan = result.seconds
        if self.world > 1:
            import torch.distributed as dist
            gathered = [None] * self.world
            dist.all_gather_object(gathered, (result.node, result.seconds))
            per_node = [g[0] for g in gathered]
            makespan = max(g[1] for g in gathered)
        cfg = config if config is not None else {"app": self.app.name, "n": self.app.n, "world": self.world}
        return run_metrics(cfg, self.app.n, per_node, makespan, costs=costs, wall_time=result.seconds)


def run_allpairs(app: B200Application, **kw) -> RunResult:
    """Convenience wrapper: build an engine, run once, release it."""
    eng = AllPairsEngine(app, **kw)
    try:
        return eng.run()
    finally:
        eng.close()
