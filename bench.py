#!/usr/bin/env python
"""All-pairs PRNU PCE benchmark (BASELINE.json configs[1]): pairs/sec on B200.

Workload (`config.workload`): N=4,096 synthetic PRNU-like patterns of
1024x1024 fp32, all C(N,2) = 8,386,560 pairs through the PCE compare.  One
step = one full all-pairs job: preprocess every item from its HBM-resident
parsed pattern into the device slot tier, then every quadtree leaf of this
rank's share through the fused compare kernels.

  value   pairs/s over all ranks, inputs resident in HBM at the start of the
          timed region, timed with CUDA events on the engine stream, max over ranks
  e2e     the same job through the public engine API from pinned HOST patterns,
          H2D inside the timed region, plus the D2H of the packed result triangle
  roofline  dominant kernel = one PCE compare launch (pce_cluster; pce2k_pair at 2048^2),
          per-launch time from sampled CUDA events on the engine stream
  parity  sampled pair ids of the timed job recomputed by the float64 oracle
  perf_model  the Rocket efficiency (T_min/p)/T (perfmodel.py:99-114) with t_pre and
          t_cmp measured in an isolated single-GPU pass before the timed steps
  cpu_baseline  the float64 oracle (oracle/pce.py) on a bounded pair sample

Other workloads: `--items 16384 --side 2048` is BASELINE configs[2] (C3: 256 GiB
of patterns, more than one GPU's HBM): every rank generates and preprocesses
only its home items (k mod N) and fetches the others from their home GPU over
NVLink; it needs N >= 2.  `--items 128 --side 256` is configs[0] (C1).
`--app gmm` is configs[3], `--app cv` configs[4].

`--gpus N` without torchrun relaunches itself under torch.distributed.run with N
ranks; under torchrun, WORLD_SIZE must equal --gpus.  NCCL is used once per job,
to reduce the disjoint result triangles to rank 0.

`python bench.py --impl reference` times the reference-side CPU path (the
float64 oracle port -- the reference itself has no PCE kernel) on the same
workload, config and metric, one bounded pair sample per step.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
PCE_RTOL = 1e-4


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--items", type=int, default=0, help="items (default: the app's BASELINE config)")
    ap.add_argument("--side", type=int, default=1024, help="pattern side (default 1024)")
    ap.add_argument("--leaf", type=int, default=8)
    ap.add_argument("--cameras", type=int, default=0, help="PRNU cameras (default 64; 256 at C3)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--slots", type=int, default=0, help="home-only mode: device cache slots per GPU")
    ap.add_argument("--home-only", action="store_true",
                    help="force the C3 placement (items generated on their home GPU only) at any size")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    ap.add_argument("--parity-samples", type=int, default=32)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-steal", action="store_true", help="N > 1: static leaf shares, no cross-GPU stealing")
    ap.add_argument("--steal-chunk", type=int, default=0, help="N > 1: leaves per work-queue grab (0: one batch)")
    ap.add_argument("--trace-dir", default="",
                    help="pce: after the timed steps, run one traced step and write the reference-schema "
                         "trace (JSONL) and run-metrics document of each rank here")
    ap.add_argument("--app", default="pce", choices=["pce", "ncc", "gmm", "cv"],
                    help="pce: configs[1] (default); ncc: the zero-lag NCC Gram of the same items (C3-Gram with "
                         "--items 16384 --side 2048); gmm: configs[3]; cv: configs[4]")
    ap.add_argument("--angles", type=int, default=36, help="gmm: rotation grid K")
    ap.add_argument("--mean-nnz", type=float, default=5e5, help="cv: mean tokens per item")
    args = ap.parse_args(argv)
    if args.items <= 0:
        args.items = {"pce": 4096, "ncc": 4096, "gmm": 1000, "cv": 2500}[args.app]
    if args.cameras <= 0:
        args.cameras = 256 if args.items >= 16384 else 64
    return args


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return dict(PEAKS_FALLBACK), "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# Workload description shared by both arms (identical config dicts)

def workload(args, world):
    n = args.items
    pairs_total = n * (n - 1) // 2
    metric = "pairs/sec (whole box)"
    if args.app in ("pce", "ncc"):
        side = args.side
        cfg_name = {(128, 256): " (BASELINE configs[0])", (4096, 1024): " (BASELINE configs[1])",
                    (16384, 2048): " (BASELINE configs[2])"}.get((n, side), "")
        name = f"PRNU PCE all-pairs, N={n} patterns of {side}x{side} fp32{cfg_name}"
        if args.app == "ncc":
            name = (f"zero-lag NCC all-pairs as a tcgen05 TF32 Gram, N={n} patterns of {side}x{side} fp32"
                    f"{cfg_name.replace(')', ', C3-Gram of SURVEY 8(d))') if cfg_name else ''}")
        pat = n * side * side * 4
        cfg = {"workload": name, "n": n, "side": side, "pairs": pairs_total, "leaf_block": args.leaf,
               "cameras": args.cameras, "parallelism": f"pairs{world}",
               "l2": f"inputs ({2 * pat / 2**30:.1f} GiB patterns + spectra) >> L2 (126 MB): no flush needed"}
        if home_only(args):
            cfg["placement"] = "home-only: item k generated + preprocessed on GPU k mod N, peers fetch over NVLink"
        return metric, cfg, "tf32" if args.app == "ncc" else "fp32"
    if args.app == "gmm":
        name = (f"particle fusion (GMM/Bhattacharyya), N={n} particles of ~300 localizations, "
                f"K={args.angles} rotations (BASELINE configs[3])")
        cfg = {"workload": name, "n": n, "pairs": pairs_total, "angles": args.angles, "leaf_block": 16,
               "parallelism": f"pairs{world}", "l2": "items 4.6 MB, L2-resident by design (compute-bound)"}
        return metric, cfg, "fp32"
    name = (f"composition-vector cosine, N={n} variable-length items, nnz lognormal in [1e5, 1.8e6] "
            f"(mean {args.mean_nnz:.0f}) (BASELINE configs[4])")
    cfg = {"workload": name, "n": n, "pairs": pairs_total, "mean_nnz": args.mean_nnz, "leaf_block": 16,
           "parallelism": f"pairs{world}", "l2": f"items ~{16 * n * args.mean_nnz / 2**30:.0f} GiB >> L2"}
    return metric, cfg, "fp64"


def home_only(args) -> bool:
    """C3-sized PCE jobs: patterns + spectra of all items do not fit one GPU."""
    return args.app in ("pce", "ncc") and (getattr(args, "home_only", False) or
                                           2 * args.items * args.side * args.side * 4 > (120 << 30))


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None
        self.error = None

    def _query_once(self):
        try:
            r = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
            parts = [p.strip() for p in r.stdout.strip().split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)
        except Exception as exc:  # pragma: no cover - box without nvidia-smi
            self.error = str(exc)[:100]

    def start(self):
        self._query_once()   # one sample at the start of the timed region
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception as exc:
            self.proc = None
            self.error = str(exc)[:100]
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self) -> dict:
        self._query_once()   # and one at its end, so short regions still have samples
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)
        sm, smax, reasons, loaded = [], None, set(), []
        for r in self.rows:
            try:
                mhz = float(r[1])
                smax = float(r[2])
                pw = float(r[3])
            except ValueError:
                continue
            sm.append(mhz)
            if pw > 300.0:
                loaded.append(mhz)
            for name, val in zip(self.NAMES, r[5:9]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "error": self.error or "no nvidia-smi samples"}
        src = sorted(loaded) if loaded else sorted(sm)
        return {"sm_mhz": src[len(src) // 2], "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "samples_under_load": len(loaded)}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the float64 oracle port (TEST-INFRASTRUCTURE code,
# used only as the timed reference arm and the parity checker, never as the
# product path).  Workers are pinned one per host core; each owns a block of
# item keys whose items are generated and preprocessed when the pool starts
# (the load stage, amortised over the whole job); a step is a fixed number of
# compares per worker, so ms_per_step is measured, not extrapolated.

_W = {}


def _init_worker(spec, blocks, barrier):
    """Pool initializer: pin this worker to one host core, then generate and
    preprocess its block of items (the load stage, untimed)."""
    import multiprocessing as mp
    ident = mp.current_process()._identity
    wid = ((ident[0] - 1) if ident else 0) % len(blocks)
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else [0]
    try:
        os.sched_setaffinity(0, {cores[wid % len(cores)]})
    except Exception:
        pass
    _W.clear()
    _W.update(spec=spec, barrier=barrier, cursor=0)
    keys = blocks[wid]
    app = spec["app"]
    if app == "pce":
        from oracle import pce as opce
        side = spec["side"]
        items = {k: opce.preprocess(opce.prnu_patterns(side, side, k, 1, spec["cameras"], spec["seed"])[0])
                 for k in keys}
    elif app == "ncc":
        from oracle import ncc as oncc
        from oracle import pce as opce
        side = spec["side"]
        items = {k: oncc.preprocess(opce.prnu_patterns(side, side, k, 1, spec["cameras"], spec["seed"])[0])
                 for k in keys}
    elif app == "gmm":
        from paper_2009_04755_b200.synthdata import particle
        items = {k: particle(k, spec["seed"]) for k in keys}
    else:
        from oracle import cv as ocv
        from paper_2009_04755_b200.synthdata import cv_parsed_host
        items = {q: ocv.preprocess(b) for q, b in enumerate(cv_parsed_host(keys, spec["seed"] + wid))}
    ks = sorted(items)
    _W["items"] = items
    _W["pairs"] = [(a, b) for ai, a in enumerate(ks) for b in ks[ai + 1:]]


def _worker_step(count):
    """`count` compares from this worker's pair list (cyclic); returns busy seconds.
    The barrier makes every one of the pool's workers take exactly one task."""
    _W["barrier"].wait()
    spec = _W["spec"]
    pairs, items = _W["pairs"], _W["items"]
    t0 = time.perf_counter()
    for _ in range(count):
        i, j = pairs[_W["cursor"] % len(pairs)]
        _W["cursor"] += 1
        if spec["app"] == "pce":
            from oracle import pce as opce
            opce.compare(items[i], items[j], spec["side"], spec["side"])
        elif spec["app"] == "ncc":
            from oracle import ncc as oncc
            oncc.compare(items[i], items[j])
        elif spec["app"] == "gmm":
            from oracle import gmm as ogmm
            ogmm.compare(items[i], items[j], spec["angles"])
        else:
            from oracle import cv as ocv
            ocv.compare(items[i], items[j])
    return time.perf_counter() - t0


class CpuArm:
    """The oracle port on every host core (one pinned process per core)."""

    @staticmethod
    def host_cores() -> int:
        return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)

    def __init__(self, args, step_seconds: float):
        import multiprocessing as mp
        import random
        self.args = args
        self.cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
        spec = {"app": args.app, "side": args.side, "cameras": args.cameras, "seed": args.seed,
                "angles": args.angles, "mean_nnz": args.mean_nnz}
        rng = random.Random(args.seed)
        n = args.items
        blocks = []
        if args.app == "cv":
            from paper_2009_04755_b200.synthdata import cv_nnz
            sizes = cv_nnz(n, args.mean_nnz, args.seed)
            self.block = 6
            for _ in range(self.cores):
                b = rng.randrange(0, max(1, n - self.block))
                blocks.append([int(x) for x in sizes[b:b + self.block]])
        else:
            self.block = 12 if args.app in ("pce", "ncc") else 24
            for _ in range(self.cores):
                b = rng.randrange(0, max(1, n - self.block))
                blocks.append(list(range(b, min(n, b + self.block))))
        ctx = mp.get_context("spawn")
        t0 = time.perf_counter()
        self.pool = ctx.Pool(self.cores, initializer=_init_worker, initargs=(spec, blocks, ctx.Barrier(self.cores)))
        # calibrate the per-step compare count so a step takes ~step_seconds (the first
        # call also waits for every worker's initializer)
        self.pool.map(_worker_step, [1] * self.cores, chunksize=1)
        self.setup_s = time.perf_counter() - t0
        busy = max(self.pool.map(_worker_step, [2] * self.cores, chunksize=1)) / 2
        self.per_worker = max(1, int(step_seconds / max(busy, 1e-4)))
        wall = self.step()[1]            # refine once against a whole step's wall time
        self.per_worker = max(1, int(self.per_worker * step_seconds / max(wall, 1e-4)))

    def step(self):
        t0 = time.perf_counter()
        busy = self.pool.map(_worker_step, [self.per_worker] * self.cores, chunksize=1)
        wall = time.perf_counter() - t0
        return self.per_worker * self.cores, wall, max(busy)

    def describe(self, what):
        return (f"{self.per_worker} {what} per worker per step on {self.cores} pinned worker processes "
                f"(one per host core; {self.block}-item key blocks generated + preprocessed at pool start, "
                f"{self.setup_s:.1f}s, untimed load stage); value = compares / wall time of the timed steps")

    def close(self):
        self.pool.terminate()


def cpu_what(args):
    if args.app == "pce":
        return f"{args.side}x{args.side} PCE compares (numpy float64 irfft2 + peak/energy)"
    if args.app == "ncc":
        return f"{args.side}x{args.side} zero-lag NCC compares (numpy float64 dot of normalised items)"
    if args.app == "gmm":
        return f"particle-pair GMM costs (K={args.angles}, numpy float64)"
    return "composition-vector cosines (pure-Python merge of the reference's compare)"


def cpu_baseline(args, budget_s):
    """One bounded CPU measurement for the GPU arm's `cpu_baseline` key (rank 0, N = 1)."""
    arm = CpuArm(args, step_seconds=max(1.0, budget_s / 3))
    done, wall = 0, 0.0
    for _ in range(3):
        p, w, _ = arm.step()
        done, wall = done + p, wall + w
    arm.close()
    return {"value": done / wall, "unit": "pairs/s", "cores": arm.cores, "kind": "port",
            "sample": arm.describe(cpu_what(args)) + f"; 3 steps, {done} compares in {wall:.1f}s"}


def realengine_sample(args, n_items=16, lanes=1):
    """BASELINE.md section 3's harness: the reference's own RealEngine
    (realrun.py:28-176, staged in oracle/_ref by oracle/Makefile) running a float64
    numpy Application (oracle/pce.py, or oracle/ncc.py) over n_items of this
    workload: real mode, one node, `lanes` device lanes, cpu_width = host cores,
    stage_cost = 0.  Returns pairs/s of the whole run (load stage included)."""
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "allpairs")):
        return {"unavailable": "oracle/_ref not staged (make -C oracle where /root/reference exists)"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import struct

    import numpy as np
    from allpairs.apps import Application, ItemData, PairResult, Stage
    from allpairs.config import NodeShape, RunConfig
    from allpairs.realrun import RealEngine

    from oracle import ncc as oncc
    from oracle import pce as opce
    side, ncc = args.side, args.app == "ncc"

    class NumpyApp(Application):
        name = "numpy-" + ("ncc" if ncc else "pce")

        def path_for_key(self, key):
            return f"prnu/{key:06d}.f32"

        def fetch_raw(self, path):
            return opce.prnu_patterns(side, side, int(path[5:11]), 1, args.cameras, args.seed)[0].tobytes()

        def parse(self, key, raw):
            return ItemData(Stage.PARSED, raw.payload)

        def preprocess(self, key, parsed):
            x = np.frombuffer(parsed.payload, dtype=np.float32).reshape(side, side)
            y = oncc.preprocess(x) if ncc else opce.preprocess(x)
            return ItemData(Stage.PREPROCESSED, y.tobytes(), sim_bytes=self.slot_size)

        def compare(self, left, right):
            (i, a), (j, b) = left, right
            if ncc:
                v = oncc.compare(np.frombuffer(a.payload), np.frombuffer(b.payload))
            else:
                sa = np.frombuffer(a.payload, dtype=np.complex128).reshape(side, side // 2 + 1)
                sb = np.frombuffer(b.payload, dtype=np.complex128).reshape(side, side // 2 + 1)
                v = opce.compare(sa, sb, side, side)
            return struct.pack("<d", v)

        def postprocess(self, pair, raw):
            (v,) = struct.unpack("<d", raw)
            return PairResult(pair[0], pair[1], v, match=v >= (0.02 if ncc else 60.0))

        def stage_cost(self, stage, i, j=None):
            return 0.0

    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    app = NumpyApp(n_items, slot_size=side * (side // 2 + 1) * 16)
    cfg = RunConfig(app={"kind": app.name}, mode="real", leaf_block=args.leaf,
                    nodes=[NodeShape(device_speeds=[1.0] * lanes, device_slots=n_items, host_slots=n_items,
                                     cpu_width=cores)])
    t0 = time.perf_counter()
    master = RealEngine(cfg, app, run_timeout=600).run()
    wall = time.perf_counter() - t0
    pairs = n_items * (n_items - 1) // 2
    return {"value": pairs / wall, "unit": "pairs/s", "pairs": pairs, "seconds": wall, "device_lanes": lanes,
            "cpu_width": cores, "ledger_full": bool(master.ledger.full),
            "what": f"reference RealEngine (oracle/_ref) + float64 numpy app, {n_items} items of {side}^2, "
                    "real mode, one node, load stage included"}


def reference_arm(args, rank):
    """`--impl reference`: the reference-side CPU path, timed like our arm (W + K steps)."""
    if rank != 0:
        return 0
    metric, cfg, _ = workload(args, args.gpus)
    arm = CpuArm(args, step_seconds=max(0.5, min(2.0, args.cpu_seconds / 8)))
    for _ in range(args.warmup):
        arm.step()
    done, wall, step_ms = 0, 0.0, []
    for _ in range(args.steps):
        p, w, _ = arm.step()
        done += p
        wall += w
        step_ms.append(w * 1e3)
    arm.close()
    value = done / wall
    harness = None
    if args.app in ("pce", "ncc") and not args.no_cpu:
        # the reference's own engine on a bounded sample, one and
        # all device lanes; a reported figure beside the value, which is the (faster) port
        n_re = 16 if args.side >= 1024 else min(args.items, 32)
        try:
            harness = [realengine_sample(args, n_re, lanes) for lanes in (1, CpuArm.host_cores())]
        except Exception as exc:   # the arm's value stands without it
            harness = {"error": str(exc)[:200]}
    line = {"metric": metric, "value": value, "unit": "pairs/s", "impl": "reference", "n_gpus": args.gpus,
            "host_only": True, "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg, "extrapolated": False,
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": arm.cores, "kind": "port",
                             "sample": arm.describe(cpu_what(args)),
                             "pairs_per_step": done // max(1, args.steps), "step_ms": step_ms},
            "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "realengine": harness}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm helpers

class _At:   # pointer view at a byte offset (the C ABI only needs data_ptr())
    def __init__(self, t, off):
        self.t, self.off = t, off

    def data_ptr(self):
        return self.t.data_ptr() + self.off


def pce_parity(args, n, side, out, flags, items=None, gen_stream=None):
    """Recompute sampled pair ids of the finished job with the float64 oracle.

    Pairs are drawn among the ids this rank computed (flags != 0); items come
    from the resident device patterns or are regenerated (home-only mode)."""
    import numpy as np
    import torch

    from oracle import pce as opce
    from oracle import scheduler as osch
    from paper_2009_04755_b200 import device
    f = flags.cpu().numpy()
    mine = np.flatnonzero(f)
    if len(mine) == 0:
        return {"sampled": 0, "max_rel_err": None, "tolerance": PCE_RTOL, "pass": False}
    rng = np.random.default_rng(args.seed + 99)
    pids = sorted(int(x) for x in rng.choice(mine, size=min(args.parity_samples, len(mine)), replace=False))
    pairs = [osch.pair_from_id(n, p) for p in pids]
    keys = sorted({k for p in pairs for k in p})
    ss = side * side
    host = {}
    if items is not None:
        for k in keys:
            host[k] = items[k * ss:(k + 1) * ss].cpu().numpy().reshape(side, side)
    else:
        buf = torch.empty(ss, dtype=torch.float32, device="cuda")
        for k in keys:
            device.synth_prnu(side, side, k, 1, args.cameras, args.seed, buf)
            host[k] = buf.cpu().numpy().reshape(side, side)
    kidx = {k: q for q, k in enumerate(keys)}
    stack = np.stack([host[k] for k in keys])
    want = opce.pairs_batched(stack, [(kidx[i], kidx[j]) for i, j in pairs], batch=4 if side >= 2048 else 16)
    got = out.cpu().numpy()[pids]
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-300)
    fl = f[pids]
    flags_ok = bool(np.all(np.where(want >= 60.0, fl == 3, fl == 1)))
    return {"sampled": len(pids), "max_rel_err": float(rel.max()), "tolerance": PCE_RTOL,
            "flags_match": flags_ok, "pass": bool(rel.max() <= PCE_RTOL and flags_ok),
            "oracle": "oracle/pce.py float64 (scipy-batched irfft2)"}


def ncc_parity(args, n, side, out, flags, items=None):
    """Sampled pair ids of the finished NCC job against the float64 oracle (|err| <= 2e-4, TF32)."""
    import numpy as np
    import torch

    from oracle import ncc as oncc
    from oracle import scheduler as osch
    from paper_2009_04755_b200 import device
    f = flags.cpu().numpy()
    mine = np.flatnonzero(f)
    if len(mine) == 0:
        return {"sampled": 0, "max_abs_err": None, "tolerance": 2e-4, "pass": False}
    rng = np.random.default_rng(args.seed + 99)
    pids = sorted(int(x) for x in rng.choice(mine, size=min(args.parity_samples, len(mine)), replace=False))
    ss = side * side
    buf = torch.empty(ss, dtype=torch.float32, device="cuda")
    vec = {}
    for p in pids:
        for k in osch.pair_from_id(n, p):
            if k not in vec:
                if items is not None:
                    x = items[k * ss:(k + 1) * ss].cpu().numpy()
                else:
                    device.synth_prnu(side, side, k, 1, args.cameras, args.seed, buf)
                    x = buf.cpu().numpy()
                vec[k] = oncc.preprocess(x)
    want = np.array([oncc.compare(*(vec[k] for k in osch.pair_from_id(n, p))) for p in pids])
    got = out.cpu().numpy()[pids]
    err = float(np.max(np.abs(got - want)))
    flags_ok = bool(np.all(np.where(got >= 0.02, f[pids] == 3, f[pids] == 1)))
    return {"sampled": len(pids), "max_abs_err": err, "tolerance": 2e-4, "flags_match": flags_ok,
            "pass": bool(err <= 2e-4 and flags_ok), "oracle": "oracle/ncc.py float64"}


def calibrate_ncc(args, params_fn, side, cameras, seed):
    """Isolated single-GPU NCC stage costs: t_pre per item (normalise), t_cmp per pair
    of a resident Gram over m items (m large enough for > 1 wave of 256 x 256 tiles)."""
    import torch

    from paper_2009_04755_b200 import device
    ss = side * side
    free = torch.cuda.mem_get_info()[0]
    m = int(min(args.items, 4096, (free - (24 << 30)) // (ss * 4)) // 256 * 256)
    m = max(m, 256)
    app = device.DeviceApp(params_fn(m))
    slots = app.alloc_slots(m)
    raw = torch.empty(256 * ss, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    t_pre = 0.0
    for c0 in range(0, m, 256):
        cnt = min(256, m - c0)
        device.synth_prnu(side, side, c0, cnt, cameras, seed, raw)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        app.preprocess(raw, ss * 4, cnt, slots, list(range(c0, c0 + cnt)))
        e1.record(s)
        torch.cuda.synchronize()
        t_pre += e0.elapsed_time(e1) / 1e3
    del raw
    out = torch.zeros(m * (m - 1) // 2, dtype=torch.float64, device="cuda")
    app.gram(slots, m, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(2):
        app.gram(slots, m, out)
    e1.record(s)
    torch.cuda.synchronize()
    t_cmp = e0.elapsed_time(e1) / 1e3 / (2 * m * (m - 1) // 2)
    app.close()
    del slots, out
    torch.cuda.empty_cache()
    return t_pre / m, t_cmp


def leaf_ordered_pairs(m, leaf):
    """All (i, j), i < j < m, in leaf order: leaf x leaf blocks of the upper
    triangle (block rows, then block columns), pairs row-major inside a block."""
    lb = max(1, int(leaf))
    pairs = [(i, j) for bi in range(0, m, lb) for bj in range(bi, m, lb)
             for i in range(bi, min(bi + lb, m)) for j in range(max(bj, i + 1), min(bj + lb, m))]
    assert len(pairs) == m * (m - 1) // 2
    return pairs


def calibrate_pce(args, params_fn, side, cameras, seed):
    """Isolated single-GPU stage costs for the perf model (perfmodel.py:99-114):
    t_pre = preprocess time per item, t_cmp = compare time per pair, each from
    CUDA events on a fresh app with nothing else running on the GPU."""
    import torch

    from paper_2009_04755_b200 import device
    m = 64
    app = device.DeviceApp(params_fn(m))
    ss = side * side
    raw = torch.empty(m * ss, dtype=torch.float32, device="cuda")
    device.synth_prnu(side, side, 0, m, cameras, seed, raw)
    slots = app.alloc_slots(m)
    import ctypes as C

    from paper_2009_04755_b200 import _lib
    # pairs in the engine's leaf order (leaf_block x leaf_block blocks of the
    # triangle, pairs row-major inside a block): a round of the persistent compare
    # grid then draws on as few spectra as it does in a job
    plist = [(i, j, i, j) for i, j in leaf_ordered_pairs(m, args.leaf)]
    pairs = (_lib.Pair * len(plist))(*[_lib.Pair(*p) for p in plist])   # built once: no host gaps
    out = torch.zeros(m * (m - 1) // 2, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    idx = (C.c_int32 * m)(*range(m))

    def pre():
        _lib.check(_lib.lib.rk_preprocess(app.handle, raw.data_ptr(), ss * 4, m, slots.data_ptr(), app.slot_stride,
                                          idx, s.cuda_stream))

    def cmp():
        _lib.check(_lib.lib.rk_compare_pairs(app.handle, slots.data_ptr(), app.slot_stride, pairs, len(plist),
                                             out.data_ptr(), None, s.cuda_stream))
    pre()
    cmp()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(s)
    for _ in range(3):
        pre()
    e[1].record(s)
    e[2].record(s)
    for _ in range(3):
        cmp()
    e[3].record(s)
    torch.cuda.synchronize()
    t_pre = e[0].elapsed_time(e[1]) / 1e3 / (3 * m)
    t_cmp = e[2].elapsed_time(e[3]) / 1e3 / (3 * len(plist))
    app.close()
    del raw, slots, out
    torch.cuda.empty_cache()
    return t_pre, t_cmp


# ---------------------------------------------------------------------------

def main_pce(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2009_04755_b200 import _lib, device
    from paper_2009_04755_b200.engine import gather_triangle
    from paper_2009_04755_b200 import perfmodel

    n, side = args.items, args.side
    pairs_total = n * (n - 1) // 2
    metric, cfg, dtype = workload(args, world)
    streamed = home_only(args)
    if streamed and world < 2:
        print(json.dumps({"metric": metric, "value": None, "unit": "pairs/s", "n_gpus": world, "config": cfg,
                          "error": f"{n} patterns of {side}^2 need {2 * n * side * side * 4 / 2**30:.0f} GiB "
                                   "(patterns + spectra), more than one GPU's HBM: run with --gpus >= 2"}))
        return 2

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if world > 1:
            dist.barrier()

    ss = side * side
    parsed_bytes = ss * 4

    ncc = args.app == "ncc"

    def params_fn(m):
        if ncc:
            return _lib.app_params(_lib.APP_NCC, m, height=side, width=side, threshold=0.02)
        return _lib.app_params(_lib.APP_PCE, m, height=side, width=side, threshold=60.0)

    # isolated single-GPU stage costs (rank 0 alone on its GPU; the others wait)
    t_pre = t_cmp = None
    if rank == 0:
        calib = calibrate_ncc if ncc else calibrate_pce
        t_pre, t_cmp = calib(args, params_fn, side, args.cameras, args.seed)
    barrier()

    items = None
    if not streamed:
        items = torch.empty(n * ss, dtype=torch.float32, device="cuda")
        device.synth_prnu(side, side, 0, n, args.cameras, args.seed, items)
    params = params_fn(n)
    # N > 1: peer-GPU tier -- each rank preprocesses its home items (k % N == rank),
    # every other item it needs is copied from its home GPU over NVLink (CUDA IPC)
    # NCC whose items fit every GPU: each rank keeps all items resident and takes its
    # round-robin share of the Gram tiles (a C2-size Gram is only ~1.8 waves of
    # 256 x 256 tiles on one GPU, too little to split into peer-fetched sub-blocks);
    # the peer tier carries C3-Gram (home-only)
    peer = world > 1 and (not ncc or streamed)
    steal = peer and not args.no_steal and not ncc     # the Gram deals its blocks statically
    if streamed:
        home_cnt = len(range(rank, n, world))
        free = torch.cuda.mem_get_info()[0]
        slot_bytes = ss * 4
        # cache slots: what is left after the home region, T scratch and the result triangle
        budget = free - home_cnt * slot_bytes - pairs_total * 9 - (12 << 30)
        dslots = args.slots or max(64, int(budget // slot_bytes))
        if ncc:   # two fetch buffers of (at most) 2,048 items: the Gram's key sub-blocks
            dslots = args.slots or min(4096, int(budget // slot_bytes) // 256 * 256)
    elif ncc and peer:
        dslots = args.slots or min(4096, (n // world + 255) // 256 * 256 * 2)
    else:
        dslots = n
    eng = device.DeviceEngine(params, leaf_block=args.leaf, device_slots=dslots, rank=rank, world=world,
                              device=local_rank, peer_tier=peer, steal=steal, steal_chunk=args.steal_chunk)
    out = torch.zeros(pairs_total, dtype=torch.float64, device="cuda")
    flags = torch.zeros(pairs_total, dtype=torch.uint8, device="cuda")
    estream = torch.cuda.ExternalStream(eng.stream())
    gen = torch.empty((256 if streamed else 0) * ss, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    state = {"connected": False}

    load_ms = []

    def load_home_streamed():
        # the load stage of home-only mode: generate (storage) + preprocess, 256 items at a time
        home = list(range(rank, n, world))
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(estream)
        with torch.cuda.stream(estream):
            for m0 in range(0, len(home), 256):
                cnt = min(256, len(home) - m0)
                for q in range(cnt):
                    device.synth_prnu(side, side, home[m0 + q], 1, args.cameras, args.seed,
                                      gen.narrow(0, q * ss, ss), stream=estream)
                eng.load_home_range(m0, cnt, device_items=gen, parsed_stride=parsed_bytes)
        h1.record(estream)
        h1.synchronize()
        load_ms.append(h0.elapsed_time(h1))

    def step(host_home=None, host_all=None):
        """One full job on this rank: [home preprocess + barrier] + all of its pairs [+ barrier]."""
        if peer:
            if streamed:
                load_home_streamed()
            elif host_home is not None:
                eng.load_home(host_items=host_home, parsed_stride=parsed_bytes)
            else:
                eng.load_home(device_items=_At(items, rank * parsed_bytes), parsed_stride=world * parsed_bytes)
            if not state["connected"]:
                eng.connect_peers()
                state["connected"] = True
            if steal:
                eng.queue_reset()
            eng.ledger_reset()          # rank 0 clears the job's shared exactly-once ledger
            barrier()
            eng.run(out, flags, host_items=host_home if not streamed else None,
                    device_items=None if (host_home is not None or streamed) else items,
                    parsed_stride=parsed_bytes)
            barrier()
        else:
            if world > 1:   # the job's shared ledger on rank 0 (IPC), reset before the barrier
                if not state["connected"]:
                    eng.connect_peers()
                    state["connected"] = True
                eng.ledger_reset()
                barrier()
            if host_all is not None:
                eng.run(out, flags, host_items=host_all, parsed_stride=parsed_bytes)
            else:
                eng.run(out, flags, device_items=items, parsed_stride=parsed_bytes)
            if world > 1:
                barrier()

    for _ in range(args.warmup):
        step()
    eng.reset_stats()
    eng.set_profiling(every=3, max_samples=8192)
    clocks = ClockSampler(local_rank)
    out.zero_()
    flags.zero_()
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(estream)
    kms, ksamples, kpairs = 0.0, 0, 0
    load_ms.clear()
    for _ in range(args.steps):
        step()
        a, b, c = eng.kernel_time()
        kms += a
        ksamples += b
        kpairs += c
    ev1.record(estream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    ms = ev0.elapsed_time(ev1)
    st = eng.stats()
    my_pairs = st["pairs_done"]
    t = torch.tensor([ms, float(my_pairs)], dtype=torch.float64, device="cuda")
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        ms, all_pairs = float(tmax[0]), float(t[1])
    else:
        all_pairs = float(my_pairs)
    value = all_pairs / (ms / 1e3)
    breakdown = None
    if streamed:
        # per job: the home load stage (generation = the storage read, + preprocess) and the
        # rest (barrier, all pairs, barrier), max over ranks
        lt = torch.tensor([sum(load_ms) / max(1, len(load_ms))], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(lt, op=dist.ReduceOp.MAX)
        breakdown = {"home_load_ms": float(lt[0]), "pairs_ms": ms / args.steps - float(lt[0]),
                     "what": "home_load = synthetic generation (the storage read) + preprocess of this rank's "
                             "home items; pairs = the rest of the job (max over ranks)"}
    eng.set_profiling(0)
    # cache accounting over the whole job (runner.py:41 R = loads / n; slotcache.py:252-260 tiers)
    ct = torch.tensor([st["loads"], st["hits"], st["misses"], st["peer_fetches"], st["steals"],
                       st["peer_bytes"]], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ct, op=dist.ReduceOp.SUM)
    loads_all, hits_all, misses_all, peer_all, steals_all, pbytes_all = \
        [float(x) / max(1, args.steps) for x in ct.tolist()]
    # the last timed job's exactly-once ledger (rank 0 holds the job's shared one)
    ledger = eng.ledger() if rank == 0 else None

    parity = None
    if rank == 0 and not args.no_parity:
        parity = (ncc_parity if ncc else pce_parity)(args, n, side, out, flags, items=items)

    # ---- e2e: pinned host patterns -> engine -> packed triangle back on host
    e2e = None
    if streamed:
        e2e = {"value": None, "unit": "pairs/s",
               "reason": f"home-only mode: the {n * parsed_bytes / 2**30:.0f} GiB of patterns are generated on "
                         "their home GPUs (no host copy of the workload exists)"}
    elif not args.no_e2e:
        try:
            if peer:
                # a rank needs only its home items on the host (every other item comes over NVLink)
                host = torch.empty((len(range(rank, n, world)), ss), dtype=torch.float32, pin_memory=True)
                host.copy_(items.view(n, ss)[rank::world])
                host_home, host_all = host, None
            else:
                host = torch.empty(n * ss, dtype=torch.float32, pin_memory=True)
                host.copy_(items)
                host_home, host_all = None, host
            res_host = torch.empty(pairs_total, dtype=torch.float64, pin_memory=True)
            flags_host = torch.empty(pairs_total, dtype=torch.uint8, pin_memory=True)
            del items
            items = None
            torch.cuda.empty_cache()
            step(host_home=host_home, host_all=host_all)   # warm the H2D path
            eng.reset_stats()
            barrier()
            torch.cuda.synchronize()
            # events on torch's stream bracket the engine's stream work: rk_engine_run is
            # synchronous, and the D2H of the results follows it on this stream
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                out.zero_()       # every job delivers a fresh triangle (the reduce below is in place)
                flags.zero_()
                step(host_home=host_home, host_all=host_all)
                gather_triangle(out, flags)            # disjoint pair ids: exact gather to rank 0
                res_host.copy_(out, non_blocking=True)
                flags_host.copy_(flags, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            ems = e0.elapsed_time(e1)
            st2 = eng.stats()
            tt = torch.tensor([ems], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt[0])
            e2e = {"value": all_pairs / (ems / 1e3), "unit": "pairs/s",
                   "h2d_bytes_per_step": int(st2["h2d_bytes"] // max(1, args.steps)),
                   "d2h_bytes_per_step": pairs_total * 9,
                   "peer_bytes_per_step": int(st2.get("peer_bytes", 0) // max(1, args.steps))}
            if rank == 0:
                fh = flags_host.numpy()
                e2e["check"] = {"flags_exactly_once": bool(((fh == 1) | (fh == 3)).all()),
                                "what": "every delivered flag is 1 or 3 after the last step's gather"}
        except RuntimeError as exc:  # e.g. pinned-memory exhaustion
            e2e = {"value": None, "unit": "pairs/s", "error": str(exc)[:200]}

    if args.trace_dir and not streamed and items is not None:
        # one extra (untimed) step with trace events: the reference's trace JSONL per
        # rank and its RunMetrics document (metrics.py) with the perf-model efficiency
        from paper_2009_04755_b200 import metrics as rk_metrics
        os.makedirs(args.trace_dir, exist_ok=True)
        eng.set_trace(200000)
        eng.reset_stats()
        step()
        ev = eng.trace(node=rank)
        eng.set_trace(0)
        rk_metrics.write_trace(os.path.join(args.trace_dir, f"trace_rank{rank}.jsonl"), ev)
        span = (max(e["end_ns"] for e in ev) - min(e["start_ns"] for e in ev)) / 1e9 if ev else 0.0
        node = rk_metrics.node_metrics(rank, eng.stats(), span, n, ev)
        nodes = [(node, span)]
        if world > 1:
            nodes = [None] * world
            dist.all_gather_object(nodes, (node, span))
        if rank == 0:
            costs = perfmodel.StageCosts(t_preprocess=t_pre, t_comparison=t_cmp)
            doc = rk_metrics.run_metrics({"workload": cfg["workload"], "n": n, "side": side,
                                          "leaf_block": args.leaf, "world": world}, n, [x[0] for x in nodes],
                                         max(x[1] for x in nodes), costs=costs)
            rk_metrics.write_metrics(os.path.join(args.trace_dir, "metrics.json"), doc)

    if rank != 0:
        eng.close()
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks, peaks_src = load_peaks()
    hbm = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    slot_bytes = ss * 4
    alg_bytes_per_pair = 2 * slot_bytes          # two half-spectra per pair
    roofline = None
    traffic = None
    try:   # dram bytes of one compare launch from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "pce_cluster_traffic.json")) as fh:
            tj = json.load(fh)
        rec = tj.get(str(side), tj) if isinstance(tj, dict) else tj
        traffic_per_pair = (rec["dram_bytes_read_per_launch"] + rec["dram_bytes_write_per_launch"]) / \
            rec["pairs_per_launch"]
        if rec.get("side", 1024) != side:
            traffic_per_pair = None      # the capture is for another pattern size
    except Exception:
        traffic_per_pair = None
    if ncc:
        # tensor-bound: 2 D flops per pair over the whole job (preprocess and fetches included)
        tf32, tf32_src = None, None
        try:
            with open(os.path.join(ROOT, "profiles", "r2_tf32_peak.json")) as fh:
                tf32 = float(json.load(fh)["tf32"]["burst_tflops"])
            tf32_src = "profiles/r2_tf32_peak.json (cuBLAS TF32 8192^3 on B200, burst)"
        except Exception:
            tf32 = 0.5 * float(peaks.get("bf16_tflops", PEAKS_FALLBACK["bf16_tflops"]))
            tf32_src = "fallback: half the measured dense BF16 (MEASURED_PEAKS.json)"
        achieved = 2.0 * ss * (all_pairs / max(1, args.steps)) / (ms / 1e3 / args.steps) / 1e12
        roofline = {"bound": "tensor", "achieved": achieved, "peak": tf32 * world, "unit": "TFLOP/s",
                    "frac": achieved / (tf32 * world), "traffic": None, "peak_source": tf32_src,
                    "kernel": "ncc_gram2_kernel (tcgen05.mma.cta_group::2.kind::tf32, 256x256 item tiles, TMA)",
                    "flops_per_pair": 2 * ss, "what": "whole job (normalise + fetches + Gram) per step"}
    elif ksamples:
        per_launch_ms = kms / ksamples
        batch = kpairs / ksamples
        achieved = alg_bytes_per_pair * batch / (per_launch_ms / 1e3) / 1e9
        if traffic_per_pair is not None:
            traffic = traffic_per_pair * batch
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "traffic": traffic,
                    "traffic_source": "profiles/pce_cluster_traffic.json (ncu dram__bytes_read+write, per launch)",
                    "kernel": ("pce_cluster" if side <= 1024 else "pce2k_pair")
                              + " (persistent, one CTA = one SM per pair in flight: column + row pass)",
                    "pairs_per_launch": batch, "ms_per_launch": per_launch_ms, "launches_sampled": ksamples,
                    "alg_bytes_per_pair": alg_bytes_per_pair, "peak_source": peaks_src,
                    "fp32_flops_per_pair": 2 * 5 * (side // 2) * side * math.log2(side),
                    "grid": {"round_barrier": os.environ.get("RK_PCE_LOCKSTEP", "1") != "0" and side >= 1024,
                             "l2opts": int(os.environ.get("RK_PCE_L2OPTS", "3" if side == 2048 else "0")),
                             "what": "persistent-grid round barrier and L2 hints (bit 0 T evict_first, "
                                     "bit 1 spectra evict_last) the compare kernel ran with"}}

    t_min = n * t_pre + pairs_total * t_cmp
    perf = {"t_pre_s": t_pre, "t_cmp_s": t_cmp, "T_min_s": t_min, "p": world, "T_s": ms / 1e3 / args.steps,
            "efficiency": perfmodel.efficiency(t_min, world, ms / 1e3 / args.steps),
            "method": "t_pre, t_cmp from an isolated single-GPU pass (64 items, 2,016 pairs, CUDA events) "
                      "before the timed steps; efficiency = (T_min / p) / T, perfmodel.py:99-114"}

    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_baseline(args, args.cpu_seconds)

    line = {"metric": metric, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": dtype, "data": "synthetic", "config": cfg,
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk, "parity": parity,
            "perf_model": perf, "job_breakdown": breakdown, "gpu_launches": st["kernel_launches"],
            "ledger": dict(ledger, what="device bitmap of C(n,2) bits set by every compare epilogue "
                                        "(atomicOr over NVLink into rank 0's ledger at N > 1), last timed job"),
            "cache": {"R": loads_all / n, "loads_per_step": loads_all, "device_slots_per_gpu": dslots,
                      "device_hit_rate": hits_all / max(1.0, hits_all + misses_all),
                      "device_hits_per_step": hits_all, "device_misses_per_step": misses_all,
                      "peer_fetches_per_step": peer_all, "peer_gib_per_step": pbytes_all / 2**30,
                      "peer_hit_rate": peer_all / max(1.0, misses_all) if world > 1 else None,
                      "steals_per_step": steals_all if world > 1 else None}}
    print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main_app(args, rank, world, local_rank):
    """gmm (configs[3]) / cv (configs[4]): same contract as the PCE line."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2009_04755_b200 import _lib, device, synthdata
    from paper_2009_04755_b200.engine import gather_triangle
    n = args.items
    pairs_total = n * (n - 1) // 2
    metric, cfg, dtype = workload(args, world)
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if world > 1:
            dist.barrier()

    if args.app == "gmm":
        host_np, msum = synthdata.gmm_parsed(n, args.seed, 400)
        stride = host_np.shape[1]
        items = torch.from_numpy(host_np.reshape(-1)).cuda()
        params = _lib.app_params(_lib.APP_GMM, n, max_entries=400, gmm_angles=args.angles)
        work = args.angles * (float(msum.sum()) ** 2 - float((msum.astype(np.float64) ** 2).sum())) / 2.0
    else:
        items, stride, cap, nnz = synthdata.cv_parsed_device(n, args.mean_nnz, args.seed)
        params = _lib.app_params(_lib.APP_CV, n, max_entries=cap, threshold=0.5)
        work = 16.0 * (n - 1) * float(nnz.sum())   # sum over pairs of 16 (nnz_i + nnz_j) bytes
    multi = world > 1
    eng = device.DeviceEngine(params, leaf_block=16, device_slots=n, rank=rank, world=world, device=local_rank,
                              peer_tier=multi, steal=multi and not args.no_steal, steal_chunk=args.steal_chunk)
    out = torch.zeros(pairs_total, dtype=torch.float64, device="cuda")
    flags = torch.zeros(pairs_total, dtype=torch.uint8, device="cuda")
    estream = torch.cuda.ExternalStream(eng.stream())
    state = {"connected": False}

    def step(host=None):
        src = host if host is not None else items
        if multi:
            eng.load_home(**({"host_items": _At(src, rank * stride)} if host is not None
                             else {"device_items": _At(src, rank * stride)}), parsed_stride=world * stride)
            if not state["connected"]:
                eng.connect_peers()
                state["connected"] = True
            if eng.steal:
                eng.queue_reset()
            eng.ledger_reset()
            barrier()
        eng.run(out, flags, **({"host_items": host} if host is not None else {"device_items": items}),
                parsed_stride=stride)
        if multi:
            barrier()

    for _ in range(args.warmup):
        step()
    eng.reset_stats()
    clocks = ClockSampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(estream)
    for _ in range(args.steps):
        step()
    ev1.record(estream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    st = eng.stats()
    t = torch.tensor([ms, float(st["pairs_done"]), float(st["loads"]), float(st["hits"]), float(st["misses"])],
                     dtype=torch.float64, device="cuda")
    if multi:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        ms = float(tmax[0])
    all_pairs, loads_all, hits_all, misses_all = [float(x) for x in t[1:].tolist()]
    value = all_pairs / (ms / 1e3)
    ledger = eng.ledger() if rank == 0 else None
    e2e = None
    parsed_total = n * stride
    try:   # pinned host copy of every parsed item: at most a third of the host's memory
        host_ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError, AttributeError):
        host_ram = 64 << 30
    if not args.no_e2e and parsed_total <= host_ram // 3:
        host = torch.empty(parsed_total, dtype=torch.uint8, pin_memory=True)
        host.copy_(items)
        res_host = torch.empty(pairs_total, dtype=torch.float64, pin_memory=True)
        flags_host = torch.empty(pairs_total, dtype=torch.uint8, pin_memory=True)
        step(host)
        eng.reset_stats()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            out.zero_()        # fresh triangle per job: the NCCL reduce below is in place
            flags.zero_()
            step(host)
            gather_triangle(out, flags)
            res_host.copy_(out, non_blocking=True)
            flags_host.copy_(flags, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ems = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        st2 = eng.stats()
        if multi:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": pairs_total * args.steps / (float(ems[0]) / 1e3), "unit": "pairs/s",
               "h2d_bytes_per_step": int(st2["h2d_bytes"] // max(1, args.steps)),
               "d2h_bytes_per_step": pairs_total * 9}
        if rank == 0:
            fh = flags_host.numpy()
            e2e["check"] = {"flags_exactly_once": bool(((fh == 1) | (fh == 3)).all())}
    sm_mhz = clk.get("sm_mhz") or 1965.0
    per_job_s = ms / 1e3 / args.steps
    if args.app == "gmm":
        peak = 148 * 16 * sm_mhz * 1e6 * world
        roofline = {"bound": "sfu", "achieved": work / per_job_s / 1e12, "peak": peak / 1e12, "unit": "Tex2/s",
                    "frac": work / per_job_s / peak, "traffic": None,
                    "peak_source": f"148 SMs x 16 MUFU.EX2/clk x measured {sm_mhz:.0f} MHz x {world} GPU(s)",
                    "kernel": "gmm_pair_kernel (CTA per pair x 12-angle block)", "ex2_per_job": work}
    else:
        peaks, src = load_peaks()
        peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])) * world
        roofline = {"bound": "hbm", "achieved": work / per_job_s / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": work / per_job_s / 1e9 / peak, "traffic": None, "peak_source": src,
                    "kernel": "cv_work (merge-path units, coalesced token windows)",
                    "alg_bytes_per_job": work}
    cpu = None
    if rank == 0 and not args.no_cpu and world == 1:
        cpu = cpu_baseline(args, args.cpu_seconds)
    if rank == 0:
        steps = max(1, args.steps)
        print(json.dumps({"metric": metric, "value": value, "unit": "pairs/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                          "dtype": dtype, "data": "synthetic", "config": cfg,
                          "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
                          "gpu_launches": st["kernel_launches"], "ledger": ledger,
                          "cache": {"R": loads_all / steps / n, "loads_per_step": loads_all / steps,
                                    "device_hit_rate": hits_all / max(1.0, hits_all + misses_all),
                                    "steals": st["steals"], "peer_fetches": st["peer_fetches"]}}), flush=True)
    eng.close()
    if multi:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------

def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args_gpus: int) -> int:
    """`--gpus N` outside torchrun: run this script under torch.distributed.run with N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args_gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank)
    if env_world is None and args.gpus > 1:
        return relaunch(args.gpus)
    world = int(env_world or "1")
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop torchrun and let --gpus relaunch", file=sys.stderr)
        return 2
    if args.app not in ("pce", "ncc"):
        return main_app(args, rank, world, local_rank)
    return main_pce(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
