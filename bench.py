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
  cpu_baseline  the float64 oracle (oracle/pce.py) on a bounded pair sample

`python bench.py --impl reference` times the reference-side CPU path (the
oracle port; the reference itself has no PCE) on the same workload.
Multi-GPU: launched under torchrun, leaves are sharded across ranks (strong
scaling of one job); every item is preprocessed once on its home GPU (k mod N)
and other ranks fetch it over NVLink (peer tier, CUDA IPC); NCCL is used once,
to reduce the result triangle to rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--items", type=int, default=4096, help="items (default: configs[1], 4,096)")
    ap.add_argument("--side", type=int, default=1024, help="pattern side (default 1024)")
    ap.add_argument("--leaf", type=int, default=8)
    ap.add_argument("--cameras", type=int, default=64)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-steal", action="store_true", help="N > 1: static leaf shares, no cross-GPU stealing")
    ap.add_argument("--trace-dir", default="",
                    help="pce: after the timed steps, run one traced step and write the reference-schema "
                         "trace (JSONL) and run-metrics document of each rank here")
    ap.add_argument("--app", default="pce", choices=["pce", "gmm", "cv"],
                    help="pce: configs[1] (default); gmm: configs[3]; cv: configs[4]")
    ap.add_argument("--angles", type=int, default=36, help="gmm: rotation grid K")
    ap.add_argument("--mean-nnz", type=float, default=5e5, help="cv: mean tokens per item")
    return ap.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d, "measured"
    except Exception:
        return dict(PEAKS_FALLBACK), "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        if os.environ.get("RK_NO_CLOCKS"):   # diagnosis: measure without the sampler
            self.proc = None
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = []
        smax = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
            except ValueError:
                continue
            for name, val in zip(names, r[5:9]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: float64 oracle on a bounded pair sample (TEST-INFRASTRUCTURE code
# used only as the timed reference arm, never as the product path).

def _cpu_worker(args):
    side, seed, cameras, keys, budget = args
    from oracle import pce as opce
    # item generation is the load stage (fetch_raw), not part of the timed work
    items = {k: opce.prnu_patterns(side, side, k, 1, cameras, seed)[0] for k in keys}
    pairs = [(a, b) for ai, a in enumerate(keys) for b in keys[ai + 1:]]
    spectra = {}
    done = 0
    t0 = time.perf_counter()
    for (i, j) in pairs:
        for k in (i, j):
            if k not in spectra:
                spectra[k] = opce.preprocess(items[k])      # rfft2, charged like the GPU preprocess
        opce.compare(spectra[i], spectra[j], side, side)
        done += 1
        if time.perf_counter() - t0 > budget:
            break
    return done, time.perf_counter() - t0, len(spectra)


def cpu_baseline(n, side, cameras, seed, budget_s):
    """Pairs/s of the float64 oracle port over all host cores (one process per core).

    Each worker takes a 24-item leaf-like block of keys, generates the items
    (untimed, the load stage), then preprocesses (rfft2) and compares its
    block's pairs until the budget expires; value = pairs / slowest worker."""
    import multiprocessing as mp
    import random
    cores = os.cpu_count() or 1
    rng = random.Random(seed)
    blocks = []
    for w in range(cores):
        base = rng.randrange(0, max(1, n - 24))
        blocks.append(list(range(base, min(n, base + 24))))
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_cpu_worker, [(side, seed, cameras, blk, budget_s) for blk in blocks])
    wall = time.perf_counter() - t0
    pairs = sum(r[0] for r in res)
    busy = max(r[1] for r in res)
    return {"value": pairs / busy, "unit": "pairs/s", "cores": cores, "kind": "port",
            "sample": f"{pairs} pairs of {side}x{side} PCE (24-item blocks per process, rfft2 preprocess "
                      f"included, item generation excluded) on {cores} processes, {busy:.1f}s timed "
                      f"({wall:.1f}s wall incl. spawn and generation)"}


def _gmm_worker(args):
    keys, seed, angles, budget = args
    from oracle import gmm as ogmm
    from paper_2009_04755_b200.synthdata import particle
    parts = {k: particle(k, seed) for k in keys}          # load stage, untimed
    done, t0 = 0, time.perf_counter()
    for ai, a in enumerate(keys):
        for b in keys[ai + 1:]:
            ogmm.compare(parts[a], parts[b], angles)
            done += 1
            if time.perf_counter() - t0 > budget:
                return done, time.perf_counter() - t0
    return done, time.perf_counter() - t0


def _cv_worker(args):
    sizes, seed, budget = args
    from oracle import cv as ocv
    from paper_2009_04755_b200.synthdata import cv_parsed_host
    blobs = cv_parsed_host(sizes, seed)                    # load stage, untimed
    done, t0 = 0, time.perf_counter()
    vecs = {}
    for a in range(len(blobs)):
        for b in range(a + 1, len(blobs)):
            for k in (a, b):
                if k not in vecs:
                    vecs[k] = ocv.preprocess(blobs[k])     # count -> freq, charged like the GPU preprocess
            ocv.compare(vecs[a], vecs[b])
            done += 1
            if time.perf_counter() - t0 > budget:
                return done, time.perf_counter() - t0
    return done, time.perf_counter() - t0


def cpu_baseline_app(app, n, seed, budget_s, angles=36, mean_nnz=5e5):
    """The oracle's CPU compare (oracle/gmm.py numpy, oracle/cv.py the reference's
    sequential merge restated) on all host cores over a bounded pair sample."""
    import multiprocessing as mp
    import random
    cores = os.cpu_count() or 1
    rng = random.Random(seed)
    if app == "gmm":
        jobs = []
        for _ in range(cores):
            base = rng.randrange(0, max(1, n - 24))
            jobs.append((list(range(base, min(n, base + 24))), seed, angles, budget_s))
        worker, what = _gmm_worker, f"particle pairs (K={angles}, numpy float64)"
    else:
        from paper_2009_04755_b200.synthdata import cv_nnz
        sizes = cv_nnz(n, mean_nnz, seed)
        jobs = [([int(x) for x in sizes[rng.randrange(0, n - 6):][:6]], seed + w, budget_s) for w in range(cores)]
        worker, what = _cv_worker, "composition-vector pairs (pure-Python merge of the reference's compare)"
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(worker, jobs)
    wall = time.perf_counter() - t0
    pairs = sum(r[0] for r in res)
    busy = max(r[1] for r in res)
    return {"value": pairs / busy, "unit": "pairs/s", "cores": cores, "kind": "port",
            "sample": f"{pairs} {what} on {cores} processes, {busy:.1f}s timed ({wall:.1f}s wall incl. "
                      f"spawn and item generation)"}


def main_app(args, rank, world, local_rank):
    """gmm (configs[3]) / cv (configs[4]): same contract as the PCE line."""
    import numpy as np
    n = args.items if args.items != 4096 else (1000 if args.app == "gmm" else 2500)
    pairs_total = n * (n - 1) // 2
    if args.app == "gmm":
        workload = (f"particle fusion (GMM/Bhattacharyya), N={n} particles of ~300 localizations, "
                    f"K={args.angles} rotations (BASELINE configs[3])")
    else:
        workload = (f"composition-vector cosine, N={n} variable-length items, nnz lognormal in [1e5, 1.8e6] "
                    f"(mean {args.mean_nnz:.0f}) (BASELINE configs[4])")
    metric = "pairs/sec (whole box)"
    budget = max(3.0, args.cpu_seconds / 3)
    if args.impl == "reference":
        if rank != 0:
            return 0
        vals, cb = [], None
        for _ in range(max(1, args.warmup) + args.steps):
            cb = cpu_baseline_app(args.app, n, args.seed, budget, args.angles, args.mean_nnz)
            vals.append(cb["value"])
        value = sum(vals[args.warmup:] or vals) / len(vals[args.warmup:] or vals)
        print(json.dumps({"metric": metric, "value": value, "unit": "pairs/s", "impl": "reference", "n_gpus": args.gpus, "host_only": True,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * pairs_total / value,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic", "config": {"workload": workload, "n": n,
                                                          "parallelism": f"cpu{cb['cores']}"},
                          "cpu_baseline": dict(cb, value=value),
                          "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return 0

    import torch
    import torch.distributed as dist
    from paper_2009_04755_b200 import _lib, device
    from paper_2009_04755_b200.engine import gather_triangle
    from paper_2009_04755_b200 import synthdata
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
                              peer_tier=multi, steal=multi and not args.no_steal)
    out = torch.zeros(pairs_total, dtype=torch.float64, device="cuda")
    flags = torch.zeros(pairs_total, dtype=torch.uint8, device="cuda")
    estream = torch.cuda.ExternalStream(eng.stream())

    class _At:
        def __init__(self, t, off):
            self.t, self.off = t, off

        def data_ptr(self):
            return self.t.data_ptr() + self.off

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
    t = torch.tensor([ms, float(st["pairs_done"])], dtype=torch.float64, device="cuda")
    if multi:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        ms = float(tmax[0])
    value = float(t[1]) / (ms / 1e3)
    e2e = None
    parsed_total = n * stride
    if not args.no_e2e and parsed_total <= (24 << 30):
        host = torch.empty(parsed_total, dtype=torch.uint8, pin_memory=True)
        host.copy_(items)
        res_host = torch.empty(pairs_total, dtype=torch.float64, pin_memory=True)
        step(host)
        eng.reset_stats()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step(host)
            gather_triangle(out, flags)
            res_host.copy_(out, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ems = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        st2 = eng.stats()
        if multi:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": pairs_total * args.steps / (float(ems[0]) / 1e3), "unit": "pairs/s",
               "h2d_bytes_per_step": int(st2["h2d_bytes"] // max(1, args.steps)),
               "d2h_bytes_per_step": pairs_total * 8}
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
        cpu = cpu_baseline_app(args.app, n, args.seed, budget, args.angles, args.mean_nnz)
    if rank == 0:
        print(json.dumps({"metric": metric, "value": value, "unit": "pairs/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                          "dtype": "fp32" if args.app == "gmm" else "fp64", "data": "synthetic",
                          "config": {"workload": workload, "n": n, "pairs": pairs_total, "leaf_block": 16,
                                     "parallelism": f"pairs{world}",
                                     "l2": f"items {parsed_total / 2**30:.1f} GiB parsed"},
                          "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
                          "gpu_launches": st["kernel_launches"],
                          "cache": {"R": st["loads"] / n, "device_hit_rate":
                                    st["hits"] / max(1, st["hits"] + st["misses"]),
                                    "steals": st["steals"], "peer_fetches": st["peer_fetches"]}}), flush=True)
    eng.close()
    if multi:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------

def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.app != "pce":
        return main_app(args, rank, world, local_rank)
    n, side = args.items, args.side
    pairs_total = n * (n - 1) // 2
    cfg_name = {(4096, 1024): " (BASELINE configs[1])", (16384, 2048): " (BASELINE configs[2])"}.get((n, side), "")
    workload = f"PRNU PCE all-pairs, N={n} patterns of {side}x{side} fp32{cfg_name}"
    metric = "pairs/sec (whole box)"

    if args.impl == "reference":
        if rank != 0:
            return 0
        steps = []
        cb = None
        for _ in range(max(1, args.warmup) + args.steps):
            cb = cpu_baseline(n, side, args.cameras, args.seed, max(3.0, args.cpu_seconds / 3))
            steps.append(cb["value"])
        vals = steps[args.warmup:] or steps
        value = sum(vals) / len(vals)
        line = {"metric": metric, "value": value, "unit": "pairs/s", "impl": "reference", "n_gpus": args.gpus, "host_only": True,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * pairs_total / value,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": workload, "n": n, "side": side, "parallelism": f"cpu{cb['cores']}"},
                "cpu_baseline": dict(cb, value=value),
                "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import torch
    import torch.distributed as dist
    from paper_2009_04755_b200 import _lib, device
    from paper_2009_04755_b200.engine import gather_triangle

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if world > 1:
            dist.barrier()

    parsed_bytes = side * side * 4
    items = torch.empty(n * side * side, dtype=torch.float32, device="cuda")
    device.synth_prnu(side, side, 0, n, args.cameras, args.seed, items)
    params = _lib.app_params(_lib.APP_PCE, n, height=side, width=side, threshold=60.0)
    # N > 1: peer-GPU tier -- each rank preprocesses its home items (k % N == rank),
    # every other item it needs is copied from its home GPU over NVLink (CUDA IPC)
    peer = world > 1
    # and ranks take leaf chunks from device work-queue words, stealing across GPUs
    steal = peer and not args.no_steal
    eng = device.DeviceEngine(params, leaf_block=args.leaf, device_slots=n, rank=rank, world=world,
                              device=local_rank, peer_tier=peer, steal=steal)
    out = torch.zeros(pairs_total, dtype=torch.float64, device="cuda")
    flags = torch.zeros(pairs_total, dtype=torch.uint8, device="cuda")
    estream = torch.cuda.ExternalStream(eng.stream())
    torch.cuda.synchronize()

    class _At:   # pointer view at a byte offset (the C ABI only needs data_ptr())
        def __init__(self, t, off):
            self.t, self.off = t, off

        def data_ptr(self):
            return self.t.data_ptr() + self.off

    state = {"connected": False}

    def step(host_home=None, host_all=None):
        """One full job on this rank: [home preprocess + barrier] + all of its pairs [+ barrier]."""
        if peer:
            if host_home is not None:
                eng.load_home(host_items=host_home, parsed_stride=parsed_bytes)
            else:
                eng.load_home(device_items=_At(items, rank * parsed_bytes), parsed_stride=world * parsed_bytes)
            if not state["connected"]:
                eng.connect_peers()
                state["connected"] = True
            if steal:
                eng.queue_reset()
            barrier()
            eng.run(out, flags, host_items=host_home, device_items=None if host_home is not None else items,
                    parsed_stride=parsed_bytes)
            barrier()
        elif host_all is not None:
            eng.run(out, flags, host_items=host_all, parsed_stride=parsed_bytes)
        else:
            eng.run(out, flags, device_items=items, parsed_stride=parsed_bytes)

    for _ in range(args.warmup):
        step()
    eng.reset_stats()
    eng.set_profiling(every=3, max_samples=4096)
    clocks = ClockSampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(estream)
    kms, ksamples, kpairs = 0.0, 0, 0
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
    eng.set_profiling(0)
    # cache accounting over the whole job (runner.py:41 R = loads / n; slotcache.py:252-260 tiers)
    ct = torch.tensor([st["loads"], st["hits"], st["misses"], st["peer_fetches"], st["steals"]],
                      dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ct, op=dist.ReduceOp.SUM)
    loads_all, hits_all, misses_all, peer_all, steals_all = [float(x) / max(1, args.steps) for x in ct.tolist()]

    # ---- e2e: pinned host patterns -> engine -> packed triangle back on host
    e2e = None
    if not args.no_e2e:
        try:
            if peer:
                # a rank needs only its home items on the host (every other item comes over NVLink)
                host = torch.empty((len(range(rank, n, world)), side * side), dtype=torch.float32, pin_memory=True)
                host.copy_(items.view(n, side * side)[rank::world])
                host_home, host_all = host, None
            else:
                host = torch.empty(n * side * side, dtype=torch.float32, pin_memory=True)
                host.copy_(items)
                host_home, host_all = None, host
            res_host = torch.empty(pairs_total, dtype=torch.float64, pin_memory=True)
            del items
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
                step(host_home=host_home, host_all=host_all)
                gather_triangle(out, flags)            # disjoint pair ids: exact gather to rank 0
                res_host.copy_(out, non_blocking=True)
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
                   "d2h_bytes_per_step": pairs_total * 8,
                   "peer_bytes_per_step": int(st2.get("peer_bytes", 0) // max(1, args.steps))}
        except RuntimeError as exc:  # e.g. pinned-memory exhaustion
            e2e = {"value": None, "unit": "pairs/s", "error": str(exc)[:200]}

    if args.trace_dir:
        # one extra (untimed) step with trace events: the reference's trace JSONL per
        # rank and its RunMetrics document (metrics.py) with the perf-model efficiency
        from paper_2009_04755_b200 import metrics as rk_metrics
        from paper_2009_04755_b200 import perfmodel
        os.makedirs(args.trace_dir, exist_ok=True)
        eng.set_trace(200000)
        eng.reset_stats()
        step()
        ev = eng.trace(node=rank)
        eng.set_trace(0)
        rk_metrics.write_trace(os.path.join(args.trace_dir, f"trace_rank{rank}.jsonl"), ev)
        span = (max(e["end_ns"] for e in ev) - min(e["start_ns"] for e in ev)) / 1e9 if ev else 0.0
        node = rk_metrics.node_metrics(rank, eng.stats(), span, n, ev)
        comp = [e for e in ev if e["label"] == "compare"]
        pre = [e for e in ev if e["label"] == "preprocess"]
        t_cmp = sum(e["end_ns"] - e["start_ns"] for e in comp) / 1e9 / max(1, sum(e["count"] for e in comp))
        t_pre = sum(e["end_ns"] - e["start_ns"] for e in pre) / 1e9 / max(1, sum(e["count"] for e in pre))
        nodes = [(node, span, t_cmp, t_pre)]
        if world > 1:
            nodes = [None] * world
            dist.all_gather_object(nodes, (node, span, t_cmp, t_pre))
        if rank == 0:
            costs = perfmodel.StageCosts(t_preprocess=max(x[3] for x in nodes), t_comparison=max(x[2] for x in nodes))
            doc = rk_metrics.run_metrics({"workload": workload, "n": n, "side": side, "leaf_block": args.leaf,
                                          "world": world}, n, [x[0] for x in nodes], max(x[1] for x in nodes),
                                         costs=costs)
            rk_metrics.write_metrics(os.path.join(args.trace_dir, "metrics.json"), doc)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks, peaks_src = load_peaks()
    hbm = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    slot_bytes = side * side * 4
    alg_bytes_per_pair = 2 * slot_bytes          # two half-spectra per pair
    roofline = None
    traffic = None
    try:   # dram bytes of one pce_cluster launch from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "pce_cluster_traffic.json")) as fh:
            tj = json.load(fh)
        traffic_per_pair = (tj["dram_bytes_read_per_launch"] + tj["dram_bytes_write_per_launch"]) / tj["pairs_per_launch"]
        if tj.get("side", 1024) != side:
            traffic_per_pair = None      # the capture is for another pattern size
    except Exception:
        traffic_per_pair = None
    if ksamples:
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
                    "pairs_per_launch": batch, "ms_per_launch": per_launch_ms,
                    "alg_bytes_per_pair": alg_bytes_per_pair, "peak_source": peaks_src,
                    "fp32_flops_per_pair": 2 * 5 * (side // 2) * side * math.log2(side)}

    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline(n, side, args.cameras, args.seed, args.cpu_seconds)

    line = {"metric": metric, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": {"workload": workload, "n": n, "side": side, "pairs": pairs_total, "leaf_block": args.leaf,
                       "parallelism": f"pairs{world}", "l2": f"inputs ({2 * n * slot_bytes / 2**30:.0f} GiB patterns + spectra) >> L2 (126 MB)"},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
            "gpu_launches": st["kernel_launches"],
            "cache": {"R": loads_all / n, "loads_per_step": loads_all,
                      "device_hit_rate": hits_all / max(1.0, hits_all + misses_all),
                      "device_hits_per_step": hits_all, "device_misses_per_step": misses_all,
                      "peer_fetches_per_step": peer_all,
                      "peer_hit_rate": peer_all / max(1.0, misses_all) if world > 1 else None,
                      "steals_per_step": steals_all if world > 1 else None}}
    print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
