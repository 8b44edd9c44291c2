"""BASELINE configs[2] (C3): PCE all-pairs over N = 16,384 patterns of 2048^2 fp32
(256 GiB, more than one GPU's HBM) on the GPUs of one box.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \\
      --master-port 29600 tools/c3_run.py [--items 16384] [--side 2048] [--slots 4500]

Each rank generates only its home patterns (k % world == rank: 64 GiB at 4
GPUs, 32 GiB at 8), 256 at a time, preprocesses them into its home region
(rk_engine_load_home_range), then runs its share of the quadtree leaves through the cross-GPU work
queue (stealing on), fetching every other item from its home GPU over NVLink
into its device slot tier.  Reported (one JSON line, rank 0):

  job_s          max over ranks of (home preprocess + all-pairs run), CUDA events / sync'd wall
  pairs_per_s    C(n,2) / job_s
  efficiency     the Rocket performance model (perfmodel.py:99-114): (T_min / p) / T with
                 T_min = n t_pre + C(n,2) t_cmp, t_pre = home-preprocess time per item and
                 t_cmp = sampled compare-launch time per pair, both measured in this run
  cache          R = loads / n (home preprocesses + reloads), device hit rate, peer fetches, bytes, steals
  p2p_gbs        the peer-tier D2D copy bandwidth (rank 0 <- rank 1), vs ~900 GB/s NVLink 5
  check          sampled pairs recomputed on rank 0 by the single-GPU path (bit-exact)
                 and every flag in {1, 3} (each pair written exactly once)
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2009_04755_b200 import _lib, device  # noqa: E402
from paper_2009_04755_b200.engine import gather_triangle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--items", type=int, default=16384)
    ap.add_argument("--side", type=int, default=2048)
    ap.add_argument("--slots", type=int, default=4500, help="device cache slots per GPU (besides the home region)")
    ap.add_argument("--leaf", type=int, default=8)
    ap.add_argument("--cameras", type=int, default=256)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--samples", type=int, default=8)
    ap.add_argument("--no-steal", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    n, side = args.items, args.side
    ss = side * side
    pairs_total = n * (n - 1) // 2

    params = _lib.app_params(_lib.APP_PCE, n, height=side, width=side, threshold=60.0)
    eng = device.DeviceEngine(params, leaf_block=args.leaf, device_slots=args.slots, rank=rank, world=world,
                              device=local_rank, peer_tier=world > 1, steal=world > 1 and not args.no_steal)
    out = torch.zeros(pairs_total, dtype=torch.float64, device="cuda")
    flags = torch.zeros(pairs_total, dtype=torch.uint8, device="cuda")

    # home patterns only, generated chunk by chunk (the load stage: generation untimed),
    # each chunk preprocessed into the home region (synchronous, timed)
    home = list(range(rank, n, world))
    chunk = 256
    raw = torch.empty(chunk * ss, dtype=torch.float32, device="cuda")
    dist.barrier()
    t_home = 0.0
    for m0 in range(0, len(home), chunk):
        cnt = min(chunk, len(home) - m0)
        for q in range(cnt):
            device.synth_prnu(side, side, home[m0 + q], 1, args.cameras, args.seed, raw.narrow(0, q * ss, ss))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.load_home_range(m0, cnt, device_items=raw, parsed_stride=ss * 4)
        t_home += time.perf_counter() - t0
    del raw
    torch.cuda.empty_cache()
    eng.connect_peers()
    if eng.steal:
        eng.queue_reset()
    dist.barrier()

    free, total = torch.cuda.mem_get_info()
    mem_used = total - free   # engine arena (cache + home slots) + result triangle + scratch
    eng.reset_stats()
    eng.set_profiling(every=8, max_samples=8192)
    estream = torch.cuda.ExternalStream(eng.stream())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(estream)
    eng.run(out, flags, parsed_stride=ss * 4)
    ev1.record(estream)
    torch.cuda.synchronize()
    t_run = ev0.elapsed_time(ev1) / 1e3
    kms, ksamples, kpairs = eng.kernel_time()
    st = eng.stats()
    dist.barrier()

    p2p = None
    if world > 1 and rank == 0:
        p2p = eng.peer_bandwidth(1, 64 * ss * 4)

    # cross-rank reductions
    t = torch.tensor([t_home + t_run, t_home, t_run], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    c = torch.tensor([st["loads"] + len(home), st["hits"], st["misses"], st["peer_fetches"], st["peer_bytes"], st["steals"],
                      st["pairs_done"], t_home / max(1, len(home)), kms / max(1, kpairs)],
                     dtype=torch.float64, device="cuda")
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    per_rank_pairs = torch.tensor([float(st["pairs_done"])], dtype=torch.float64, device="cuda")
    gathered = [torch.zeros_like(per_rank_pairs) for _ in range(world)]
    dist.all_gather(gathered, per_rank_pairs)

    tg0 = time.perf_counter()
    gather_triangle(out, flags)
    torch.cuda.synchronize()
    t_gather = time.perf_counter() - tg0

    if rank == 0:
        job_s, home_s, run_s = t.tolist()
        loads, hits, misses, fetches, fbytes, steals, pairs_done, tpre_sum, tcmp_ms_sum = c.tolist()
        t_pre = tpre_sum / world
        t_cmp = tcmp_ms_sum / world / 1e3
        t_min = n * t_pre + pairs_total * t_cmp
        # coverage: every pair written exactly once
        ok_flags = bool(((flags == 1) | (flags == 3)).all().item())
        # bit-exact recompute of sampled pairs by the single-GPU path
        g = torch.Generator().manual_seed(args.seed)
        sample = []
        while len(sample) < args.samples:
            i, j = sorted(torch.randint(0, n, (2,), generator=g).tolist())
            if i != j:
                sample.append((i, j))
        app = device.DeviceApp(params)
        items = torch.empty(2 * ss, dtype=torch.float32, device="cuda")
        slots = app.alloc_slots(2)
        ref = torch.zeros(pairs_total, dtype=torch.float64, device="cuda")
        mism = 0
        for (i, j) in sample:
            device.synth_prnu(side, side, i, 1, args.cameras, args.seed, items.narrow(0, 0, ss))
            device.synth_prnu(side, side, j, 1, args.cameras, args.seed, items.narrow(0, ss, ss))
            app.preprocess(items, ss * 4, 2, slots, [0, 1])
            app.compare_pairs(slots, [(i, j, 0, 1)], ref)
            torch.cuda.synchronize()
            pid = i * (2 * n - i - 1) // 2 + (j - i - 1)
            if ref[pid].item() != out[pid].item():
                mism += 1
        line = {
            "workload": f"PRNU PCE all-pairs, N={n} patterns of {side}x{side} fp32 (BASELINE configs[2])",
            "n_gpus": world, "pairs": pairs_total, "job_s": job_s, "home_preprocess_s": home_s, "run_s": run_s,
            "gather_s": t_gather, "pairs_per_s": pairs_total / job_s,
            "perf_model": {"t_pre_s": t_pre, "t_cmp_s": t_cmp, "T_min_s": t_min, "p": world,
                           "efficiency": (t_min / world) / job_s},
            "cache": {"device_slots_per_gpu": args.slots, "R": loads / n,
                      "device_hit_rate": hits / max(1.0, hits + misses), "peer_fetches": fetches,
                      "peer_gib": fbytes / 2**30, "steals": steals,
                      "pairs_per_rank": [float(x.item()) for x in gathered]},
            "p2p_gbs": p2p, "check": {"flags_all_written_once": ok_flags, "sampled_pairs": len(sample),
                                      "bit_exact_mismatches": mism},
            "hbm_used_gib_rank0": mem_used / 2**30,
        }
        print(json.dumps(line), flush=True)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
