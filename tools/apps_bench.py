"""Throughput of the irregular apps at their BASELINE configs on one B200.

  python tools/apps_bench.py gmm [--items 1000] [--angles 36]     # configs[3] (C4)
  python tools/apps_bench.py cv  [--items 2500] [--mean-nnz 500000] # configs[4] (C5)
  (multi-GPU: python -m torch.distributed.run --nproc-per-node N ... tools/apps_bench.py cv)

GMM: N particles of ~300 localizations (synthdata.particle), max over K
rotations of the Gaussian-overlap cost; bound = SFU exponentials, K*m_i*m_j per
pair, against 148 SMs x 16 ex2/clk x clock.
CV: N sparse k-mer composition vectors with log-normally skewed nnz in
[1e5, 1.8e6], generated directly in the reference's parsed byte
format (<I dim> + dim x <Q token><I count>); bound = HBM, 16*(nnz_i + nnz_j)
bytes per pair.  Items are HBM-resident before the timed region; one step = the
whole all-pairs job through the C++ engine (preprocess + every pair).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2009_04755_b200 import _lib, device  # noqa: E402


def run_engine(params, parsed, stride: int, n: int, leaf: int, steps: int, warmup: int):
    """One job per step; under torchrun every rank holds all parsed items, owns its
    home items (peer tier) and takes leaf chunks from the cross-GPU work queue."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    items = parsed if isinstance(parsed, torch.Tensor) else torch.from_numpy(parsed).cuda()
    multi = world > 1
    eng = device.DeviceEngine(params, leaf_block=leaf, device_slots=n, rank=rank, world=world,
                              device=torch.cuda.current_device(), peer_tier=multi, steal=multi)
    total = n * (n - 1) // 2
    out = torch.zeros(total, dtype=torch.float64, device="cuda")
    estream = torch.cuda.ExternalStream(eng.stream())

    class _At:
        def __init__(self, off):
            self.off = off

        def data_ptr(self):
            return items.data_ptr() + self.off

    connected = [False]

    def step():
        if multi:
            eng.load_home(device_items=_At(rank * stride), parsed_stride=world * stride)
            if not connected[0]:
                eng.connect_peers()
                connected[0] = True
            eng.queue_reset()
            dist.barrier()
        eng.run(out, device_items=items, parsed_stride=stride)
        if multi:
            dist.barrier()

    for _ in range(warmup):
        step()
    eng.reset_stats()
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(estream)
    for _ in range(steps):
        step()
    e1.record(estream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    st = eng.stats()
    if multi:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        c = torch.tensor([st["pairs_done"], st["steals"], st["peer_fetches"]], dtype=torch.float64, device="cuda")
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        st = dict(st, pairs_done=int(c[0].item()) // steps, steals=int(c[1].item()),
                  peer_fetches=int(c[2].item()))
    eng.close()
    return ms, st, out


def bench_gmm(args):
    from paper_2009_04755_b200.synthdata import gmm_parsed
    n, maxp = args.items, 400
    stride = 8 + 12 * maxp
    host, msum = gmm_parsed(n, args.seed, maxp)
    params = _lib.app_params(_lib.APP_GMM, n, max_entries=maxp, gmm_angles=args.angles)
    ms, st, _ = run_engine(params, host.reshape(-1), stride, n, args.leaf, args.steps, args.warmup)
    pairs = n * (n - 1) // 2
    exps = args.angles * (msum.sum() ** 2 - (msum ** 2).sum()) / 2.0
    clk_ghz = args.clock_ghz
    sfu_peak = 148 * 16 * clk_ghz * 1e9 * int(os.environ.get("WORLD_SIZE", "1"))   # whole box
    return {"app": "gmm", "workload": f"particle fusion, N={n} particles of ~300 localizations, K={args.angles} "
                                      f"rotations (BASELINE configs[3])",
            "pairs": pairs, "ms_per_job": ms, "pairs_per_s": pairs / (ms / 1e3),
            "roofline": {"bound": "sfu", "achieved_exp_per_s": exps / (ms / 1e3), "peak_exp_per_s": sfu_peak,
                         "frac": exps / (ms / 1e3) / sfu_peak, "exps_per_job": exps,
                         "peak_source": f"148 SMs x 16 ex2/clk x {clk_ghz} GHz"},
            "launches": st["kernel_launches"]}


def cv_items(n: int, mean_nnz: float, seed: int):
    from paper_2009_04755_b200.synthdata import cv_parsed_device
    return cv_parsed_device(n, mean_nnz, seed)


def bench_cv(args):
    n = args.items
    buf, stride, cap, nnz = cv_items(n, args.mean_nnz, args.seed)
    params = _lib.app_params(_lib.APP_CV, n, max_entries=cap, threshold=0.5)
    ms, st, _ = run_engine(params, buf, stride, n, args.leaf, args.steps, args.warmup)
    pairs = n * (n - 1) // 2
    alg = 16.0 * (n - 1) * nnz.sum()        # sum over pairs of 16 (nnz_i + nnz_j)
    hbm = 6544.3
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            hbm = float(json.load(fh).get("hbm_gbs", hbm))
    except Exception:
        pass
    hbm *= int(os.environ.get("WORLD_SIZE", "1"))   # whole box
    return {"app": "cv", "workload": f"composition-vector cosine, N={n} items, nnz lognormal in [1e5, 1.8e6] "
                                     f"(mean {nnz.mean():.0f}, max {nnz.max()}) (BASELINE configs[4])",
            "pairs": pairs, "ms_per_job": ms, "pairs_per_s": pairs / (ms / 1e3),
            "roofline": {"bound": "hbm", "achieved_gbs": alg / (ms / 1e3) / 1e9, "peak_gbs": hbm,
                         "frac": alg / (ms / 1e3) / 1e9 / hbm, "alg_bytes_per_job": alg},
            "launches": st["kernel_launches"], "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
            "steals": st.get("steals"), "peer_fetches": st.get("peer_fetches")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("app", choices=["gmm", "cv"])
    ap.add_argument("--items", type=int, default=0)
    ap.add_argument("--angles", type=int, default=36)
    ap.add_argument("--mean-nnz", type=float, default=5e5)
    ap.add_argument("--leaf", type=int, default=16)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--clock-ghz", type=float, default=1.965)
    args = ap.parse_args()
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist
        lr = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(lr)
        dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    rank0 = int(os.environ.get("RANK", "0")) == 0
    if args.app == "gmm":
        args.items = args.items or 1000
        line = bench_gmm(args)
    else:
        args.items = args.items or 2500
        line = bench_cv(args)
    if rank0:
        print(json.dumps(line), flush=True)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
