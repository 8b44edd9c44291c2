"""Peer-tier copy bandwidth over NVLink (rank 0 <- rank 1), per copy mechanism.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_bw.py

The copy is the engine's own (rk_engine_peer_bandwidth): for an NCC engine one
block copy per call, by the copy engine (RK_PEER_COPY_CTAS=0, cudaMemcpyAsync) or
by an SM-driven copy kernel with RK_PEER_COPY_CTAS CTAs; for a PCE engine the
slot-sized cudaMemcpyAsync pieces of a peer fetch.  Prints one JSON line (rank 0).
NVLink 5 is ~900 GB/s per direction per GPU.
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def nvlink_counters(gpu: int):
    """Summed NVLink data Tx / Rx KiB counters of one GPU (nvidia-smi nvlink -gt d), or None."""
    import re
    import subprocess
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(gpu)], capture_output=True, text=True,
                             timeout=30).stdout
    except Exception:
        return None
    tx = sum(int(x) for x in re.findall(r"Tx:\s*(\d+)\s*KiB", out))
    rx = sum(int(x) for x in re.findall(r"Rx:\s*(\d+)\s*KiB", out))
    return {"tx_kib": tx, "rx_kib": rx, "links": len(re.findall(r"Link \d+", out)) // 2 or None, "raw": out[:600]}


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2009_04755_b200 import _lib, device
    side, n = 1024, 2048
    res = {"world": world}
    for kind in ("ncc", "pce"):
        appk = _lib.APP_NCC if kind == "ncc" else _lib.APP_PCE
        params = _lib.app_params(appk, n, height=side, width=side)
        eng = device.DeviceEngine(params, device_slots=1024, rank=rank, world=world, device=local, peer_tier=True)
        items = torch.empty((len(range(rank, n, world)), side * side), dtype=torch.float32, device="cuda")
        for q, k in enumerate(range(rank, n, world)):
            device.synth_prnu(side, side, k, 1, 8, 3, items[q])
        eng.load_home(device_items=items, parsed_stride=side * side * 4)
        eng.connect_peers()
        dist.barrier()
        if rank == 0:
            nbytes = 1024 * side * side * 4        # 4 GiB: one 1,024-item block
            variants = [0, 16, 32, 64, 148, 296] if kind == "ncc" else [0]
            for ctas in variants:
                os.environ["RK_PEER_COPY_CTAS"] = str(ctas)
                eng.peer_bandwidth(1, nbytes)      # warm
                c0 = nvlink_counters(local)
                res[f"{kind}_ctas{ctas}_gbs"] = max(eng.peer_bandwidth(1, nbytes) for _ in range(3))
                c1 = nvlink_counters(local)
                res.setdefault("nvlink_raw_sample", (c1 or {}).get("raw"))
                if c0 and c1:
                    # rank 0 reads rank 1's home region: the bytes arrive on rank 0's links (Rx)
                    res[f"{kind}_ctas{ctas}_nvlink"] = {"rx_gib": (c1["rx_kib"] - c0["rx_kib"]) / 2**20,
                                                        "tx_gib": (c1["tx_kib"] - c0["tx_kib"]) / 2**20,
                                                        "copied_gib": 3 * nbytes / 2**30, "links": c1["links"]}
            os.environ.pop("RK_PEER_COPY_CTAS", None)
        dist.barrier()
        eng.close()
        del items
        torch.cuda.empty_cache()
        dist.barrier()
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
