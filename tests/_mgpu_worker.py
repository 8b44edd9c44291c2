"""torchrun worker for tests/test_multigpu_gpu.py (not collected by pytest: leading underscore).

Every rank runs its share of a PCE and a CV all-pairs job (peer tier + work
stealing, NCCL reduce to rank 0); rank 0 recomputes both jobs alone on its GPU
and compares bit for bit, and checks PCE against the float64 oracle."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2009_04755_b200 import _lib, device, synthdata
    from paper_2009_04755_b200.apps import PCEApp
    from paper_2009_04755_b200.engine import AllPairsEngine, gather_triangle
    report = {"world": world}

    # PCE through the public engine (leaf 4, tight slot tier, chunks of 1 leaf: steals happen)
    n, side = 40, 256
    app = PCEApp(n, side=side, cameras=4, seed=21, device=local)
    eng = AllPairsEngine(app, leaf_block=4, device_slots=12, rank=rank, world=world, steal_chunk=1)
    res = eng.run()
    tot = torch.tensor([res.stats["pairs_done"], res.stats["steals"], res.stats["peer_fetches"]],
                       dtype=torch.int64, device="cuda")
    dist.all_reduce(tot)
    eng.close()

    # CV (variable-length items) through the device engine, same sharing machinery
    m = 24
    buf, stride, cap, _ = synthdata.cv_parsed_device(m, 1.2e5, 3)
    params = _lib.app_params(_lib.APP_CV, m, max_entries=cap, threshold=0.5)
    ce = device.DeviceEngine(params, leaf_block=4, device_slots=m, rank=rank, world=world, device=local,
                             peer_tier=True, steal=True, steal_chunk=1)

    class _At:
        def __init__(self, off):
            self.off = off

        def data_ptr(self):
            return buf.data_ptr() + self.off

    ce.load_home(device_items=_At(rank * stride), parsed_stride=world * stride)
    ce.connect_peers()
    ce.queue_reset()
    ce.ledger_reset()
    dist.barrier()
    cv_out = torch.zeros(m * (m - 1) // 2, dtype=torch.float64, device="cuda")
    cv_flags = torch.zeros_like(cv_out, dtype=torch.uint8)
    ce.run(cv_out, cv_flags, device_items=buf, parsed_stride=stride)
    dist.barrier()
    cv_ledger = ce.check_ledger() if rank == 0 else None
    gather_triangle(cv_out, cv_flags)
    ce.close()

    if rank == 0:
        from oracle import pce as opce
        pats = np.stack([np.frombuffer(app.fetch_raw(app.path_for_key(k)), dtype=np.float32).reshape(side, side)
                         for k in range(n)])
        want = opce.all_pairs(pats)
        solo_app = PCEApp(n, side=side, cameras=4, seed=21, device=local)
        solo = AllPairsEngine(solo_app, leaf_block=4, device_slots=12)
        ref = solo.run()
        solo.close()
        cv_solo = torch.zeros_like(cv_out)
        se = device.DeviceEngine(params, leaf_block=4, device_slots=m, device=local)
        se.run(cv_solo, device_items=buf, parsed_stride=stride)
        se.close()
        report.update({
            "pce_pairs": int(tot[0].item()), "steals": int(tot[1].item()), "peer_fetches": int(tot[2].item()),
            "pce_max_rel_err": float(np.max(np.abs(res.values - want) / np.abs(want))),
            "pce_bit_exact_vs_1gpu": bool(np.array_equal(res.values, ref.values)),
            "pce_flags_once": bool(np.all((res.flags == 1) | (res.flags == 3))),
            "cv_bit_exact_vs_1gpu": bool(torch.equal(cv_out, cv_solo)),
            "cv_flags_once": bool(((cv_flags == 1) | (cv_flags == 3)).all().item()),
            "pce_ledger_full": bool(res.ledger["full"]), "cv_ledger_full": bool(cv_ledger["full"]),
        })
        print("MGPU_REPORT " + json.dumps(report), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
