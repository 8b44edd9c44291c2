"""torchrun multi-GPU parity check: every rank runs its share of a PCE all-pairs job,
the disjoint triangles are reduced onto rank 0 over NCCL, rank 0 checks the oracle.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/multi_gpu_check.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    from paper_2009_04755_b200.apps import PCEApp
    from paper_2009_04755_b200.engine import AllPairsEngine
    n, side = 48, 256
    app = PCEApp(n, side=side, cameras=4, seed=21, device=torch.cuda.current_device())
    eng = AllPairsEngine(app, leaf_block=4, device_slots=20, rank=rank, world=world)
    res = eng.run()
    done = torch.tensor([res.stats["pairs_done"]], dtype=torch.int64, device="cuda")
    dist.all_reduce(done)
    if rank == 0:
        from oracle import pce as opce
        pats = np.stack([np.frombuffer(app.fetch_raw(app.path_for_key(k)), dtype=np.float32).reshape(side, side)
                         for k in range(n)])
        want = opce.all_pairs(pats)
        err = float(np.max(np.abs(res.values - want) / np.abs(want)))
        ok = err <= 1e-4 and int(done.item()) == n * (n - 1) // 2 and np.all(res.flags > 0)
        print(f"world={world} pairs={int(done.item())} max_rel_err={err:.2e} stats={res.stats} -> {'OK' if ok else 'FAIL'}")
        if not ok:
            sys.exit(1)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
