"""World-size-2 gloo run of the multi-GPU host logic on CPU: each rank takes its
share of the quadtree leaves from the C++ scheduler, fills its pairs, and the
disjoint triangles are gathered with the same reduce the GPU path uses."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rng as orng


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, leaf, seed, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_04755_b200.engine import gather_triangle, rank_leaves
        vals = torch.zeros(n * (n - 1) // 2, dtype=torch.float64)
        flags = torch.zeros(n * (n - 1) // 2, dtype=torch.uint8)
        mine = 0
        for r0, r1, c0, c1 in rank_leaves(n, leaf, rank, world):
            for i in range(r0, r1):
                for j in range(max(c0, i + 1), c1):
                    pid = i * (2 * n - i - 1) // 2 + (j - i - 1)
                    vals[pid] = orng.synthetic_value(seed, i, j)
                    flags[pid] = 1
                    mine += 1
        counts = torch.tensor([mine], dtype=torch.int64)
        dist.all_reduce(counts)
        gather_triangle(vals, flags)
        if rank == 0:
            ret.put((vals.numpy().copy(), flags.numpy().copy(), int(counts.item()), mine))
        else:
            ret.put((None, None, int(counts.item()), mine))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_job_gathers_exact_triangle(world):
    n, leaf, seed = 61, 4, 13
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, leaf, seed, ret)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [ret.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = n * (n - 1) // 2
    full = [o for o in outs if o[0] is not None][0]
    vals, flags, count, _ = full
    assert count == total
    assert sorted(o[3] for o in outs) != [0, total]          # both ranks did work
    assert flags.tolist() == [1] * total                      # every pair exactly once
    want = [orng.synthetic_value(seed, i, j) for i in range(n) for j in range(i + 1, n)]
    assert vals.tolist() == want                              # bit-exact gather
