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


def _queue_worker(rank, world, port, n, leaf, chunk, words, lock, ret):
    """One rank of the cross-GPU work queue, on CPU: the queue words live in shared
    memory and the lock stands in for atomicCAS_system; every transition is the
    product's own rk_queue_step, the take / steal policy mirrors rk_engine_run
    (own head chunks, then the back half of the fullest peer, re-published as
    this rank's range).  Rank 0 is slow, so the others must steal from it."""
    import ctypes as C
    import time
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_04755_b200._lib import lib
        from paper_2009_04755_b200.engine import rank_leaves
        lo = sum(len(rank_leaves(n, leaf, r, world)) for r in range(rank))
        hi = lo + len(rank_leaves(n, leaf, rank, world))
        words[rank] = (lo << 32) | hi                  # rk_engine_queue_reset
        dist.barrier()

        def cas_op(v, op, arg):
            nw, got = C.c_uint64(), C.c_uint64()
            with lock:                                  # atomicCAS_system on the word
                st = lib.rk_queue_step(words[v], op, arg, C.byref(nw), C.byref(got))
                if st == 1:
                    words[v] = nw.value
            return got.value if st == 1 else None

        done, steals = [], 0
        while True:
            got = cas_op(rank, 0, chunk)
            while got is None:
                rem = [((words[v] & 0xFFFFFFFF) - (words[v] >> 32)) if v != rank else -1 for v in range(world)]
                best = max(range(world), key=lambda v: rem[v])
                if rem[best] < 2 * chunk:
                    break
                st = cas_op(best, 1, chunk)
                if st is None:
                    continue                            # lost the race: look again
                steals += 1
                with lock:
                    words[rank] = st                    # the stolen range is ours (and stealable)
                got = cas_op(rank, 0, chunk)
            if got is None:
                break
            done.extend(range(got >> 32, got & 0xFFFFFFFF))
            if rank == 0:
                time.sleep(0.02)                        # a slow GPU
        dist.barrier()
        ret.put((rank, done, steals))
    finally:
        dist.destroy_process_group()


def test_work_queue_steals_cover_every_leaf_once():
    import ctypes as C
    from paper_2009_04755_b200._lib import lib
    from paper_2009_04755_b200.engine import rank_leaves
    # the transition itself: owner head chunks, thief back halves, nothing from an empty word
    nw, got = C.c_uint64(), C.c_uint64()
    assert lib.rk_queue_step((10 << 32) | 30, 0, 4, C.byref(nw), C.byref(got)) == 1
    assert (got.value >> 32, got.value & 0xFFFFFFFF, nw.value >> 32) == (10, 14, 14)
    assert lib.rk_queue_step((10 << 32) | 30, 1, 4, C.byref(nw), C.byref(got)) == 1
    assert (got.value >> 32, got.value & 0xFFFFFFFF, nw.value & 0xFFFFFFFF) == (20, 30, 20)
    assert lib.rk_queue_step((10 << 32) | 15, 1, 4, C.byref(nw), C.byref(got)) == 0
    assert lib.rk_queue_step((7 << 32) | 7, 0, 4, C.byref(nw), C.byref(got)) == 0
    world, n, leaf, chunk = 3, 64, 4, 2
    total = sum(len(rank_leaves(n, leaf, r, world)) for r in range(world))
    ctx = mp.get_context("spawn")
    words = ctx.Array(C.c_uint64, world, lock=False)
    lock = ctx.Lock()
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_queue_worker, args=(r, world, port, n, leaf, chunk, words, lock, ret))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([ret.get(timeout=180) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    done = sorted(i for _, d, _ in outs for i in d)
    assert done == list(range(total))                   # every leaf exactly once
    assert outs[1][2] + outs[2][2] >= 1                 # the fast ranks stole from the slow one
    assert len(outs[0][1]) < max(len(outs[1][1]), len(outs[2][1]))   # the slow rank did least
