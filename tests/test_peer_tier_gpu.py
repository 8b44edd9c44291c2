"""Peer-GPU cache tier with two ranks sharing cuda:0 (CUDA IPC across processes,
gloo for the host-side handshake): each rank preprocesses only its home items
(k % 2 == rank) and fetches the other half from its peer's home region."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, ret, steal_chunk=0, delay0=0.0, n=26, side=256, slots=10):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_04755_b200.apps import PCEApp
        from paper_2009_04755_b200.engine import AllPairsEngine
        app = PCEApp(n, side=side, cameras=3, seed=17, device=0)
        eng = AllPairsEngine(app, leaf_block=4, device_slots=slots, rank=rank, world=world, peer_tier=True,
                             steal_chunk=steal_chunk)
        if rank == 0 and delay0 > 0:
            # rank 0 starts late (after the barrier): rank 1 runs dry and steals from it
            import time
            inner = eng._eng.run

            def late_run(*a, **kw):
                time.sleep(delay0)
                return inner(*a, **kw)
            eng._eng.run = late_run
        res = eng.run(gather=False)
        ret.put((rank, res.values.copy(), res.flags.copy(), dict(res.stats, ledger=res.ledger)))
        eng.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("steal_chunk,delay0", [(0, 0.0), (1, 3.0)])
def test_two_ranks_peer_fetch_match_oracle(steal_chunk, delay0):
    """Exactly-once coverage and oracle parity with the peer tier and the cross-GPU
    work queue; the second case delays rank 0 so rank 1 must steal from it."""
    import torch.multiprocessing as mp
    from oracle import pce as opce
    from paper_2009_04755_b200.apps import PCEApp
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, ret, steal_chunk, delay0)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([ret.get(timeout=300) for _ in range(2)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    values = outs[0][1] + outs[1][1]          # disjoint pair ids
    flags = outs[0][2] + outs[1][2]
    app = PCEApp(26, side=256, cameras=3, seed=17)
    pats = np.stack([np.frombuffer(app.fetch_raw(app.path_for_key(k)), dtype=np.float32).reshape(256, 256)
                     for k in range(26)])
    np.testing.assert_allclose(values, opce.all_pairs(pats), rtol=1e-4)
    assert set(np.unique(flags)) <= {1, 3}                      # every pair written exactly once
    for rank, _, _, st in outs:
        assert st["loads"] == 13                                 # only home items preprocessed: R = 1
        assert st["peer_fetches"] > 0 and st["peer_bytes"] == st["peer_fetches"] * 256 * 256 * 4
    assert outs[0][3]["pairs_done"] + outs[1][3]["pairs_done"] == 26 * 25 // 2
    led = outs[0][3]["ledger"]                                   # the job's shared ledger, on rank 0
    assert led["full"] == 1 and led["completed"] == 26 * 25 // 2 and led["dup_marks"] == 0
    if delay0 > 0:
        assert outs[1][3]["steals"] >= 1                         # the idle rank stole from the late one
        assert outs[1][3]["pairs_done"] > outs[0][3]["pairs_done"]


@pytest.mark.parametrize("world,n", [(3, 26), (8, 48)])
def test_ranks_steal_from_a_late_rank(world, n):
    """`world` ranks (IPC-shared cuda:0): rank 0 starts 3 s late, the others drain
    their shares and then steal from it -- and from each other's stolen ranges --
    while every pair is still computed exactly once (the shared device ledger on
    rank 0 and the summed flags agree) and matches the oracle.  world = 8 runs the
    8-GPU box's queue scan, 8 IPC mappings and the shared ledger on one GPU."""
    import torch.multiprocessing as mp
    from oracle import pce as opce
    from paper_2009_04755_b200.apps import PCEApp
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, ret, 1, 3.0, n)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([ret.get(timeout=600) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    total = n * (n - 1) // 2
    values = sum(o[1] for o in outs)
    flags = sum(o[2].astype(np.int32) for o in outs)
    app = PCEApp(n, side=256, cameras=3, seed=17)
    pats = np.stack([np.frombuffer(app.fetch_raw(app.path_for_key(k)), dtype=np.float32).reshape(256, 256)
                     for k in range(n)])
    np.testing.assert_allclose(values, opce.all_pairs(pats), rtol=1e-4)
    assert set(np.unique(flags)) <= {1, 3}
    assert sum(o[3]["pairs_done"] for o in outs) == total
    assert sum(o[3]["steals"] for o in outs[1:]) >= 1
    assert outs[0][3]["pairs_done"] < min(o[3]["pairs_done"] for o in outs[1:])
    assert sum(o[3]["loads"] for o in outs) == n                 # every item preprocessed once, on its home rank
    led = outs[0][3]["ledger"]
    assert led["full"] == 1 and led["completed"] == total and led["dup_marks"] == 0


def _ncc_rank(rank, world, port, ret, n, side, slots):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_04755_b200.apps import NCCApp
        from paper_2009_04755_b200.engine import AllPairsEngine
        app = NCCApp(n, side=side, cameras=4, seed=41, device=0)
        eng = AllPairsEngine(app, device_slots=slots, rank=rank, world=world)
        res = eng.run(gather=False)
        ret.put((rank, res.values.copy(), res.flags.copy(), dict(res.stats, ledger=res.ledger)))
        eng.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,side,slots", [(2, 600, 128, 256), (3, 700, 512, 256)])
def test_ncc_gram_over_the_peer_tier(world, n, side, slots):
    """NCC all-pairs through the public engine with the peer tier (ranks sharing
    cuda:0 over CUDA IPC): each rank normalises only its home items (k % world),
    cuts them into sub-blocks of half its cache arena, and multiplies its share of
    the sub-block pairs, copying every non-home partner from its owner's home
    region.  side 512 = two K chunks per block.  Every pair once (flags and the
    shared device ledger), TF32 Gram within 2e-4 of the float64 oracle."""
    import torch.multiprocessing as mp
    from oracle import ncc as oncc
    from paper_2009_04755_b200.apps import NCCApp
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ncc_rank, args=(r, world, port, ret, n, side, slots)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([ret.get(timeout=600) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    total = n * (n - 1) // 2
    values = sum(o[1] for o in outs)
    flags = sum(o[2].astype(np.int32) for o in outs)
    assert set(np.unique(flags)) <= {1, 3}
    app = NCCApp(n, side=side, cameras=4, seed=41)
    pats = np.stack([np.frombuffer(app.fetch_raw(app.path_for_key(k)), dtype=np.float32) for k in range(n)])
    assert np.max(np.abs(values - oncc.all_pairs_chunked(pats))) <= 2e-4
    assert sum(o[3]["pairs_done"] for o in outs) == total
    assert sum(o[3]["loads"] for o in outs) == n                  # home items only: R = 1
    assert all(o[3]["peer_fetches"] > 0 for o in outs)
    pairs = [o[3]["pairs_done"] for o in outs]
    assert max(pairs) <= 2 * min(pairs)                           # circulant share: balanced
    led = outs[0][3]["ledger"]
    assert led["full"] == 1 and led["completed"] == total and led["dup_marks"] == 0


def test_2048_peer_tier_two_ranks():
    """The C3 item size through the C3 path (pce2k_pair, home items k % 2, the rest
    fetched from the peer's home region, stealing on) with a device tier smaller
    than n, against the float64 oracle."""
    import torch.multiprocessing as mp
    from oracle import pce as opce
    from oracle import scheduler as osch
    from paper_2009_04755_b200.apps import PCEApp
    n, side, world = 12, 2048, 2
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, ret, 1, 0.0, n, side, 4)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([ret.get(timeout=600) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    total = n * (n - 1) // 2
    values = outs[0][1] + outs[1][1]
    flags = outs[0][2].astype(int) + outs[1][2].astype(int)
    assert set(np.unique(flags)) <= {1, 3}
    app = PCEApp(n, side=side, cameras=3, seed=17)
    pats = np.stack([np.frombuffer(app.fetch_raw(app.path_for_key(k)), dtype=np.float32).reshape(side, side)
                     for k in range(n)])
    want = opce.pairs_batched(pats, [osch.pair_from_id(n, p) for p in range(total)], batch=4)
    np.testing.assert_allclose(values, want, rtol=1e-4)
    assert sum(o[3]["loads"] for o in outs) == n and all(o[3]["peer_fetches"] > 0 for o in outs)
    led = outs[0][3]["ledger"]
    assert led["full"] == 1 and led["completed"] == total


def _chunk_rank(rank, world, port, ret, n, side):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_04755_b200 import device
        from paper_2009_04755_b200.apps import PCEApp
        from paper_2009_04755_b200.engine import AllPairsEngine
        app = PCEApp(n, side=side, cameras=3, seed=23, device=0)
        eng = AllPairsEngine(app, leaf_block=4, device_slots=6, rank=rank, world=world)
        buf = torch.empty(4 * side * side, dtype=torch.float32, device="cuda")

        def home_chunks(m0, count):   # this rank's home items, generated where they live (C3 style)
            for q in range(count):
                device.synth_prnu(side, side, rank + (m0 + q) * world, 1, 3, 23,
                                  buf[q * side * side:(q + 1) * side * side])
            return buf
        res = eng.run(gather=False, home_chunks=home_chunks, chunk=4)
        ret.put((rank, res.values.copy(), res.flags.copy(), dict(res.stats, ledger=res.ledger)))
        eng.close()
    finally:
        dist.destroy_process_group()


def test_public_api_home_chunks():
    """AllPairsEngine.run(home_chunks=...): no rank ever holds all items -- each
    generates its home items chunk by chunk where they live, the rest arrive over
    the peer tier (the C3 placement through the public API)."""
    import torch.multiprocessing as mp
    from oracle import pce as opce
    from paper_2009_04755_b200.apps import PCEApp
    n, side, world = 22, 256, 2
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_rank, args=(r, world, port, ret, n, side)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([ret.get(timeout=300) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    values = outs[0][1] + outs[1][1]
    app = PCEApp(n, side=side, cameras=3, seed=23)
    pats = np.stack([np.frombuffer(app.fetch_raw(app.path_for_key(k)), dtype=np.float32).reshape(side, side)
                     for k in range(n)])
    np.testing.assert_allclose(values, opce.all_pairs(pats), rtol=1e-4)
    assert sum(o[3]["loads"] for o in outs) == n
    assert outs[0][3]["ledger"]["full"] == 1
