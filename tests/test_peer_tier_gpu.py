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


def _rank(rank, world, port, ret):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_04755_b200.apps import PCEApp
        from paper_2009_04755_b200.engine import AllPairsEngine
        app = PCEApp(26, side=256, cameras=3, seed=17, device=0)
        eng = AllPairsEngine(app, leaf_block=4, device_slots=10, rank=rank, world=world, peer_tier=True)
        res = eng.run(gather=False)
        ret.put((rank, res.values.copy(), res.flags.copy(), res.stats))
        eng.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_peer_fetch_match_oracle():
    import torch.multiprocessing as mp
    from oracle import pce as opce
    from paper_2009_04755_b200.apps import PCEApp
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, ret)) for r in range(2)]
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
