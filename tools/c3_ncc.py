"""C3-Gram NCC: zero-lag NCC of N = 16,384 items of 2048^2 fp32
(256 GiB; no GPU holds them all) as a blocked tcgen05 Gram over the GPUs of one box.

Round-1 standalone version over the C ABI (contiguous key blocks, serpentine
owners).  Since round 2 the engine itself runs this job over the peer tier
(`ncc_peer_run`; `bench.py --gpus N --app ncc --items 16384 --side 2048`,
`AllPairsEngine` with device_slots < n); this script is kept as the comparison
point quoted in DESIGN.md.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \\
      --master-port 29700 tools/c3_ncc.py [--items 16384] [--side 2048] [--block 2048]

Items are split into key blocks of `block` items; block b lives on GPU
owner(b) (serpentine over the ranks, so every rank gets the same triangle
work).  A rank computes the block pairs (I, J), I one of its home blocks and
J >= I: home J in place, other J copied from the owner's arena over NVLink (CUDA
IPC, double-buffered on a copy stream so the next block arrives while the
current one is multiplied).  Each block pair is one rk_ncc_gram_block call
(CTA-pair tcgen05 TF32 kernel, K-chunked); the pairs of one J with the
different home blocks run on their own streams, so together they fill the SMs.  The disjoint triangles are summed
onto rank 0 with one NCCL reduce.  Reported: Gram time (max over ranks, CUDA
events), pairs/s, TF32 TFLOP/s, bytes fetched, every pair written once, and
sampled pairs against the fp32 per-pair path (|diff| <= 2e-4).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2009_04755_b200 import _lib, device  # noqa: E402
from paper_2009_04755_b200._lib import check, lib  # noqa: E402
from paper_2009_04755_b200.engine import gather_triangle  # noqa: E402


class _Ptr:
    def __init__(self, p):
        self.p = p

    def data_ptr(self):
        return self.p


def owner(b: int, world: int) -> int:
    r, pos = divmod(b, world)
    return pos if r % 2 == 0 else world - 1 - pos


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--items", type=int, default=16384)
    ap.add_argument("--side", type=int, default=2048)
    ap.add_argument("--block", type=int, default=2048)
    ap.add_argument("--cameras", type=int, default=256)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--samples", type=int, default=16)
    ap.add_argument("--copy-streams", type=int, default=1,
                    help="concurrent D2D copies per block fetch (measured: 1: 0.676 s, 2: 0.711 s, 4: 0.707 s)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, side, bs = args.items, args.side, args.block
    d = side * side
    assert n % bs == 0 and bs % 256 == 0
    nblk = n // bs
    home = [b for b in range(nblk) if owner(b, world) == rank]
    row_of_home = {b: h * bs for h, b in enumerate(home)}
    fetch_rows = [(len(home) + f) * bs for f in range(2)]
    n_rows = (len(home) + 2) * bs

    app = device.DeviceApp(_lib.app_params(_lib.APP_NCC, n, height=side, width=side, threshold=0.02), device=local)
    stride = app.slot_stride
    arena_p = C.c_void_p()
    check(lib.rk_device_alloc(n_rows * stride, local, C.byref(arena_p)))
    arena = _Ptr(arena_p.value)

    # home items: generate (untimed load stage) and normalise into the home rows
    chunk = 128
    raw = torch.empty(chunk * d, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    t_pre = 0.0
    for b in home:
        for c0 in range(0, bs, chunk):
            device.synth_prnu(side, side, b * bs + c0, chunk, args.cameras, args.seed, raw)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            app.preprocess(raw, d * 4, chunk, arena, list(range(row_of_home[b] + c0, row_of_home[b] + c0 + chunk)))
            t_pre += time.perf_counter() - t0
    del raw
    torch.cuda.empty_cache()

    # every rank's arena over CUDA IPC
    h = (C.c_uint8 * 64)()
    check(lib.rk_ipc_handle(arena_p, h))
    everyone = [None] * world
    dist.all_gather_object(everyone, bytes(h))
    peer = {}
    for r, hb in enumerate(everyone):
        if r != rank:
            p = C.c_void_p()
            check(lib.rk_ipc_open((C.c_uint8 * 64)(*hb), local, C.byref(p)))
            peer[r] = p.value
    home_of = {r: [b for b in range(nblk) if owner(b, world) == r] for r in range(world)}

    total = n * (n - 1) // 2
    out = torch.zeros(total, dtype=torch.float64, device="cuda")
    flags = torch.zeros(total, dtype=torch.uint8, device="cuda")
    comp = torch.cuda.Stream()
    copies = [torch.cuda.Stream() for _ in range(args.copy_streams)]
    lanes = [torch.cuda.Stream() for _ in home]            # one compute stream per home block
    fetched = [[torch.cuda.Event() for _ in copies] for _ in range(2)]
    used = [[torch.cuda.Event() for _ in home] for _ in range(2)]
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for ls in lanes:
        ls.wait_stream(comp)
    nf, fetched_bytes, block_pairs = 0, 0, 0
    js = sorted({j for i in home for j in range(i, nblk)})
    for j in js:
        mine = [i for i in home if i <= j]
        if j in row_of_home:
            jrow = row_of_home[j]
        else:
            f = nf % 2
            o = owner(j, world)
            src = peer[o] + home_of[o].index(j) * bs * stride
            dst = arena_p.value + fetch_rows[f] * stride
            piece = (bs * stride) // len(copies)
            for q, cs in enumerate(copies):           # the block in len(copies) concurrent pieces
                if nf >= 2:
                    for ev in used[f]:                # buffer f's previous block is done
                        cs.wait_event(ev)
                nbytes = piece if q < len(copies) - 1 else bs * stride - piece * q
                check(lib.rk_memcpy_d2d(C.c_void_p(dst + q * piece), C.c_void_p(src + q * piece), nbytes,
                                        C.c_void_p(cs.cuda_stream)))
                fetched[f][q].record(cs)
            for ls in lanes:
                for ev in fetched[f]:
                    ls.wait_event(ev)
            jrow = fetch_rows[f]
            fetched_bytes += bs * stride
        for i in mine:
            device.ncc_gram_block(app, arena, n_rows, row_of_home[i], i * bs, bs, jrow, j * bs, bs, out, flags,
                                  stream=lanes[home.index(i)])
            block_pairs += 1
        if j not in row_of_home:
            for k, ls in enumerate(lanes):
                used[nf % 2][k].record(ls)
            nf += 1
    for ls in lanes:
        comp.wait_stream(ls)
    e1.record(comp)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms, t_pre], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    c = torch.tensor([fetched_bytes, block_pairs], dtype=torch.float64, device="cuda")
    dist.all_reduce(c)
    dist.barrier()
    gather_triangle(out, flags)
    torch.cuda.synchronize()

    if rank == 0:
        ms_max, pre_max = t.tolist()
        once = bool(((flags == 1) | (flags == 3)).all().item())
        # sampled pairs inside rank 0's home blocks against the fp32 per-pair path
        g = torch.Generator().manual_seed(args.seed)
        keys = [b * bs + k for b in home for k in range(bs)]
        pairs = []
        while len(pairs) < args.samples:
            a, b = sorted(keys[x] for x in torch.randint(0, len(keys), (2,), generator=g).tolist())
            if a != b:
                pairs.append((a, b))
        slot = {b * bs + k: row_of_home[b] + k for b in home for k in range(bs)}
        ref = torch.zeros(total, dtype=torch.float64, device="cuda")
        app.compare_pairs(arena, [(a, b, slot[a], slot[b]) for a, b in pairs], ref)
        torch.cuda.synchronize()
        err = max(abs(float(ref[i * (2 * n - i - 1) // 2 + (j - i - 1)]) -
                      float(out[i * (2 * n - i - 1) // 2 + (j - i - 1)])) for i, j in pairs)
        flop = 2.0 * d * total
        print(json.dumps({
            "workload": f"zero-lag NCC all-pairs as a blocked tcgen05 TF32 Gram, N={n} items of {side}x{side} fp32 "
                        f"(C3-Gram, SURVEY 8(d)), {bs}-item key blocks",
            "n_gpus": world, "pairs": total, "gram_s": ms_max / 1e3, "pairs_per_s": total / (ms_max / 1e3),
            "tf32_tflops_useful": flop / (ms_max / 1e3) / 1e12,
            "tf32_tflops_useful_per_gpu": flop / (ms_max / 1e3) / 1e12 / world,
            "preprocess_s_max_rank": pre_max, "block_pairs": int(c[1].item()),
            "fetched_gib": c[0].item() / 2**30, "copy_streams": args.copy_streams,
            "check": {"flags_all_written_once": once, "sampled_pairs": len(pairs),
                      "max_abs_diff_vs_fp32_pairs_path": err}}), flush=True)
    for p in peer.values():
        lib.rk_ipc_close(C.c_void_p(p))
    dist.barrier()
    check(lib.rk_device_free(arena_p))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
