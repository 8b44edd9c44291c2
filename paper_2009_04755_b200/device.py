"""Thin object wrappers over the librocket handles (rk_app, rk_engine).

Device memory and streams are PyTorch plumbing: tensors are handed to the C
ABI as raw pointers; all arithmetic happens in librocket's kernels.
"""

from __future__ import annotations

import ctypes as C
from typing import Iterable, Optional, Sequence

import torch

from . import _lib
from ._lib import check, lib


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class DeviceApp:
    """One rk_app on one device: preprocess and compare entry points."""

    def __init__(self, params: _lib.AppParams, device: int = 0):
        self.params = params
        self.device = device
        handle = C.c_void_p()
        check(lib.rk_app_create(C.byref(params), device, C.byref(handle)))
        self.handle = handle
        self.slot_bytes = int(lib.rk_app_slot_bytes(handle))
        self.parsed_bytes = int(lib.rk_app_parsed_bytes(handle))
        self.slot_stride = (self.slot_bytes + 255) // 256 * 256
        self.slot_group = int(lib.rk_app_slot_group(handle))

    def close(self) -> None:
        if self.handle:
            lib.rk_app_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def alloc_slots(self, count: int) -> torch.Tensor:
        g = self.slot_group   # interleaved slot groups: whole groups only
        count = (count + g - 1) // g * g
        return torch.empty(count * self.slot_stride, dtype=torch.uint8, device=f"cuda:{self.device}")

    def preprocess(self, parsed: torch.Tensor, parsed_stride: int, n_items: int, slots: torch.Tensor,
                   slot_idx: Sequence[int], stream=None) -> None:
        idx = (C.c_int32 * len(slot_idx))(*slot_idx)
        check(lib.rk_preprocess(self.handle, _ptr(parsed), parsed_stride, n_items, _ptr(slots),
                                self.slot_stride, idx, _stream(stream)))

    def compare_pairs(self, slots: torch.Tensor, pairs: Iterable[tuple[int, int, int, int]], out: torch.Tensor,
                      flags: Optional[torch.Tensor] = None, stream=None) -> None:
        plist = list(pairs)
        arr = (_lib.Pair * len(plist))(*[_lib.Pair(*p) for p in plist])
        check(lib.rk_compare_pairs(self.handle, _ptr(slots), self.slot_stride, arr, len(plist), _ptr(out),
                                   _ptr(flags), _stream(stream)))

    def set_ledger(self, region: Optional[torch.Tensor]) -> None:
        """Mark every pair this app compares in `region` (rk_ledger_bytes(n) zeroed
        device bytes, see ledger_region()); None turns the ledger off."""
        check(lib.rk_app_set_ledger(self.handle, _ptr(region)))

    def ledger_region(self) -> torch.Tensor:
        nbytes = int(lib.rk_ledger_bytes(self.params.n))
        return torch.zeros(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")

    def ledger(self, region: torch.Tensor) -> dict:
        st = _lib.LedgerStats()
        check(lib.rk_ledger_read(_ptr(region), self.params.n, C.byref(st)))
        return st.as_dict()

    def gram(self, slots: torch.Tensor, n_rows: int, out: torch.Tensor, flags: Optional[torch.Tensor] = None,
             rank: int = 0, world: int = 1, stream=None) -> None:
        """NCC all-pairs over resident slots (slot k = item k) as the tcgen05 Gram (rk_ncc_gram)."""
        check(lib.rk_ncc_gram(self.handle, _ptr(slots), self.slot_stride, n_rows, rank, world, _ptr(out),
                              _ptr(flags), _stream(stream)))

    def compare_tile(self, slots: Optional[torch.Tensor], r0: int, r1: int, c0: int, c1: int,
                     slot_of_key: Sequence[int], out: torch.Tensor, flags: Optional[torch.Tensor] = None,
                     stream=None) -> None:
        sok = (C.c_int32 * max(1, len(slot_of_key)))(*slot_of_key)
        check(lib.rk_compare_tile(self.handle, _ptr(slots), self.slot_stride, r0, r1, c0, c1, sok, _ptr(out),
                                  _ptr(flags), _stream(stream)))


def ncc_gram_block(app: "DeviceApp", slots: torch.Tensor, n_rows: int, a_row0: int, a_key0: int, a_cnt: int,
                   b_row0: int, b_key0: int, b_cnt: int, out: torch.Tensor, flags: Optional[torch.Tensor] = None,
                   stream=None) -> None:
    """One NCC Gram block (rk_ncc_gram_block) over an arena holding a subset of the items."""
    check(lib.rk_ncc_gram_block(app.handle, _ptr(slots), app.slot_stride, n_rows, a_row0, a_key0, a_cnt, b_row0,
                                b_key0, b_cnt, _ptr(out), _ptr(flags), _stream(stream)))


def synth_prnu(h: int, w: int, first_key: int, n_items: int, cameras: int, seed: int,
               out: torch.Tensor, stream=None) -> torch.Tensor:
    """Deterministic PRNU-like fp32 patterns into `out` (device, n_items*h*w floats)."""
    assert out.dtype == torch.float32 and out.is_cuda and out.numel() >= n_items * h * w
    check(lib.rk_synth_prnu(h, w, first_key, n_items, cameras, seed & ((1 << 64) - 1), _ptr(out),
                            _stream(stream)))
    return out


class DeviceEngine:
    """rk_engine: quadtree tiles over an HBM slot tier, fed by host or device items."""

    def __init__(self, params: _lib.AppParams, *, leaf_block: int = 8, device_slots: int = 0,
                 rank: int = 0, world: int = 1, device: int = 0, peer_tier: bool = False, steal: bool = False,
                 steal_chunk: int = 0, host_slots: int = 0):
        self.params = params
        self.device = device
        self.rank, self.world = rank, world
        slots = device_slots if device_slots > 0 else max(2, params.n)
        ep = _lib.EngineParams(leaf_block, slots, 1, rank, world, int(bool(peer_tier and world > 1)),
                               int(bool(steal and world > 1)), steal_chunk, host_slots)
        handle = C.c_void_p()
        check(lib.rk_engine_create(C.byref(params), C.byref(ep), device, C.byref(handle)))
        self.handle = handle
        self.engine_params = ep

    def close(self) -> None:
        if self.handle:
            self.close_peers()
            lib.rk_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def run(self, out: torch.Tensor, flags: Optional[torch.Tensor] = None, *,
            host_items: Optional[torch.Tensor] = None, device_items: Optional[torch.Tensor] = None,
            parsed_stride: int = 0) -> None:
        # the engine runs on its own stream: order it after the caller's pending work
        # (e.g. the initialisation of out/flags on torch's stream)
        torch.cuda.current_stream(self.device).synchronize()
        check(lib.rk_engine_run(self.handle, _ptr(host_items), _ptr(device_items), parsed_stride, _ptr(out),
                                _ptr(flags)))

    def stats(self) -> dict:
        st = _lib.EngineStats()
        check(lib.rk_engine_stats_get(self.handle, C.byref(st)))
        return st.as_dict()

    def reset_stats(self) -> None:
        check(lib.rk_engine_reset_stats(self.handle))

    def ledger(self) -> dict:
        """The exactly-once ledger this engine marks into (the job's shared one on
        rank 0 after connect_peers): total, completed, dup_marks, full."""
        st = _lib.LedgerStats()
        check(lib.rk_engine_ledger(self.handle, C.byref(st)))
        return st.as_dict()

    def check_ledger(self) -> dict:
        """Raise AssertionError (PairLedger.mark, scheduler.py:233-241) if any pair
        completed twice; returns the ledger otherwise."""
        led = self.ledger()
        if led["dup_marks"]:
            i, j = C.c_int64(), C.c_int64()
            check(lib.rk_pair_from_id(self.params.n, led["first_dup_pid"], C.byref(i), C.byref(j)))
            raise AssertionError(f"pair ({i.value}, {j.value}) completed twice ({led['dup_marks']} duplicate marks)")
        return led

    def use_ledger(self, region_ptr: int) -> None:
        """Mark into the ledger region at a device address (e.g. another engine's)."""
        check(lib.rk_engine_use_ledger(self.handle, region_ptr))

    def ledger_region_ptr(self) -> int:
        arena, stride = C.c_void_p(), C.c_size_t()
        check(lib.rk_engine_arena(self.handle, C.byref(arena), C.byref(stride)))
        off, nbytes = C.c_size_t(), C.c_size_t()
        check(lib.rk_engine_ledger_region(self.handle, C.byref(off), C.byref(nbytes)))
        return int(arena.value) + int(off.value)

    def ledger_reset(self) -> None:
        """Clear the shared ledger (rank 0; a no-op elsewhere) before the pre-run barrier."""
        check(lib.rk_engine_ledger_reset(self.handle))

    def set_profiling(self, every: int, max_samples: int = 1024) -> None:
        check(lib.rk_engine_set_profiling(self.handle, every, max_samples))

    _TRACE_LANES = {0: ("gpu", "compare"), 1: ("up", "preprocess"), 2: ("up", "fetch")}

    def set_trace(self, max_events: int) -> None:
        """Record up to max_events trace events per run (0 disables)."""
        check(lib.rk_engine_set_trace(self.handle, max_events))

    def trace(self, node: int = 0) -> list[dict]:
        """The last run's events in the reference's TraceEvent schema (metrics.py:14-29):
        lane gpu<d> for compare batches, up<d> for loads / peer fetches; i, j = first
        pair (or first key and -1) of the group; ns from the start of the run."""
        n = int(lib.rk_engine_trace_get(self.handle, None, 0))
        buf = (_lib.TraceEvent * max(1, n))()
        lib.rk_engine_trace_get(self.handle, buf, n)
        out = []
        for ev in buf[:n]:
            kind, label = self._TRACE_LANES[int(ev.lane)]
            out.append({"node": node, "lane": f"{kind}{self.device}", "label": label,
                        "start_ns": int(ev.start_ns), "end_ns": int(ev.end_ns), "i": int(ev.i), "j": int(ev.j),
                        "count": int(ev.count)})
        return out

    def kernel_time(self) -> tuple[float, int, int]:
        """(summed ms, sampled launches, pairs in those launches) of the last run."""
        ms = C.c_double()
        cnt = C.c_int64()
        pairs = C.c_int64()
        check(lib.rk_engine_kernel_time(self.handle, C.byref(ms), C.byref(cnt), C.byref(pairs)))
        return float(ms.value), int(cnt.value), int(pairs.value)

    def stream(self) -> int:
        return int(lib.rk_engine_stream(self.handle) or 0)

    # -- peer-GPU tier (one process per GPU; needs torch.distributed) ----------------
    @property
    def peer_tier(self) -> bool:
        return bool(self.engine_params.peer_tier)

    def load_home(self, *, host_items=None, device_items=None, parsed_stride: int = 0) -> None:
        torch.cuda.current_stream(self.device).synchronize()
        check(lib.rk_engine_load_home(self.handle, _ptr(host_items), _ptr(device_items), parsed_stride))

    def load_home_range(self, m0: int, count: int, *, host_items=None, device_items=None,
                        parsed_stride: int = 0) -> None:
        """Home items m0 .. m0+count-1 (item m0+q at items + q*parsed_stride)."""
        torch.cuda.current_stream(self.device).synchronize()
        check(lib.rk_engine_load_home_range(self.handle, _ptr(host_items), _ptr(device_items), parsed_stride,
                                            m0, count))

    @property
    def steal(self) -> bool:
        return bool(self.engine_params.steal)

    def connect_peers(self) -> None:
        """Map every rank's slot arena over CUDA IPC (handles travel through
        torch.distributed): the home regions (peer tier) and the work-queue words
        (stealing) are offsets into it."""
        import torch.distributed as dist
        base, nbytes = C.c_void_p(), C.c_size_t()
        check(lib.rk_engine_home_region(self.handle, C.byref(base), C.byref(nbytes)))
        arena, stride = C.c_void_p(), C.c_size_t()
        check(lib.rk_engine_arena(self.handle, C.byref(arena), C.byref(stride)))
        qword = C.c_void_p()
        check(lib.rk_engine_queue_word(self.handle, C.byref(qword)))
        loff, lbytes = C.c_size_t(), C.c_size_t()
        check(lib.rk_engine_ledger_region(self.handle, C.byref(loff), C.byref(lbytes)))
        hbuf = (C.c_uint8 * 64)()
        check(lib.rk_ipc_handle(arena, hbuf))
        a0 = int(arena.value)
        mine = (bytes(hbuf), int(base.value or a0) - a0, int(qword.value) - a0, int(loff.value))
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine)
        homes = (C.c_void_p * self.world)()
        queues = (C.c_void_p * self.world)()
        self._opened = []
        ledger0 = None
        for r, (h, hoff, qoff, lo) in enumerate(everyone):
            if r == self.rank:
                pbase = a0
            else:
                peer = C.c_void_p()
                check(lib.rk_ipc_open((C.c_uint8 * 64)(*h), self.device, C.byref(peer)))
                self._opened.append(peer)
                pbase = int(peer.value)
            homes[r] = pbase + hoff
            queues[r] = pbase + qoff
            if r == 0:
                ledger0 = pbase + lo
        # one exactly-once ledger for the whole job: rank 0's, marked over NVLink
        check(lib.rk_engine_use_ledger(self.handle, ledger0))
        if self.peer_tier:
            check(lib.rk_engine_set_peer_homes(self.handle, self.world, homes))
        if self.steal:
            check(lib.rk_engine_set_peer_queues(self.handle, self.world, queues))

    def peer_bandwidth(self, src_rank: int, nbytes: int) -> float:
        """GB/s of the peer-tier D2D copy from src_rank's home region (between runs only)."""
        gbs = C.c_double()
        check(lib.rk_engine_peer_bandwidth(self.handle, src_rank, nbytes, C.byref(gbs)))
        return float(gbs.value)

    def queue_reset(self) -> None:
        """Own work-queue word <- this rank's share; every rank, then a barrier, before run()."""
        check(lib.rk_engine_queue_reset(self.handle))

    def close_peers(self) -> None:
        for p in getattr(self, "_opened", []):
            lib.rk_ipc_close(p)
        self._opened = []
