"""ctypes binding of librocket (include/rocket.h).

The product path always goes through this library: there is no CPU fallback.
Importing the package on a machine without the built ``librocket.so`` raises
immediately, and every failing C call raises the Python exception that the
reference would raise for the same condition (errors.py taxonomy).
"""

from __future__ import annotations

import ctypes as C
import math
import os

from .errors import AppError, MalformedInput, NoEvictableSlot, SlotOverflow

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librocket.so")

RK_OK = 0
RK_ERR_VALUE = 1
RK_ERR_MALFORMED = 2
RK_ERR_SLOT_OVERFLOW = 3
RK_ERR_NO_EVICTABLE = 4
RK_ERR_DEVICE = 5
RK_ERR_UNSUPPORTED = 6
RK_ERR_DUPLICATE = 7

APP_SYNTHETIC = 0
APP_CV = 1
APP_PCE = 2
APP_NCC = 3
APP_GMM = 4


class AppParams(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("n", C.c_int32),
        ("height", C.c_int32),
        ("width", C.c_int32),
        ("seed", C.c_uint64),
        ("threshold", C.c_double),
        ("max_entries", C.c_int32),
        ("batch_pairs", C.c_int32),
        ("gmm_angles", C.c_int32),
        ("gmm_scale", C.c_float),
    ]


class Pair(C.Structure):
    _fields_ = [("i", C.c_int32), ("j", C.c_int32), ("slot_a", C.c_int32), ("slot_b", C.c_int32)]


class EngineParams(C.Structure):
    _fields_ = [
        ("leaf_block", C.c_int32),
        ("device_slots", C.c_int32),
        ("streams", C.c_int32),
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("peer_tier", C.c_int32),
        ("steal", C.c_int32),
        ("steal_chunk", C.c_int32),
        ("host_slots", C.c_int32),
    ]


class EngineStats(C.Structure):
    _fields_ = [
        ("pairs_done", C.c_int64),
        ("loads", C.c_int64),
        ("hits", C.c_int64),
        ("misses", C.c_int64),
        ("evictions", C.c_int64),
        ("tiles", C.c_int64),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("peer_fetches", C.c_int64),
        ("peer_bytes", C.c_int64),
        ("steals", C.c_int64),
        ("pinned_at_end", C.c_int64),
        ("writing_at_end", C.c_int64),
        ("ledger_marked", C.c_int64),
        ("dup_marks", C.c_int64),
        ("host_hits", C.c_int64),
        ("host_misses", C.c_int64),
        ("host_evictions", C.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class LedgerStats(C.Structure):
    _fields_ = [("total", C.c_int64), ("completed", C.c_int64), ("dup_marks", C.c_int64),
                ("first_dup_pid", C.c_int64), ("full", C.c_int32), ("shared", C.c_int32)]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class TraceEvent(C.Structure):
    _fields_ = [("lane", C.c_int32), ("i", C.c_int32), ("j", C.c_int32), ("count", C.c_int32),
                ("start_ns", C.c_int64), ("end_ns", C.c_int64)]


# (name, restype, argtypes) for every symbol declared in include/rocket.h
SIGNATURES = [
    ("rk_abi_version", C.c_int, []),
    ("rk_last_error", C.c_char_p, []),
    ("rk_status_name", C.c_char_p, [C.c_int]),
    ("rk_pair_id", C.c_int64, [C.c_int64, C.c_int64, C.c_int64]),
    ("rk_pair_from_id", C.c_int, [C.c_int64, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("rk_app_create", C.c_int, [C.POINTER(AppParams), C.c_int, C.POINTER(C.c_void_p)]),
    ("rk_app_destroy", None, [C.c_void_p]),
    ("rk_app_slot_bytes", C.c_size_t, [C.c_void_p]),
    ("rk_app_parsed_bytes", C.c_size_t, [C.c_void_p]),
    ("rk_app_slot_group", C.c_int32, [C.c_void_p]),
    ("rk_preprocess", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_size_t,
                                C.POINTER(C.c_int32), C.c_void_p]),
    ("rk_compare_pairs", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(Pair), C.c_int,
                                   C.c_void_p, C.c_void_p, C.c_void_p]),
    ("rk_compare_tile", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_int32, C.POINTER(C.c_int32), C.c_void_p, C.c_void_p, C.c_void_p]),
    ("rk_ncc_gram", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_int32, C.c_int32,
                              C.c_void_p, C.c_void_p, C.c_void_p]),
    ("rk_ncc_gram_block", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("rk_synth_prnu", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64,
                                C.c_void_p, C.c_void_p]),
    ("rk_engine_create", C.c_int, [C.POINTER(AppParams), C.POINTER(EngineParams), C.c_int,
                                   C.POINTER(C.c_void_p)]),
    ("rk_engine_destroy", None, [C.c_void_p]),
    ("rk_engine_run", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    ("rk_engine_stats_get", C.c_int, [C.c_void_p, C.POINTER(EngineStats)]),
    ("rk_engine_reset_stats", C.c_int, [C.c_void_p]),
    ("rk_engine_set_profiling", C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    ("rk_engine_kernel_time", C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64)]),
    ("rk_engine_stream", C.c_void_p, [C.c_void_p]),
    ("rk_engine_home_region", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    ("rk_engine_arena", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    ("rk_engine_load_home", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    ("rk_engine_load_home_range", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_int32]),
    ("rk_engine_set_peer_homes", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    ("rk_engine_set_trace", C.c_int, [C.c_void_p, C.c_int32]),
    ("rk_engine_ledger_region", C.c_int, [C.c_void_p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    ("rk_engine_use_ledger", C.c_int, [C.c_void_p, C.c_void_p]),
    ("rk_engine_ledger_reset", C.c_int, [C.c_void_p]),
    ("rk_engine_ledger", C.c_int, [C.c_void_p, C.POINTER(LedgerStats)]),
    ("rk_ledger_bytes", C.c_size_t, [C.c_int64]),
    ("rk_app_set_ledger", C.c_int, [C.c_void_p, C.c_void_p]),
    ("rk_ledger_read", C.c_int, [C.c_void_p, C.c_int64, C.POINTER(LedgerStats)]),
    ("rk_engine_trace_get", C.c_int64, [C.c_void_p, C.c_void_p, C.c_int64]),
    ("rk_engine_peer_bandwidth", C.c_int, [C.c_void_p, C.c_int32, C.c_size_t, C.POINTER(C.c_double)]),
    ("rk_engine_queue_word", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("rk_engine_queue_reset", C.c_int, [C.c_void_p]),
    ("rk_engine_set_peer_queues", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    ("rk_device_alloc", C.c_int, [C.c_size_t, C.c_int, C.POINTER(C.c_void_p)]),
    ("rk_device_free", C.c_int, [C.c_void_p]),
    ("rk_memcpy_d2d", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("rk_ipc_handle", C.c_int, [C.c_void_p, C.POINTER(C.c_uint8)]),
    ("rk_ipc_open", C.c_int, [C.POINTER(C.c_uint8), C.c_int, C.POINTER(C.c_void_p)]),
    ("rk_ipc_close", C.c_int, [C.c_void_p]),
    ("rk_tier_create", C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    ("rk_tier_destroy", None, [C.c_void_p]),
    ("rk_tier_acquire", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("rk_tier_publish", C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    ("rk_tier_abort", C.c_int, [C.c_void_p, C.c_int32]),
    ("rk_tier_release", C.c_int, [C.c_void_p, C.c_int32]),
    ("rk_tier_stats", C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    ("rk_tier_slot_key", C.c_int32, [C.c_void_p, C.c_int32]),
    ("rk_queue_step", C.c_int32, [C.c_uint64, C.c_int32, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("rk_leaves", C.c_int64, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int64]),
]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the all-pairs engine has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, restype, argtypes in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    return lib


lib = _load()


def last_error() -> str:
    return (lib.rk_last_error() or b"").decode(errors="replace")


def check(status: int) -> None:
    """Raise the reference's exception type for a failing status."""
    if status == RK_OK:
        return
    msg = last_error()
    if status == RK_ERR_VALUE:
        raise ValueError(msg)
    if status == RK_ERR_MALFORMED:
        raise MalformedInput(msg)
    if status == RK_ERR_SLOT_OVERFLOW:
        raise SlotOverflow(msg)
    if status == RK_ERR_NO_EVICTABLE:
        raise NoEvictableSlot(msg)
    if status == RK_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if status == RK_ERR_DUPLICATE:
        raise AssertionError(msg)      # PairLedger.mark (scheduler.py:233-241)
    raise AppError(f"librocket device failure: {msg}")


def app_params(kind: int, n: int, *, height: int = 0, width: int = 0, seed: int = 0,
               threshold: float | None = None, max_entries: int = 0, batch_pairs: int = 0,
               gmm_angles: int = 0, gmm_scale: float = 0.0) -> AppParams:
    return AppParams(kind, n, height, width, seed & ((1 << 64) - 1),
                     math.nan if threshold is None else float(threshold),
                     max_entries, batch_pairs, gmm_angles, gmm_scale)
