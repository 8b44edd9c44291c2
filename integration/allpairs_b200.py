"""Reference-side binding: drop-in ``allpairs.apps.Application`` classes whose
preprocess / compare run in librocket (include/rocket.h) through ctypes.

This is the file a maintainer adds next to the reference package
(INTEGRATION.md).  It needs the reference's ``allpairs`` package on the path and
a CUDA device; the engines (``SimEngine``, ``RealEngine``) are unchanged: they
only call the callbacks and read ``ItemData.stage / payload / sim_bytes``.

    from allpairs.realrun import RealEngine
    master = RealEngine(config, B200CompositionVectorApp(corpus_dir)).run()

* ``B200CompositionVectorApp`` subclasses the reference's ``CompositionVectorApp``
  (apps.py:251-363): corpus I/O and ``parse`` are the reference's own; the
  parsed bytes (``<I dim`` + dim x ``<QI``) go straight to ``rk_preprocess``.
* ``B200PCEApp`` is the forensics compare (PRNU PCE); the user's subclass
  supplies ``path_for_key / fetch_raw / parse`` (pattern bytes, fp32 row-major).

Device state: one rk_app and one HBM slot pool per app (slot = item key, so an
item is preprocessed once however the reference's cache tiers evict its
descriptor).  The reference calls preprocess/compare from one ``gpu<d>`` lane
thread per device (realrun.py:140-152); librocket's rk_app is single-stream, so
every call into it holds a lock.
"""

from __future__ import annotations

import ctypes as C
import os
import struct
import threading

from allpairs.apps import (Application, CompositionVectorApp, ItemData, PairResult, Stage,  # the reference
                           require_stage)
from allpairs.errors import AppError, MalformedInput, SlotOverflow

LIB_PATH = os.environ.get("ROCKET_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                      "paper_2009_04755_b200", "librocket.so"))
lib = C.CDLL(LIB_PATH)


class RkAppParams(C.Structure):          # rk_app_params, include/rocket.h
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("height", C.c_int32), ("width", C.c_int32),
                ("seed", C.c_uint64), ("threshold", C.c_double), ("max_entries", C.c_int32),
                ("batch_pairs", C.c_int32), ("gmm_angles", C.c_int32), ("gmm_scale", C.c_float)]


class RkPair(C.Structure):               # rk_pair
    _fields_ = [("i", C.c_int32), ("j", C.c_int32), ("slot_a", C.c_int32), ("slot_b", C.c_int32)]


lib.rk_last_error.restype = C.c_char_p
lib.rk_pair_id.restype = C.c_int64
lib.rk_pair_id.argtypes = [C.c_int64] * 3
lib.rk_app_create.argtypes = [C.POINTER(RkAppParams), C.c_int, C.POINTER(C.c_void_p)]
lib.rk_app_destroy.argtypes = [C.c_void_p]
lib.rk_app_slot_bytes.restype = C.c_size_t
lib.rk_app_slot_bytes.argtypes = [C.c_void_p]
lib.rk_app_parsed_bytes.restype = C.c_size_t
lib.rk_app_parsed_bytes.argtypes = [C.c_void_p]
lib.rk_preprocess.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_size_t,
                              C.POINTER(C.c_int32), C.c_void_p]
lib.rk_compare_pairs.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(RkPair), C.c_int, C.c_void_p,
                                 C.c_void_p, C.c_void_p]

RK_APP_CV, RK_APP_PCE = 1, 2
_ERRORS = {1: ValueError, 2: MalformedInput, 3: SlotOverflow, 7: AssertionError}   # rk_status -> errors.py


def _check(st: int) -> None:
    if st == 0:
        return
    raise _ERRORS.get(st, AppError)(lib.rk_last_error().decode())


class _Rocket:
    """One rk_app on one device with a slot pool where slot k holds item k."""

    def __init__(self, params: RkAppParams, n: int, device: int):
        import torch
        if not torch.cuda.is_available():
            raise AppError("librocket needs a CUDA device (there is no CPU fallback)")
        self.n, self.device = n, device
        self.lock = threading.Lock()
        self.app = C.c_void_p()
        _check(lib.rk_app_create(C.byref(params), device, C.byref(self.app)))
        self.slot_bytes = int(lib.rk_app_slot_bytes(self.app))
        self.parsed_bytes = int(lib.rk_app_parsed_bytes(self.app))
        self.stride = (self.slot_bytes + 255) // 256 * 256
        self.slots = torch.empty(n * self.stride, dtype=torch.uint8, device=f"cuda:{device}")
        self.out = torch.zeros(n * (n - 1) // 2, dtype=torch.float64, device=f"cuda:{device}")
        self.staging = torch.zeros(self.parsed_bytes, dtype=torch.uint8, device=f"cuda:{device}")

    def preprocess(self, key: int, parsed: bytes) -> None:
        import torch
        if len(parsed) > self.parsed_bytes:
            raise SlotOverflow(f"parsed item of {len(parsed)} bytes exceeds {self.parsed_bytes}")
        host = torch.zeros(self.parsed_bytes, dtype=torch.uint8)
        host[:len(parsed)] = torch.frombuffer(bytearray(parsed), dtype=torch.uint8)
        slot = (C.c_int32 * 1)(key)
        with self.lock:
            self.staging.copy_(host)
            torch.cuda.current_stream(self.device).synchronize()
            _check(lib.rk_preprocess(self.app, C.c_void_p(self.staging.data_ptr()), self.parsed_bytes, 1,
                                     C.c_void_p(self.slots.data_ptr()), self.stride, slot, None))
            torch.cuda.synchronize(self.device)

    def compare(self, i: int, j: int) -> float:
        pair = RkPair(i, j, i, j)
        with self.lock:
            _check(lib.rk_compare_pairs(self.app, C.c_void_p(self.slots.data_ptr()), self.stride, C.byref(pair), 1,
                                        C.c_void_p(self.out.data_ptr()), None, None))
            return float(self.out[lib.rk_pair_id(self.n, i, j)])   # synchronising scalar read

    def close(self) -> None:
        if self.app:
            lib.rk_app_destroy(self.app)
            self.app = C.c_void_p()


def _key_of(data: ItemData, key: int) -> int:
    require_stage(data, Stage.PREPROCESSED)
    (stored,) = struct.unpack("<i", data.payload[:4])
    if stored != key:
        raise ValueError(f"item {key} carries the descriptor of item {stored}")
    return stored


class B200PCEApp(Application):
    """PRNU PCE with device-resident spectra.  path_for_key / fetch_raw / parse
    stay the user's I/O (a subclass); parse yields side*side fp32 (row-major)."""

    name = "pce-b200"

    def __init__(self, n: int, side: int = 1024, threshold: float = 60.0, device: int = 0):
        super().__init__(n, slot_size=side * side * 4)
        self.side, self.threshold, self.device = side, threshold, device
        self._rk = _Rocket(RkAppParams(kind=RK_APP_PCE, n=n, height=side, width=side, threshold=threshold),
                           n, device)

    def preprocess(self, key, parsed):                  # gpu lane, engine.py:464-472
        require_stage(parsed, Stage.PARSED)
        self._rk.preprocess(key, parsed.payload)
        return ItemData(Stage.PREPROCESSED, struct.pack("<i", key), sim_bytes=self.slot_size)

    def compare(self, left, right):                     # gpu lane, engine.py:519-528
        (i, a), (j, b) = left, right
        if not i < j:
            raise ValueError(f"pairs are evaluated with left < right, got ({i}, {j})")
        _key_of(a, i), _key_of(b, j)
        return struct.pack("<d", self._rk.compare(i, j))

    def postprocess(self, pair, raw):                   # cpu lane, engine.py:541-548
        (value,) = struct.unpack("<d", raw)
        return PairResult(pair[0], pair[1], value, match=value >= self.threshold)

    def stage_cost(self, stage, i, j=None):
        return 0.0   # real work: RealEngine must not wait out NOMINAL_COSTS (realrun.py:113-114)


class B200CompositionVectorApp(CompositionVectorApp):
    """The reference's composition-vector app with preprocess / compare on the B200.

    Same corpus, k, threshold and slot_size as CompositionVectorApp; the device
    slot holds up to (slot_size - 16) // 16 (token, freq) entries, the
    reference's preprocessed item (4 + 16 * dim bytes) rounded to the device
    layout, so SlotOverflow fires at the same item sizes up to that header."""

    name = "cv-b200"

    def __init__(self, corpus_dir: str, *, device: int = 0, **kw):
        super().__init__(corpus_dir, **kw)
        self.device = device
        cap = max(1, (self.slot_size - 16) // 16)
        self._rk = _Rocket(RkAppParams(kind=RK_APP_CV, n=self.n, threshold=self.threshold, max_entries=cap),
                           self.n, device)

    def preprocess(self, key, parsed):                  # replaces apps.py:304-318 (count -> freq on device)
        require_stage(parsed, Stage.PARSED)
        (dim,) = struct.unpack_from("<I", parsed.payload, 0)
        self._rk.preprocess(key, parsed.payload)
        return ItemData(Stage.PREPROCESSED, struct.pack("<i", key), sim_bytes=4 + 16 * dim)

    def compare(self, left, right):                     # replaces apps.py:331-354 (sorted-merge cosine)
        (i, a), (j, b) = left, right
        if not i < j:
            raise ValueError(f"pairs are evaluated with left < right, got ({i}, {j})")
        _key_of(a, i), _key_of(b, j)
        return struct.pack("<d", self._rk.compare(i, j))

    def stage_cost(self, stage, i, j=None):
        return 0.0
