"""Reference-side binding: a drop-in ``allpairs.apps.Application`` whose
preprocess / compare run in librocket (include/rocket.h) through ctypes.

This is the file a maintainer adds next to the reference package
(INTEGRATION.md).  It needs the reference's ``allpairs`` package on the path and
a CUDA device; the engines (``SimEngine``, ``RealEngine``) are unchanged: they
only call the callbacks and read ``ItemData.stage / payload / sim_bytes``.

    from allpairs.realrun import RealEngine
    master = RealEngine(config, B200PCEApp(n=128, side=256)).run()
"""

from __future__ import annotations

import ctypes as C
import os
import struct

from allpairs.apps import Application, ItemData, PairResult, Stage, require_stage  # the reference
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
lib.rk_preprocess.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_size_t,
                              C.POINTER(C.c_int32), C.c_void_p]
lib.rk_compare_pairs.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(RkPair), C.c_int, C.c_void_p,
                                 C.c_void_p, C.c_void_p]

_ERRORS = {1: ValueError, 2: MalformedInput, 3: SlotOverflow}   # rk_status -> errors.py


def _check(st: int) -> None:
    if st == 0:
        return
    raise _ERRORS.get(st, AppError)(lib.rk_last_error().decode())


class B200PCEApp(Application):
    """PRNU PCE with device-resident spectra (slot k holds item k)."""

    name = "pce-b200"

    def __init__(self, n: int, side: int = 1024, threshold: float = 60.0, device: int = 0):
        import torch
        super().__init__(n, slot_size=side * side * 4)
        self.side, self.threshold, self.device = side, threshold, device
        self.app = C.c_void_p()
        _check(lib.rk_app_create(C.byref(RkAppParams(kind=2, n=n, height=side, width=side, threshold=threshold)),
                                 device, C.byref(self.app)))
        self.slots = torch.empty(n * self.slot_size, dtype=torch.uint8, device=f"cuda:{device}")
        self.out = torch.zeros(n * (n - 1) // 2, dtype=torch.float64, device=f"cuda:{device}")

    # path_for_key / fetch_raw / parse stay the user's I/O (cpu and io lanes)

    def preprocess(self, key, parsed):                  # gpu lane, engine.py:464-472
        import torch
        require_stage(parsed, Stage.PARSED)
        x = torch.frombuffer(bytearray(parsed.payload), dtype=torch.float32).to(f"cuda:{self.device}")
        slot = (C.c_int32 * 1)(key)
        _check(lib.rk_preprocess(self.app, C.c_void_p(x.data_ptr()), self.slot_size, 1,
                                 C.c_void_p(self.slots.data_ptr()), self.slot_size, slot, None))
        torch.cuda.synchronize(self.device)
        return ItemData(Stage.PREPROCESSED, struct.pack("<i", key), sim_bytes=self.slot_size)

    def compare(self, left, right):                     # gpu lane, engine.py:519-528
        (i, a), (j, b) = left, right
        if not i < j:
            raise ValueError(f"pairs are evaluated with left < right, got ({i}, {j})")
        pair = RkPair(i, j, struct.unpack("<i", a.payload)[0], struct.unpack("<i", b.payload)[0])
        _check(lib.rk_compare_pairs(self.app, C.c_void_p(self.slots.data_ptr()), self.slot_size,
                                    C.byref(pair), 1, C.c_void_p(self.out.data_ptr()), None, None))
        return struct.pack("<d", float(self.out[lib.rk_pair_id(self.n, i, j)]))

    def postprocess(self, pair, raw):                   # cpu lane, engine.py:541-548
        (value,) = struct.unpack("<d", raw)
        return PairResult(pair[0], pair[1], value, match=value >= self.threshold)

    def stage_cost(self, stage, i, j=None):
        return 0.0   # real work: RealEngine must not wait out NOMINAL_COSTS (realrun.py:113-114)
