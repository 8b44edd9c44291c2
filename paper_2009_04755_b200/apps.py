"""The reference's plugin contract, restated, with B200-backed applications behind it.

Mirrors /root/reference/pkg/src/allpairs/apps.py:
  Stage :24-29, ItemData :32-52, PairResult :55-66, require_stage :69-71,
  Application :74-125 (path_for_key / fetch_raw / raw_size / parse / preprocess /
  compare / postprocess / stage_cost / describe), _check_slot :128-132.

Each GPU application keeps the reference's per-item / per-pair callbacks (so it
can be driven one pair at a time by a reference-style engine: preprocess returns
an ItemData whose payload is a small descriptor of the item's HBM slot, compare
runs the CUDA kernel on the two slots) and adds the batched path used by
``AllPairsEngine``: parsed items packed at a fixed stride for the C-ABI engine.
There is no CPU fallback: constructing a GPU application without librocket or
without a CUDA device raises.
"""

from __future__ import annotations

import enum
import gzip
import math
import os
import struct
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .errors import AppError, MalformedInput, SlotOverflow

ItemKey = int


class Stage(enum.IntEnum):
    """Progress of one item through the load pipeline; only moves forward."""

    RAW_FILE = 0
    PARSED = 1
    PREPROCESSED = 2


@dataclass(frozen=True)
class ItemData:
    """Loaded bytes for one item at a given pipeline stage (apps.py:32-52)."""

    stage: Stage
    payload: bytes
    sim_bytes: int = -1

    def __post_init__(self) -> None:
        if self.sim_bytes < 0:
            object.__setattr__(self, "sim_bytes", len(self.payload))

    @property
    def byte_length(self) -> int:
        return len(self.payload)


@dataclass(frozen=True)
class PairResult:
    """Outcome of comparing items left < right (apps.py:55-66)."""

    left: ItemKey
    right: ItemKey
    value: float
    match: Optional[bool] = None

    def __post_init__(self) -> None:
        if not self.left < self.right:
            raise ValueError(f"pair must satisfy left < right, got ({self.left}, {self.right})")


def require_stage(data: ItemData, stage: Stage) -> None:
    if data.stage != stage:
        raise ValueError(f"expected stage {stage.name}, got {data.stage.name}")


def match_from_flag(flag: int) -> Optional[bool]:
    """Wire encoding of PairResult.match (wire.py:165-167): 0 None, 1 False, 3 True."""
    return None if not flag & 1 else bool(flag & 2)


class Application:
    """Base contract for an all-pairs application (apps.py:74-125)."""

    name = "app"
    n: int
    slot_size: int

    def __init__(self, n: int, slot_size: int):
        if n < 1:
            raise ValueError(f"item count must be >= 1, got {n}")
        if slot_size <= 0:
            raise ValueError("slot_size must be positive")
        self.n = n
        self.slot_size = slot_size

    def path_for_key(self, key: ItemKey) -> str:
        raise NotImplementedError

    def fetch_raw(self, path: str) -> bytes:
        raise NotImplementedError

    def raw_size(self, key: ItemKey) -> int:
        return len(self.fetch_raw(self.path_for_key(key)))

    def parse(self, key: ItemKey, raw: ItemData) -> ItemData:
        raise NotImplementedError

    def preprocess(self, key: ItemKey, parsed: ItemData) -> ItemData:
        raise NotImplementedError

    def compare(self, left: tuple[ItemKey, ItemData], right: tuple[ItemKey, ItemData]) -> bytes:
        raise NotImplementedError

    def postprocess(self, pair: tuple[ItemKey, ItemKey], raw: bytes) -> PairResult:
        raise NotImplementedError

    def stage_cost(self, stage: str, i: ItemKey, j: Optional[ItemKey] = None) -> Optional[float]:
        return None

    def describe(self) -> dict:
        return {"kind": self.name, "n": self.n, "slot_size": self.slot_size}


# ---------------------------------------------------------------------------
# B200-backed applications

_DESC = struct.Struct("<4sIiiq")   # magic, device, slot, key, pool id
_MAGIC = b"RKSL"


class B200Application(Application):
    """An Application whose preprocess/compare run in librocket on one GPU.

    Per-item path: preprocess() copies the parsed bytes to the device and runs
    rk_preprocess into a slot of this application's HBM slot pool; the returned
    ItemData carries a descriptor of that slot (sim_bytes = the slot size, as
    the reference charges transfers by logical size).  compare() runs
    rk_compare_pairs on the two slots and returns the 8-byte little-endian
    float64 result, exactly like the reference apps.
    """

    kind: int = -1

    def __init__(self, n: int, *, device: int = 0, threshold: Optional[float] = None, **params):
        self.device = device
        self.threshold = threshold
        self._params = params
        self._dev = None
        self._pool = None
        self._slot_of_key: dict[int, int] = {}
        self._free: list[int] = []
        self._pool_id = id(self) & 0x7FFFFFFFFFFF
        super().__init__(n, self._slot_bytes())

    # -- subclass hooks ------------------------------------------------------
    def app_params(self) -> _lib.AppParams:
        return _lib.app_params(self.kind, self.n, threshold=self.threshold, **self._params)

    def _slot_bytes(self) -> int:
        return self.device_app().slot_bytes

    def parsed_bytes(self) -> int:
        """Fixed stride of one parsed item in the batched (engine) path."""
        return self.device_app().parsed_bytes

    def parsed_array(self, parsed: ItemData) -> np.ndarray:
        """Parsed payload as a uint8 array of exactly parsed_bytes()."""
        buf = np.frombuffer(parsed.payload, dtype=np.uint8)
        out = np.zeros(self.parsed_bytes(), dtype=np.uint8)
        if buf.size > out.size:
            raise SlotOverflow(f"parsed item of {buf.size} bytes exceeds {out.size}")
        out[: buf.size] = buf
        return out

    # -- device plumbing -----------------------------------------------------
    def device_app(self):
        if self._dev is None:
            import torch
            if not torch.cuda.is_available():
                raise AppError("B200 applications need a CUDA device (no CPU fallback)")
            from .device import DeviceApp
            self._dev = DeviceApp(self.app_params(), self.device)
        return self._dev

    def _ensure_pool(self):
        if self._pool is None:
            dev = self.device_app()
            self._pool = dev.alloc_slots(self.n)
            self._free = list(range(self.n - 1, -1, -1))
        return self._pool

    def _descriptor(self, key: int, slot: int) -> bytes:
        return _DESC.pack(_MAGIC, self.device, slot, key, self._pool_id)

    def _slot_from(self, key: int, data: ItemData) -> int:
        require_stage(data, Stage.PREPROCESSED)
        magic, device, slot, dkey, pool = _DESC.unpack(data.payload)
        if magic != _MAGIC or pool != self._pool_id or dkey != key:
            raise ValueError(f"item {key} was not preprocessed by this application")
        return slot

    # -- contract -------------------------------------------------------------
    def preprocess(self, key: ItemKey, parsed: ItemData) -> ItemData:
        require_stage(parsed, Stage.PARSED)
        import torch
        dev = self.device_app()
        pool = self._ensure_pool()
        slot = self._slot_of_key.get(key)
        if slot is None:
            if not self._free:
                raise SlotOverflow(f"device slot pool of {self.n} items is full")
            slot = self._free.pop()
            self._slot_of_key[key] = slot
        host = torch.from_numpy(self.parsed_array(parsed))
        buf = host.to(f"cuda:{self.device}")
        dev.preprocess(buf, self.parsed_bytes(), 1, pool, [slot])
        torch.cuda.synchronize(self.device)
        return ItemData(Stage.PREPROCESSED, self._descriptor(key, slot), sim_bytes=self.slot_size)

    def compare(self, left: tuple[ItemKey, ItemData], right: tuple[ItemKey, ItemData]) -> bytes:
        (i, a), (j, b) = left, right
        sa, sb = self._slot_from(i, a), self._slot_from(j, b)
        if not i < j:
            raise ValueError(f"pairs are evaluated with left < right, got ({i}, {j})")
        import torch
        dev = self.device_app()
        total = self.n * (self.n - 1) // 2
        out = torch.empty(1, dtype=torch.float64, device=f"cuda:{self.device}")
        # the kernel writes at pair_id; route it through a 1-element view
        pid = i * (2 * self.n - i - 1) // 2 + (j - i - 1)
        scratch = getattr(self, "_scratch", None)
        if scratch is None or scratch.numel() != total:
            scratch = torch.empty(total, dtype=torch.float64, device=f"cuda:{self.device}")
            self._scratch = scratch
        dev.compare_pairs(self._pool, [(i, j, sa, sb)], scratch)
        out.copy_(scratch[pid:pid + 1])
        return struct.pack("<d", float(out.item()))

    def postprocess(self, pair: tuple[ItemKey, ItemKey], raw: bytes) -> PairResult:
        (value,) = struct.unpack("<d", raw)
        match = None if self.threshold is None else value >= self.threshold
        return PairResult(pair[0], pair[1], value, match)

    def stage_cost(self, stage: str, i: ItemKey, j: Optional[ItemKey] = None) -> Optional[float]:
        # real work, not a modeled cost: a reference RealEngine must not wait
        # out NOMINAL_COSTS on top of it (engine.py:43, realrun.py:113-114)
        return 0.0

    def close(self) -> None:
        if self._dev is not None:
            self._dev.close()
            self._dev = None
        self._pool = None


class PCEApp(B200Application):
    """PRNU peak-to-correlation-energy over fp32 patterns (forensics).

    Items are square fp32 patterns (256^2, 1024^2 or 2048^2).  By default they are the
    deterministic synthetic PRNU-like patterns of rk_synth_prnu (item k =
    0.2*K[k % cameras] + N(0,1)); pass ``patterns`` (n x side x side float32) to
    compare real data.  postprocess: match = PCE >= threshold (default 60).
    """

    name = "pce"
    kind = _lib.APP_PCE

    def __init__(self, n: int, side: int = 1024, *, cameras: int = 64, seed: int = 0,
                 patterns: Optional[np.ndarray] = None, threshold: Optional[float] = 60.0, device: int = 0):
        self.side = side
        self.cameras = cameras
        self.seed = seed
        if patterns is not None:
            patterns = np.ascontiguousarray(patterns, dtype=np.float32)
            if patterns.shape != (n, side, side):
                raise ValueError(f"patterns must be {(n, side, side)}, got {patterns.shape}")
        self.patterns = patterns
        super().__init__(n, device=device, threshold=threshold, height=side, width=side)

    def path_for_key(self, key: ItemKey) -> str:
        return f"prnu/{key:06d}.f32"

    def _key_of(self, path: str) -> int:
        return int(os.path.basename(path).split(".")[0])

    def fetch_raw(self, path: str) -> bytes:
        key = self._key_of(path)
        if self.patterns is not None:
            return self.patterns[key].tobytes()
        import torch
        from .device import synth_prnu
        buf = torch.empty(self.side * self.side, dtype=torch.float32, device=f"cuda:{self.device}")
        synth_prnu(self.side, self.side, key, 1, self.cameras, self.seed, buf)
        return buf.cpu().numpy().tobytes()

    def _slot_bytes(self) -> int:
        return self.side * self.side * 4          # (N/2) x N complex64 half spectrum

    def parsed_bytes(self) -> int:
        return self.side * self.side * 4

    def raw_size(self, key: ItemKey) -> int:
        return self.side * self.side * 4

    def parse(self, key: ItemKey, raw: ItemData) -> ItemData:
        require_stage(raw, Stage.RAW_FILE)
        if len(raw.payload) != self.side * self.side * 4:
            raise MalformedInput(f"{self.path_for_key(key)}: expected {self.side}x{self.side} fp32, "
                                 f"got {len(raw.payload)} bytes")
        arr = np.frombuffer(raw.payload, dtype=np.float32)
        if not np.all(np.isfinite(arr)):
            raise MalformedInput(f"{self.path_for_key(key)}: non-finite samples")
        return ItemData(Stage.PARSED, raw.payload)

    def describe(self) -> dict:
        out = super().describe()
        out.update(side=self.side, cameras=self.cameras, seed=self.seed, threshold=self.threshold)
        return out


class NCCApp(PCEApp):
    """Zero-lag normalised cross-correlation of fp32 patterns (the paper's forensics
    compare): preprocess normalises each item to zero mean and unit
    norm, compare is the dot product -- all pairs run as a tcgen05 TF32 Gram
    (|error| <= 2e-4).  Same pattern I/O as PCEApp; match = NCC >= threshold."""

    name = "ncc"
    kind = _lib.APP_NCC

    def __init__(self, n: int, side: int = 1024, *, threshold: Optional[float] = 0.02, **kw):
        super().__init__(n, side, threshold=threshold, **kw)

    def _slot_bytes(self) -> int:
        return self.side * self.side * 4          # D normalised fp32 samples


class SyntheticApp(B200Application):
    """The reference's SyntheticApp (apps.py:154-227) with the hash compare on the GPU.

    fetch_raw / parse / preprocess / stage_cost keep the reference semantics;
    compare returns mix64(seed, 0xC0403A3E, i, j) / 2^64, bit-identical.
    """

    name = "synthetic"
    kind = _lib.APP_SYNTHETIC
    _STAGE_IDS = {"io": 1, "parse": 2, "upload": 3, "preprocess": 4, "compare": 5, "download": 6, "postprocess": 7}

    def __init__(self, n: int, slot_size: int = 1 << 16, *, seed: int = 0, payload_bytes: int = 64,
                 file_bytes: Optional[int] = None, item_bytes: Optional[int] = None,
                 costs: Optional[dict] = None, device: int = 0):
        self.seed = seed
        self.payload_bytes = payload_bytes
        self.file_bytes = file_bytes if file_bytes is not None else payload_bytes
        self.item_bytes = item_bytes if item_bytes is not None else min(slot_size, self.file_bytes)
        self.costs = dict(costs or {})
        self._slot = slot_size
        super().__init__(n, device=device, threshold=None, seed=seed)
        self.slot_size = slot_size

    def _slot_bytes(self) -> int:
        return self._slot

    def parsed_bytes(self) -> int:
        return 8

    def path_for_key(self, key: ItemKey) -> str:
        return f"items/{key:06d}.bin"

    def fetch_raw(self, path: str) -> bytes:
        from .rng import mix64
        key = int(os.path.basename(path).split(".")[0])
        out = bytearray()
        state = mix64(self.seed, 0xF11E, key)
        while len(out) < self.payload_bytes:
            state = mix64(state)
            out += state.to_bytes(8, "little")
        return bytes(out[: self.payload_bytes])

    def raw_size(self, key: ItemKey) -> int:
        return self.file_bytes

    def parse(self, key: ItemKey, raw: ItemData) -> ItemData:
        require_stage(raw, Stage.RAW_FILE)
        return ItemData(Stage.PARSED, raw.payload, sim_bytes=self.item_bytes)

    def preprocess(self, key: ItemKey, parsed: ItemData) -> ItemData:
        require_stage(parsed, Stage.PARSED)
        if parsed.sim_bytes > self.slot_size:
            raise SlotOverflow(f"preprocessed item of {parsed.sim_bytes} bytes exceeds slot size {self.slot_size}")
        # identity payload; the compare hash needs only the keys
        return ItemData(Stage.PREPROCESSED, self._descriptor(key, -1), sim_bytes=parsed.sim_bytes)

    def compare(self, left, right) -> bytes:
        (i, a), (j, b) = left, right
        self._slot_from(i, a)
        self._slot_from(j, b)
        if not i < j:
            raise ValueError(f"pairs are evaluated with left < right, got ({i}, {j})")
        import torch
        total = self.n * (self.n - 1) // 2
        scratch = getattr(self, "_scratch", None)
        if scratch is None:
            scratch = torch.empty(total, dtype=torch.float64, device=f"cuda:{self.device}")
            self._scratch = scratch
        self.device_app().compare_pairs(scratch, [(i, j, 0, 0)], scratch)
        pid = i * (2 * self.n - i - 1) // 2 + (j - i - 1)
        return struct.pack("<d", float(scratch[pid].item()))

    def postprocess(self, pair, raw: bytes) -> PairResult:
        (value,) = struct.unpack("<d", raw)
        return PairResult(pair[0], pair[1], value)

    def stage_cost(self, stage: str, i: ItemKey, j: Optional[ItemKey] = None) -> Optional[float]:
        spec = self.costs.get(stage)
        if spec is None:
            return None
        from .rng import lognormal_duration, mix64
        mean, std = spec
        seed = mix64(self.seed, 0xD07A7109, self._STAGE_IDS.get(stage, 0), i, -1 if j is None else j)
        return lognormal_duration(mean, std, seed)


class CompositionVectorApp(B200Application):
    """The reference's composition-vector cosine (apps.py:251-363) with a GPU compare.

    parse runs on the host (the reference's cpu lane) and produces the
    reference's byte layout; preprocess (count -> frequency, norm) and the
    sparse merge compare run in librocket (warp per pair, fp64).
    """

    name = "cv"
    kind = _lib.APP_CV
    _HEAD = struct.Struct("<I")
    _COUNT = struct.Struct("<QI")

    def __init__(self, corpus_dir: str, *, k: int = 3, threshold: float = 0.5, slot_size: int = 1 << 20,
                 n: Optional[int] = None, device: int = 0):
        if not 1 <= k <= 8:
            raise ValueError("k must be in 1..8 so token ids fit in 64 bits")
        files = sorted(os.path.join(corpus_dir, f) for f in os.listdir(corpus_dir)
                       if os.path.isfile(os.path.join(corpus_dir, f)))
        if not files:
            raise ValueError(f"no corpus files found in {corpus_dir}")
        if n is not None:
            files = files[:n]
        self.files = files
        self.k = k
        # slot capacity in (token, freq) entries; slot_size keeps the reference's
        # 16-byte-per-entry accounting (+4 byte header)
        max_entries = max(1, (slot_size - 4) // 16)
        super().__init__(len(files), device=device, threshold=threshold, max_entries=max_entries)
        self.slot_size = slot_size

    def _slot_bytes(self) -> int:
        return 16 + 16 * self._params["max_entries"]

    def parsed_bytes(self) -> int:
        return 4 + 12 * self._params["max_entries"]

    def path_for_key(self, key: ItemKey) -> str:
        return self.files[key]

    def fetch_raw(self, path: str) -> bytes:
        with open(path, "rb") as fh:
            return fh.read()

    @staticmethod
    def kmer_counts(text: str, k: int) -> dict[int, int]:
        """apps.py:237-248: whitespace-stripped, upper-cased, big-endian UTF-8 ids."""
        cleaned = "".join(text.split()).upper()
        counts: dict[int, int] = {}
        for pos in range(len(cleaned) - k + 1):
            token = int.from_bytes(cleaned[pos:pos + k].encode("utf-8"), "big")
            counts[token] = counts.get(token, 0) + 1
        return counts

    def parse(self, key: ItemKey, raw: ItemData) -> ItemData:
        require_stage(raw, Stage.RAW_FILE)
        blob = raw.payload
        if self.path_for_key(key).endswith(".gz"):
            blob = gzip.decompress(blob)
        try:
            text = blob.decode("utf-8")
        except UnicodeDecodeError as exc:
            raise MalformedInput(f"{self.path_for_key(key)}: not valid UTF-8") from exc
        counts = self.kmer_counts(text, self.k)
        if not counts:
            raise MalformedInput(f"{self.path_for_key(key)}: no {self.k}-mers (empty or too short)")
        out = bytearray(self._HEAD.pack(len(counts)))
        for token in sorted(counts):
            out += self._COUNT.pack(token, counts[token])
        return ItemData(Stage.PARSED, bytes(out))

    def preprocess(self, key: ItemKey, parsed: ItemData) -> ItemData:
        require_stage(parsed, Stage.PARSED)
        (dim,) = self._HEAD.unpack_from(parsed.payload, 0)
        if 4 + 16 * dim > self.slot_size:
            raise SlotOverflow(f"preprocessed item of {4 + 16 * dim} bytes exceeds slot size {self.slot_size}")
        return super().preprocess(key, parsed)

    def describe(self) -> dict:
        out = super().describe()
        out.update(k=self.k, threshold=self.threshold, corpus=[os.path.basename(f) for f in self.files])
        return out


class ParticleFusionApp(B200Application):
    """Localization-microscopy particle registration cost.

    Items are particles of up to ``max_points`` localizations (x, y, sigma);
    compare = max over a fixed rotation grid of the Gaussian-overlap
    (Bhattacharyya / GMM-L2 cross term) normalised by m_i * m_j (csrc/gmm.cu).
    By default items are deterministic synthetic particles (a ring of binding
    sites under a random rigid transform); pass ``particles`` to use real data.
    """

    name = "gmm"
    kind = _lib.APP_GMM
    _HEAD = struct.Struct("<II")

    def __init__(self, n: int, *, seed: int = 0, max_points: int = 400, angles: int = 36, scale: float = 0.0,
                 particles: Optional[list] = None, threshold: Optional[float] = None, device: int = 0):
        self.seed = seed
        self.max_points = max_points
        self.angles = angles
        self.particles = particles
        super().__init__(n, device=device, threshold=threshold, max_entries=max_points, gmm_angles=angles,
                         gmm_scale=scale)

    def _slot_bytes(self) -> int:
        return 8 + 12 * self.max_points

    def parsed_bytes(self) -> int:
        return 8 + 12 * self.max_points

    def path_for_key(self, key: ItemKey) -> str:
        return f"particles/{key:06d}.loc"

    def points(self, key: ItemKey) -> np.ndarray:
        if self.particles is not None:
            return np.asarray(self.particles[key], dtype=np.float32)
        from .synthdata import particle
        return particle(key, self.seed)

    def fetch_raw(self, path: str) -> bytes:
        pts = self.points(int(os.path.basename(path).split(".")[0]))
        return self._HEAD.pack(len(pts), 0) + pts.astype("<f4").tobytes()

    def parse(self, key: ItemKey, raw: ItemData) -> ItemData:
        require_stage(raw, Stage.RAW_FILE)
        if len(raw.payload) < 8:
            raise MalformedInput(f"{self.path_for_key(key)}: truncated header")
        m, _ = self._HEAD.unpack_from(raw.payload, 0)
        if m == 0 or len(raw.payload) != 8 + 12 * m:
            raise MalformedInput(f"{self.path_for_key(key)}: bad localization count {m}")
        if m > self.max_points:
            raise SlotOverflow(f"{self.path_for_key(key)}: {m} localizations exceed {self.max_points}")
        return ItemData(Stage.PARSED, raw.payload)
