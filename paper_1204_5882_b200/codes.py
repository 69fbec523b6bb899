"""PolarCode (the construction->decoding contract) and the PQCT code-table file.

* ``PolarCode`` mirrors construction.py:95-126: block size 2^n, frozen_mask
  uint8 of length 2^n with 1 = frozen, plus provenance.
* ``read_code_table`` / ``write_code_table`` implement the reference's binary
  format (construction.py:464-516): b"PQCT", little-endian ``<HBBddI``
  header (version, n, channel tag, channel parameter, target FER, DE bins),
  LSB-first packed mask, then an 8-byte blake2b checksum of everything before
  it.  Corruption raises ValueError exactly where the reference does.

The frozen sets of the five BASELINE.json configs were produced in the build
container by the reference's own density evolution (codes/make_codes.py) and
are shipped as PQCT files under codes/; ``load_config`` reads them back.
"""
from __future__ import annotations

import hashlib
import json
import os
import struct
from dataclasses import dataclass, field

import numpy as np

from .channel import BiAwgn, Bsc, ChannelModel, channel_from_tag, channel_tag

MAGIC = b"PQCT"
VERSION = 1
_HEAD = "<HBBddI"
TOOL_VERSION = "polarqkd-0.1.0"

CODES_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "codes")


@dataclass(frozen=True)
class PolarCode:
    n: int
    frozen_mask: np.ndarray
    channel: ChannelModel
    target_fer: float
    bins: int = 2048
    tool_version: str = TOOL_VERSION
    meta: dict = field(default_factory=dict, compare=False)

    def __post_init__(self):
        if self.frozen_mask.shape != (1 << self.n,):
            raise ValueError("frozen mask length must be exactly 2^n")

    @property
    def block_size(self) -> int:
        return 1 << self.n

    @property
    def frozen_count(self) -> int:
        return int(np.count_nonzero(self.frozen_mask))

    @property
    def rate(self) -> float:
        return 1.0 - self.frozen_count / self.block_size

    def frozen_indices(self) -> np.ndarray:
        return np.nonzero(self.frozen_mask)[0]

    def info_indices(self) -> np.ndarray:
        return np.nonzero(self.frozen_mask == 0)[0]


def _digest(data: bytes) -> int:
    return int.from_bytes(hashlib.blake2b(data, digest_size=8).digest(), "little")


def write_code_table(code: PolarCode, path) -> None:
    tag, param = channel_tag(code.channel)
    body = MAGIC + struct.pack(_HEAD, VERSION, code.n, tag, param, code.target_fer, code.bins)
    body += np.packbits(np.asarray(code.frozen_mask, np.uint8), bitorder="little").tobytes()
    with open(path, "wb") as fh:
        fh.write(body + struct.pack("<Q", _digest(body)))


def read_code_table(path) -> PolarCode:
    """construction.py:483-507 through the C ABI (pq_read_code_table): the
    same validation and ValueError messages as the reference."""
    import ctypes

    from . import _lib
    L = _lib.load()
    n, tag, bins = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    param, fer = ctypes.c_double(), ctypes.c_double()
    bpath = os.fsencode(path)

    def call(*args):
        rc = L.pq_read_code_table(bpath, *args)
        if rc == -2:
            raise FileNotFoundError(L.pq_last_error().decode())
        if rc < 0:
            raise ValueError(L.pq_last_error().decode())  # the reference's messages
        _lib.check(rc, "read_code_table")

    call(ctypes.byref(n), ctypes.byref(tag), ctypes.byref(param), ctypes.byref(fer), ctypes.byref(bins), None, 0)
    mask = np.zeros(1 << n.value, np.uint8)
    call(None, None, None, None, None, mask.ctypes.data, mask.size)
    return PolarCode(n=n.value, frozen_mask=mask, channel=channel_from_tag(tag.value, param.value),
                     target_fer=fer.value, bins=bins.value)


def read_code_table_py(path) -> PolarCode:
    """Pure-Python restatement of the same reader (cross-check in tests)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    hsz = struct.calcsize(_HEAD)
    if len(blob) < 4 + hsz + 8:
        raise ValueError("code table truncated")
    if blob[:4] != MAGIC:
        raise ValueError("bad code-table magic")
    body, stored = blob[:-8], struct.unpack("<Q", blob[-8:])[0]
    if _digest(body) != stored:
        raise ValueError("code-table checksum mismatch")
    version, n, tag, param, target_fer, bins = struct.unpack_from(_HEAD, blob, 4)
    if version != VERSION:
        raise ValueError(f"unsupported code-table version {version}")
    size = 1 << n
    raw = np.frombuffer(blob[4 + hsz: 4 + hsz + (size + 7) // 8], dtype=np.uint8)
    mask = np.unpackbits(raw, bitorder="little")[:size].astype(np.uint8)
    return PolarCode(n=n, frozen_mask=mask, channel=channel_from_tag(tag, param),
                     target_fer=target_fer, bins=bins)


def code_table_checksum(path) -> int:
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < 8:
        raise ValueError("code table truncated")
    return struct.unpack("<Q", blob[-8:])[0]


# --------------------------------------------------------------------------
# BASELINE.json configs

@dataclass(frozen=True)
class Config:
    key: str
    channel: ChannelModel
    n: int
    rate: float
    frames_per_gpu: int
    seed: int
    desc: str


CONFIGS = {
    "c1": Config("c1", Bsc(0.02), 10, 0.80, 64, 1001, "BSC p=0.02, N=2^10, rate 0.8, 64 frames"),
    "c2": Config("c2", Bsc(0.03), 16, 0.75, 1024, 1002, "BSC p=0.03, N=2^16, rate 0.75, 1024 frames/GPU"),
    "c3": Config("c3", Bsc(0.02), 20, 0.83, 256, 1003, "BSC p=0.02, N=2^20, rate 0.83, 256 frames/GPU"),
    "c4": Config("c4", BiAwgn(1.0), 20, 0.45, 256, 1004, "BIAWGN snr=1.0, N=2^20, rate 0.45, 256 frames/GPU"),
    "c5": Config("c5", BiAwgn(0.161), 24, 0.09, 32, 1005, "BIAWGN snr=0.161, N=2^24, rate 0.09, 32 frames/GPU"),
}


def codes_meta() -> dict:
    path = os.path.join(CODES_DIR, "codes.json")
    if not os.path.exists(path):
        return {}
    with open(path) as fh:
        return json.load(fh)


def available_configs() -> list[str]:
    return [k for k in CONFIGS if os.path.exists(os.path.join(CODES_DIR, f"{k}.pqct"))]


def load_config(key: str) -> PolarCode:
    """The reference-constructed rate-K code of BASELINE config `key`."""
    path = os.path.join(CODES_DIR, f"{key}.pqct")
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path}: frozen set for {key} not built (codes/make_codes.py)")
    code = read_code_table(path)
    meta = codes_meta().get(key, {})
    if meta and meta.get("checksum") not in (None, code_table_checksum(path)):
        raise ValueError(f"{path}: checksum differs from codes.json")
    return PolarCode(n=code.n, frozen_mask=code.frozen_mask, channel=code.channel,
                     target_fer=code.target_fer, bins=code.bins, meta=meta)
