"""PQCT code tables: the package reader/writer against the reference format,
and the committed BASELINE-config frozen sets."""
import os

import numpy as np
import pytest

from paper_1204_5882_b200 import codes as K
from paper_1204_5882_b200.channel import BiAwgn, Bsc


def test_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    for n in (1, 3, 10):
        mask = rng.integers(0, 2, 1 << n).astype(np.uint8)
        code = K.PolarCode(n=n, frozen_mask=mask, channel=BiAwgn(0.5), target_fer=0.1)
        p = tmp_path / f"t{n}.pqct"
        K.write_code_table(code, p)
        back = K.read_code_table(p)
        assert back.n == n and np.array_equal(back.frozen_mask, mask)
        assert back.channel == BiAwgn(0.5) and back.target_fer == 0.1


def test_corruption_rejected(tmp_path):
    code = K.PolarCode(n=4, frozen_mask=np.ones(16, np.uint8), channel=Bsc(0.1), target_fer=0.1)
    p = tmp_path / "c.pqct"
    K.write_code_table(code, p)
    blob = bytearray(p.read_bytes())
    blob[-9] ^= 1
    p.write_bytes(bytes(blob))
    with pytest.raises(ValueError, match="checksum"):
        K.read_code_table(p)
    p.write_bytes(b"XXXX" + bytes(blob[4:]))
    with pytest.raises(ValueError):
        K.read_code_table(p)
    p.write_bytes(b"PQ")
    with pytest.raises(ValueError, match="truncated"):
        K.read_code_table(p)
    with pytest.raises(ValueError):
        K.PolarCode(n=3, frozen_mask=np.ones(7, np.uint8), channel=Bsc(0.1), target_fer=0.1)


@pytest.mark.parametrize("key", list(K.CONFIGS))
def test_config_codes(key):
    if key not in K.available_configs():
        pytest.skip(f"{key}.pqct not built yet")
    code = K.load_config(key)
    cfg = K.CONFIGS[key]
    meta = K.codes_meta()[key]
    assert code.n == cfg.n and code.channel == cfg.channel
    K_info = int(round(cfg.rate * code.block_size))
    assert code.block_size - code.frozen_count == K_info == meta["K"]
    assert K.code_table_checksum(os.path.join(K.CODES_DIR, f"{key}.pqct")) == meta["checksum"]


# ---------------------------------------------------------------------------
# the C reader (pq_read_code_table, construction.py:483-507) -- host only

def test_blake2b64_matches_hashlib():
    import hashlib
    from paper_1204_5882_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(5)
    for n in list(range(0, 300)) + [1023, 1024, 1025, 65536 + 7]:
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        want = int.from_bytes(hashlib.blake2b(data, digest_size=8).digest(), "little")
        assert L.pq_blake2b64(data, len(data)) == want, n


def test_c_reader_matches_python_reader_on_committed_tables():
    paths = [os.path.join(K.CODES_DIR, f) for f in sorted(os.listdir(K.CODES_DIR)) if f.endswith(".pqct")]
    assert paths
    for p in paths:
        a, b = K.read_code_table(p), K.read_code_table_py(p)
        assert (a.n, a.channel, a.target_fer, a.bins) == (b.n, b.channel, b.target_fer, b.bins)
        assert np.array_equal(a.frozen_mask, b.frozen_mask)


@pytest.mark.parametrize("damage,msg", [
    ("truncate", "code table truncated"), ("magic", "bad code-table magic"),
    ("checksum", "code-table checksum mismatch"), ("version", "unsupported code-table version 2")])
def test_c_reader_rejections(tmp_path, damage, msg):
    import hashlib
    import struct
    code = K.PolarCode(n=6, frozen_mask=(np.arange(64) % 3 == 0).astype(np.uint8), channel=Bsc(0.05),
                       target_fer=0.1)
    p = tmp_path / "d.pqct"
    K.write_code_table(code, p)
    blob = bytearray(p.read_bytes())
    if damage == "truncate":
        blob = blob[:20]
    elif damage == "magic":
        blob[0:4] = b"PQCX"
    elif damage == "checksum":
        blob[-9] ^= 1
    else:
        blob[4:6] = struct.pack("<H", 2)
        body = bytes(blob[:-8])
        blob[-8:] = struct.pack("<Q", int.from_bytes(hashlib.blake2b(body, digest_size=8).digest(), "little"))
    p.write_bytes(bytes(blob))
    with pytest.raises(ValueError, match=msg):
        K.read_code_table(p)
    with pytest.raises(ValueError, match=msg):
        K.read_code_table_py(p)
    with pytest.raises(FileNotFoundError):
        K.read_code_table(tmp_path / "missing.pqct")


def test_c_reader_matches_reference_reader():
    """The reference's own read_code_table (imported from /root/reference when
    it is present -- build container only) on every committed table."""
    import importlib
    import sys
    ref_src = "/root/reference/pkg/src"
    if not os.path.isdir(ref_src):
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, ref_src)
    try:
        construction = importlib.import_module("polarqkd.construction")
    except Exception as e:  # numba / scipy missing
        pytest.skip(f"reference not importable: {e}")
    finally:
        sys.path.remove(ref_src)
    for f in sorted(os.listdir(K.CODES_DIR)):
        if not f.endswith(".pqct"):
            continue
        p = os.path.join(K.CODES_DIR, f)
        a, r = K.read_code_table(p), construction.read_code_table(p)
        assert a.n == r.n and a.target_fer == r.target_fer and a.bins == r.quantization.bins
        assert np.array_equal(a.frozen_mask, r.frozen_mask)
