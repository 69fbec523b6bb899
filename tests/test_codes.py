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
