"""The package's channel restatement reproduces the reference's outputs
(golden fixtures generated from /root/reference by tests/golden/make_golden.py)."""
import numpy as np
import pytest

from conftest import golden
from paper_1204_5882_b200 import channel as C


def test_make_rng_streams():
    g = golden("channel_vectors.npz")
    for seed, stream in ((0, None), (7, 3), (1003, 0), (1003, 1), (2**40 + 5, 17)):
        tag = f"{seed}_{stream}"
        r = C.make_rng(seed, stream)
        assert np.array_equal(r.integers(0, 2, 4096, dtype=np.uint8), g[f"ints_{tag}"])
        assert np.array_equal(r.random(64), g[f"unif_{tag}"])


@pytest.mark.parametrize("p", [0.0, 0.02, 0.03, 0.1, 0.5])
def test_bsc(p):
    g = golden("channel_vectors.npz")
    y = C.transmit(C.Bsc(p), g["bits"], 5, 9)
    assert np.array_equal(y, g[f"bsc_y_{p}"])
    assert np.array_equal(C.channel_llr(C.Bsc(p), y), g[f"bsc_llr_{p}"])


@pytest.mark.parametrize("snr", [1.0, 0.161, 1e6])
def test_biawgn(snr):
    g = golden("channel_vectors.npz")
    y = C.transmit(C.BiAwgn(snr), g["bits"], 5, 9)
    assert np.array_equal(y, g[f"awgn_y_{snr}"])
    assert np.array_equal(C.channel_llr(C.BiAwgn(snr), y), g[f"awgn_llr_{snr}"])


def test_frame_convention_matches_reference_c1():
    g = golden("c1_frames.npz")
    ch = C.Bsc(0.02)
    for j in range(16):
        x, y = C.frame(ch, int(g["seed"]), j, 1024)
        assert np.array_equal(x, g["x"][j]) and np.array_equal(y, g["y"][j])
        assert np.array_equal(C.channel_llr(ch, y).astype(np.float32), g["llr"][j])


def test_spec_examples():
    assert abs(C.channel_llr(C.Bsc(0.1), 0)[0] - 2.1972) < 1e-4
    assert abs(C.channel_llr(C.Bsc(0.1), 1)[0] + 2.1972) < 1e-4
    assert C.channel_llr(C.BiAwgn(0.5), 1.0)[0] == 1.0
    assert C.channel_llr(C.Bsc(0.0), 0)[0] == C.LLR_CLAMP
    with pytest.raises(ValueError):
        C.Bsc(0.6)
    with pytest.raises(ValueError):
        C.BiAwgn(0.0)
    with pytest.raises(ValueError):
        C.transmit(C.Bsc(0.1), [], 0)
