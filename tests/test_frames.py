"""Seeded BSC frames generated on the device (csrc/frames.cu)
against the reference's numpy call sequence (channel.py:66-73, :116-125): the
host seeding against numpy itself, the device frames against the reference's
own c1 frames (tests/golden/c1_frames.npz) and against channel.frame()."""
import numpy as np
import pytest

from conftest import golden
from paper_1204_5882_b200 import channel as C
from paper_1204_5882_b200.polar_core import pack_bits


@pytest.mark.parametrize("seed,stream", [(0, 0), (2012, 0), (2012, 1), (7, 5), (1003, 2 * 999 + 1),
                                         (2**40 + 5, 17), (2**63 + 11, 2**33), (2**64 - 1, 2**64 - 1)])
def test_pcg64_seed_matches_numpy(seed, stream):
    st = np.random.PCG64(np.random.SeedSequence((seed, stream))).state["state"]
    assert C.pcg64_seed(seed, stream) == (st["state"], st["inc"])


def test_device_generator_rejects_biawgn():
    with pytest.raises(TypeError):
        C.bsc_frames_device(C.BiAwgn(1.0), 1, 0, 1, 10)


@pytest.mark.gpu
def test_device_frames_equal_reference_c1(cuda):
    g = golden("c1_frames.npz")
    xw, yw = C.bsc_frames_device(C.Bsc(0.02), int(g["seed"]), 0, 16, 10, device=cuda)
    assert np.array_equal(xw.cpu().numpy().view(np.uint32), pack_bits(g["x"][:16]))
    assert np.array_equal(yw.cpu().numpy().view(np.uint32), pack_bits(g["y"][:16]))


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,seed,j0,F", [(0, 0.1, 3, 0, 4), (2, 0.3, 3, 5, 3), (3, 0.25, 9, 1, 5), (5, 0.11, 77, 0, 7),
                                           (10, 0.02, 2012, 123, 5), (13, 0.5, 5, 2**40, 3), (13, 0.0, 5, 0, 2),
                                           (16, 0.03, 2**40 + 5, 7, 3), (20, 0.02, 2020, 250, 2)])
def test_device_frames_equal_host_frames(cuda, n, p, seed, j0, F):
    ch = C.Bsc(p)
    N = 1 << n
    xw, yw = C.bsc_frames_device(ch, seed, j0, F, n, device=cuda)
    xs, ys = zip(*[C.frame(ch, seed, j0 + f, N) for f in range(F)])
    assert np.array_equal(xw.cpu().numpy().view(np.uint32), pack_bits(np.array(xs)))
    assert np.array_equal(yw.cpu().numpy().view(np.uint32), pack_bits(np.array(ys).astype(np.uint8)))


@pytest.mark.gpu
def test_device_frames_argument_errors(cuda):
    with pytest.raises(ValueError):
        C.bsc_frames_device(C.Bsc(0.1), 1, 0, 0, 10, device=cuda)
    with pytest.raises(ValueError):
        C.bsc_frames_device(C.Bsc(0.1), 1, 0, 1, 31, device=cuda)
