"""Channel models and seeded inputs -- the decoder's input contract.

Restates the parts of the reference's ``polarqkd.channel`` that produce the
decoder's inputs, with identical semantics so that identical seeds give
identical frames on a box where the reference is not installed
(tests/test_channel.py pins every function against the reference's own
outputs, committed as golden fixtures).

* LLR convention: natural log, positive favours bit 0; channel LLRs are
  clamped at +-LLR_CLAMP                      (channel.py:10-18, :29)
* ``make_rng``: PCG64 seeded through SeedSequence((seed, stream))
                                              (channel.py:66-73)
* ``transmit``: BSC flips with probability p; BIAWGN sends 1-2b plus
  N(0, 1/snr)                                 (channel.py:116-133)
* ``channel_llr``: BSC (1-2y) min(30, ln((1-p)/p)); BIAWGN clip(2 y snr, +-30)
                                              (channel.py:136-150)
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Union

import numpy as np

LLR_CLAMP = 30.0


@dataclass(frozen=True)
class Bsc:
    """Binary symmetric channel, crossover probability p (channel.py:32-44)."""

    p: float

    def __post_init__(self):
        if not 0.0 <= self.p <= 0.5:
            raise ValueError(f"BSC crossover probability must be in [0, 0.5], got {self.p}")

    @property
    def llr_magnitude(self) -> float:
        if self.p == 0.0:
            return LLR_CLAMP
        if self.p >= 0.5:
            return 0.0
        return min(LLR_CLAMP, float(np.log((1.0 - self.p) / self.p)))


@dataclass(frozen=True)
class BiAwgn:
    """Binary-input AWGN channel, snr = Es / sigma^2 (channel.py:47-60)."""

    snr: float

    def __post_init__(self):
        if not self.snr > 0.0:
            raise ValueError(f"BIAWGN snr must be positive, got {self.snr}")

    @property
    def sigma2(self) -> float:
        return 1.0 / self.snr


ChannelModel = Union[Bsc, BiAwgn]


def make_rng(seed, stream=None) -> np.random.Generator:
    entropy = seed if stream is None else (seed, stream)
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))


def transmit(ch: ChannelModel, bits, seed, stream=None) -> np.ndarray:
    bits = np.asarray(bits)
    if bits.size == 0:
        raise ValueError("transmit requires a nonempty bit vector")
    rng = make_rng(seed, stream)
    if isinstance(ch, Bsc):
        flip = (rng.random(bits.size) < ch.p).astype(np.uint8)
        return bits.astype(np.uint8) ^ flip
    if isinstance(ch, BiAwgn):
        return (1.0 - 2.0 * bits.astype(np.float64)) + rng.normal(0.0, np.sqrt(ch.sigma2), bits.size)
    raise TypeError(f"unsupported channel model: {ch!r}")


def channel_llr(ch: ChannelModel, obs) -> np.ndarray:
    obs = np.atleast_1d(np.asarray(obs))
    if isinstance(ch, Bsc):
        return (1.0 - 2.0 * obs.astype(np.float64)) * ch.llr_magnitude
    if isinstance(ch, BiAwgn):
        return np.clip(2.0 * obs.astype(np.float64) * ch.snr, -LLR_CLAMP, LLR_CLAMP)
    raise TypeError(f"unsupported channel model: {ch!r}")


def channel_tag(ch: ChannelModel) -> tuple[int, float]:
    if isinstance(ch, Bsc):
        return 0, ch.p
    if isinstance(ch, BiAwgn):
        return 1, ch.snr
    raise TypeError(f"unsupported channel model: {ch!r}")


def channel_from_tag(tag: int, param: float) -> ChannelModel:
    if tag == 0:
        return Bsc(param)
    if tag == 1:
        return BiAwgn(param)
    raise ValueError(f"unknown channel tag {tag}")


# --------------------------------------------------------------------------
# frame generation (the builder's seed convention, SURVEY.md 8(d) "Seeds"):
# frame j's key bits come from make_rng(seed, 2j), its channel noise from
# transmit(ch, x, seed, stream=2j+1); frames are independent of GPU count.

def frame_bits(seed: int, j: int, N: int) -> np.ndarray:
    return make_rng(seed, 2 * j).integers(0, 2, N, dtype=np.uint8)


def frame(ch: ChannelModel, seed: int, j: int, N: int):
    """(x bits uint8[N], observation y) for frame j."""
    x = frame_bits(seed, j, N)
    return x, transmit(ch, x, seed, stream=2 * j + 1)


def frames_batch(ch: ChannelModel, seed: int, j0: int, F: int, N: int, threads: int = 0,
                 want_y: bool = True):
    """Frames j0 .. j0+F-1 of the seed convention above, generated on host
    threads (numpy's generators release the GIL while they fill arrays):
    x uint8[F, N], fp32 channel LLRs [F, N], and the BSC received bits
    uint8[F, N] (None for BIAWGN or when not wanted).  Identical to calling
    ``frame`` / ``channel_llr`` per frame, whatever the thread count."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    x = np.empty((F, N), np.uint8)
    llr = np.empty((F, N), np.float32)
    y_bits = np.empty((F, N), np.uint8) if (want_y and isinstance(ch, Bsc)) else None

    def one(i):
        xi, yi = frame(ch, seed, j0 + i, N)
        x[i] = xi
        llr[i] = channel_llr(ch, yi)
        if y_bits is not None:
            y_bits[i] = yi

    if threads <= 0:
        threads = min(32, len(os.sched_getaffinity(0)))
    if threads == 1 or F == 1:
        for i in range(F):
            one(i)
    else:
        with ThreadPoolExecutor(max_workers=min(threads, F)) as ex:
            list(ex.map(one, range(F)))
    return x, llr, y_bits


# --------------------------------------------------------------------------
# the same frames on the device (csrc/frames.cu): BSC only -- numpy's bit and
# uniform draws are integer arithmetic on the PCG64 stream and are reproduced
# bit for bit; Generator.normal (BIAWGN) is not.

def pcg64_seed(seed: int, stream: int) -> tuple[int, int]:
    """(state, inc) of make_rng(seed, stream)'s PCG64 as the C library seeds
    it (numpy: bit_generator.state["state"]); host only."""
    import ctypes

    from . import _lib
    out = (ctypes.c_uint64 * 4)()
    _lib.check(_lib.load().pq_pcg64_seed(seed, stream, out), "pq_pcg64_seed")
    return (out[0] << 64) | out[1], (out[2] << 64) | out[3]


def bsc_frames_device(ch: Bsc, seed: int, j0: int, F: int, n: int, device=None, stream=None):
    """Frames j0 .. j0+F-1 of the seed convention above generated on the GPU:
    (x_words, y_words), int32 CUDA tensors [F, max(1, 2^n / 32)], LSB-first --
    identical to pack_bits of ``frame``'s outputs."""
    import torch

    from . import _lib
    if not isinstance(ch, Bsc):
        raise TypeError("device frame generation covers the BSC only (BIAWGN frames: frames_batch)")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    wpf = max(1, (1 << n) // 32)
    s = torch.cuda.current_stream(dev) if stream is None else stream
    with torch.cuda.device(dev), torch.cuda.stream(s):
        xw = torch.empty((F, wpf), dtype=torch.int32, device=dev)
        yw = torch.empty((F, wpf), dtype=torch.int32, device=dev)
        _lib.check(_lib.load().pq_bsc_frames(n, seed, j0, F, float(ch.p), xw.data_ptr(), yw.data_ptr(),
                                             s.cuda_stream), "pq_bsc_frames")
    return xw, yw
