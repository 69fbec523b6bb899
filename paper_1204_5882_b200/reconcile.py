"""The two ends of the decode step of the reconciliation protocol.

Only the compute chain of SPEC.md's ``reconcile`` module is in scope (SURVEY.md
section 2): Alice's disclosure transform and Bob's LLR -> SC decode ->
re-encode -> verify.  Key-rate and leakage accounting and the wire protocol
are out of scope (scalar bookkeeping, no compute).

alice_disclose(code, x)  -> (frozen_values, hash)
bob_decode(code, obs, ch, frozen_values, hash) -> outcome

Batched device forms for the throughput path: Alice's
transform + hash and Bob's decode -> re-encode -> verify -> tally stay on
the GPU; only the per-frame verdicts (1 byte) and the discarded count need
to come back to the host.
alice_disclose_batch(code, x_words)                  -> (frozen_u words, hashes)
bob_decode_batch(decoder, frozen_u, hashes, llr=..|y_words=..|llr_q88=..)
                                                     -> (verified, x_hat words)

Verification hash ("a fixed, well-known 64-bit non-cryptographic
hash, seed-keyed per session"): XXH64 of the block's packed words as
little-endian bytes, seed = the session key -- the same function on the host
(pq_xxh64) and the device (pq_hash_frames / pq_verify_frames).
"""
from __future__ import annotations

import numpy as np

from .channel import Bsc, ChannelModel, channel_llr
from .codes import PolarCode
from .polar_core import (block_hash_host, hash_frames, pack_bits, polar_transform, polar_transform_words,
                         sc_decode, verify_frames)

VERIFIED, DISCARDED = "Verified", "Discarded"


def block_hash(x, key: int = 0) -> int:
    """64-bit verification hash of a bit block: XXH64 of the
    packed words (bit i at word i>>5, bit i&31), seed = key."""
    return block_hash_host(pack_bits(np.asarray(x, np.uint8)), key)


def alice_disclose(code: PolarCode, x, key: int = 0):
    x = np.asarray(x, np.uint8)
    if x.shape[-1] != code.block_size:
        raise ValueError(f"x length {x.shape[-1]} != 2^n = {code.block_size}")
    u = polar_transform(x)  # the transform is an involution: also the inverse map
    return u[..., code.frozen_indices()].copy(), block_hash(x, key)


def bob_decode(code: PolarCode, obs, ch: ChannelModel, frozen_values, verification_hash: int,
               key: int = 0, f_mode: str = "fixed"):
    """Returns (outcome, x_hat).  On Verified, x_hat equals Alice's x up to the
    2^-64 hash-collision probability."""
    if type(ch) is not type(code.channel):
        raise ValueError("channel family must match the code's design channel")
    obs = np.asarray(obs)
    if obs.shape[-1] != code.block_size:
        raise ValueError(f"obs length {obs.shape[-1]} != 2^n = {code.block_size}")
    llr = channel_llr(ch, obs)
    u_hat = sc_decode(code, llr, frozen_values, f_mode=f_mode)
    x_hat = polar_transform(u_hat)
    ok = block_hash(x_hat, key) == verification_hash
    return (VERIFIED if ok else DISCARDED), x_hat


def alice_disclose_batch(code: PolarCode, x_words, key: int = 0, frozen_words=None, stream=None):
    """alice_disclose for [F, N/32] int32 device words of x: returns the
    revealed u-values as masked u-domain words (u & frozen mask -- the form the
    decoder reads) and the XXH64 hashes ([F] int64)."""
    import torch

    if frozen_words is None:
        frozen_words = torch.from_numpy(pack_bits(code.frozen_mask).view(np.int32).copy()).to(x_words.device)
    s = stream if stream is not None else torch.cuda.current_stream(x_words.device)
    # every op (the allocation of u, the transform, the masking, the hash) is
    # ordered on one stream: the caller's
    with torch.cuda.stream(s):
        u = polar_transform_words(x_words, code.n, stream=s)
        u &= frozen_words
        h = hash_frames(x_words, code.n, key, stream=s)
    return u, h


def bob_decode_batch(decoder, frozen_u, hashes, key: int = 0, llr=None, y_words=None, llr_mag=None,
                     llr_q88=None, n_discarded=None, stream=None):
    """bob_decode for a batch on the device: channel input (fp32 LLRs, BSC
    received words + LLR magnitude, or Q8.8 codes) -> SC decode -> x_hat =
    T(u_hat) (fused into the decoder's output) -> XXH64 compare.  Returns
    (verified [F] uint8, x_hat words); n_discarded (int32 [1] device tensor)
    accumulates the discarded count.  Nothing is copied to the host."""
    if sum(v is not None for v in (llr, y_words, llr_q88)) != 1:
        raise ValueError("give exactly one of llr, y_words, llr_q88")
    if y_words is not None:
        if llr_mag is None:
            raise ValueError("y_words needs llr_mag (the BSC LLR magnitude)")
        _, x_hat = decoder.decode_bsc(y_words, llr_mag, frozen_u, want_u=False, want_x=True, stream=stream)
    elif llr_q88 is not None:
        _, x_hat = decoder.decode_q88(llr_q88, frozen_u, want_u=False, want_x=True, stream=stream)
    else:
        _, x_hat = decoder.decode(llr, frozen_u, want_u=False, want_x=True, stream=stream)
    verified = verify_frames(x_hat, decoder.n, hashes, key, n_discarded=n_discarded, stream=stream)
    return verified, x_hat


__all__ = ["alice_disclose", "bob_decode", "block_hash", "alice_disclose_batch", "bob_decode_batch",
           "VERIFIED", "DISCARDED", "Bsc"]
