"""The two ends of the decode step of the reconciliation protocol.

Only the compute chain of SPEC.md's ``reconcile`` module is in scope (SURVEY.md
section 2): Alice's disclosure transform and Bob's LLR -> SC decode ->
re-encode -> verify.  Key-rate and leakage accounting and the wire protocol
are out of scope (scalar bookkeeping, no compute).

alice_disclose(code, x)  -> (frozen_values, hash)
bob_decode(code, obs, ch, frozen_values, hash) -> outcome
"""
from __future__ import annotations

import hashlib

import numpy as np

from .channel import Bsc, ChannelModel, channel_llr
from .codes import PolarCode
from .polar_core import pack_bits, polar_transform, sc_decode

VERIFIED, DISCARDED = "Verified", "Discarded"


def block_hash(x, key: int = 0) -> int:
    """64-bit verification hash of a bit block (a fixed,
    well-known, seed-keyed 64-bit hash; here keyed BLAKE2b-64)."""
    data = pack_bits(np.asarray(x, np.uint8)).tobytes()
    k = int(key).to_bytes(8, "little")
    return int.from_bytes(hashlib.blake2b(data, digest_size=8, key=k).digest(), "little")


def alice_disclose(code: PolarCode, x, key: int = 0):
    x = np.asarray(x, np.uint8)
    if x.shape[-1] != code.block_size:
        raise ValueError(f"x length {x.shape[-1]} != 2^n = {code.block_size}")
    u = polar_transform(x)  # the transform is an involution: also the inverse map
    return u[..., code.frozen_indices()].copy(), block_hash(x, key)


def bob_decode(code: PolarCode, obs, ch: ChannelModel, frozen_values, verification_hash: int,
               key: int = 0, f_mode: str = "exact"):
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


__all__ = ["alice_disclose", "bob_decode", "block_hash", "VERIFIED", "DISCARDED", "Bsc"]
