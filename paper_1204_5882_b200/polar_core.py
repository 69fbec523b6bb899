"""polar_core -- the SPEC's decoding module, B200-backed.

Drop-in names and argument meaning follow SPEC.md:
  polar_transform(u) -> x
  phi(x)
  sc_decode(code, llrs, frozen_values) -> u_hat
with the reference's error behaviour (ValueError on bad lengths / arguments,
SPEC.md:244 "length mismatches rejected").  Everything runs on the GPU
through libpolarsc.so (include/polarsc.h); there is no CPU path.

Batched entry points for the throughput path work on device tensors:
  ScDecoder(code, max_frames).decode(llr[F,N] fp32, frozen_u words[F,N/32])
  ScDecoder.decode_bsc(y words[F,N/32], ...)   (fused BSC front end)
  polar_transform_words(words[F,N/32], n)
Bit vectors are packed LSB-first into 32-bit words (bit i of a frame at word
i >> 5, bit i & 31), the PQCT mask order (construction.py:476).
"""
from __future__ import annotations

import ctypes
import hashlib

import numpy as np

from . import _lib
from .codes import PolarCode

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


# --------------------------------------------------------------------------
# bit packing

def words_per_frame(n: int) -> int:
    return max(1, (1 << n) // 32)


def pack_bits(bits) -> np.ndarray:
    """[..., N] {0,1} -> [..., max(1, N/32)] uint32, LSB-first."""
    b = np.asarray(bits, dtype=np.uint8) & 1
    N = b.shape[-1]
    if N < 32:
        pad = np.zeros(b.shape[:-1] + (32,), np.uint8)
        pad[..., :N] = b
        b = pad
    packed = np.packbits(b, axis=-1, bitorder="little")
    return np.ascontiguousarray(packed).view("<u4")


def unpack_bits(words, N: int) -> np.ndarray:
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32))
    bits = np.unpackbits(w.view(np.uint8), axis=-1, bitorder="little")
    return bits[..., :N]


# --------------------------------------------------------------------------
# phi (host math; SPEC.md:230-238 -- not on the decode path, which evaluates
# the same boxplus in its numerically stable form on the GPU)

def phi(x):
    """phi(x) = -ln(tanh(x/2)) for x > 0; an involution on (0, inf)."""
    xa = np.asarray(x, dtype=np.float64)
    if np.any(~(xa > 0)):
        raise ValueError("phi requires x > 0")
    out = -np.log(np.tanh(xa / 2.0))
    return float(out) if out.ndim == 0 else out


# --------------------------------------------------------------------------
# device helpers

def _require_cuda(device=None):
    if torch is None or not torch.cuda.is_available():
        raise _lib.PolarScError("a CUDA device is required (no CPU fallback)")
    if isinstance(device, torch.device):
        if device.type != "cuda":
            raise ValueError(f"device must be a CUDA device, got {device}")
        device = device.index
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
    return dev


def _stream_ptr(stream, device=None):
    """The cudaStream_t to launch on: `stream`, else the current stream of
    `device` (the handle's device, not whatever device is current)."""
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _check_words(t, frames, wpf, name):
    if t is None:
        return
    if not (t.is_cuda and t.dtype == torch.int32 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous int32 CUDA tensor of packed words")
    if t.numel() < frames * wpf:
        raise ValueError(f"{name} holds {t.numel()} words, need {frames * wpf}")


F_MODES = {"exact": _lib.PQ_F_EXACT, "fast": _lib.PQ_F_FAST, "min-sum": _lib.PQ_F_MINSUM,
           "minsum": _lib.PQ_F_MINSUM, "fixed": _lib.PQ_F_FIXED}


class ScDecoder:
    """A decoder instance: owns its device scratch (allocated here, never in
    decode) and is single-threaded, as SPEC.md:274-275 prescribes.  The code
    table is copied in and immutable afterwards."""

    def __init__(self, code: PolarCode, max_frames: int = 1, f_mode: str = "exact",
                 ssc: bool = True, subtree_log2: int = 0, device=None):
        self.device = _require_cuda(device)
        if f_mode not in F_MODES:
            raise ValueError(f"unknown f mode {f_mode!r} (exact | fast | fixed | min-sum)")
        L = _lib.load()
        self.code = code
        self.n = code.n
        self.N = 1 << code.n
        self.wpf = words_per_frame(code.n)
        self.max_frames = int(max_frames)
        self._h = ctypes.c_void_p()
        _lib.check(L.pq_decoder_create(ctypes.byref(self._h), code.n, self.max_frames,
                                       F_MODES[f_mode], self.device.index), "pq_decoder_create")
        mask = np.ascontiguousarray(code.frozen_mask, dtype=np.uint8)
        _lib.check(L.pq_decoder_set_frozen_mask(self._h, mask.tobytes()), "pq_decoder_set_frozen_mask")
        self.set_option(_lib.PQ_OPT_SSC, 1 if ssc else 0)
        if subtree_log2:
            self.set_option(_lib.PQ_OPT_SUBTREE_LOG2, subtree_log2)
        self.frozen_words = torch.from_numpy(pack_bits(mask).view(np.int32).copy()).to(self.device)

    # -- options / introspection
    def set_option(self, key: int, value: int) -> None:
        _lib.check(_lib.load().pq_decoder_set_option(self._h, key, int(value)), "pq_decoder_set_option")

    @property
    def last_config(self) -> dict:
        """Launch shape of the last decode: sub-tree width log2, threads per
        CTA, CTAs per frame."""
        vals = [ctypes.c_int(0) for _ in range(3)]
        _lib.check(_lib.load().pq_decoder_last_config(self._h, *[ctypes.byref(v) for v in vals]),
                   "pq_decoder_last_config")
        return {"subtree_log2": vals[0].value, "threads_per_cta": vals[1].value, "ctas_per_frame": vals[2].value}

    @property
    def last_ctas_per_frame(self) -> int:
        """Thread-block cluster size (CTAs per frame) of the last decode."""
        return int(_lib.load().pq_decoder_last_ctas_per_frame(self._h))

    @property
    def workspace_bytes(self) -> int:
        return int(_lib.load().pq_decoder_workspace_bytes(self._h))

    @property
    def last_launches(self) -> int:
        return int(_lib.load().pq_decoder_last_launches(self._h))

    def read_profile(self, frames: int) -> np.ndarray:
        """[frames, PQ_PROF_SLOTS] clock64 cycles per step class of the last
        decode (set_option(PQ_OPT_PROFILE, 1) first)."""
        out = np.zeros((frames, _lib.PQ_PROF_SLOTS), np.uint64)
        _lib.check(_lib.load().pq_decoder_read_profile(self._h, out.ctypes.data, frames),
                   "pq_decoder_read_profile")
        return out

    def kernel_times(self, count: int) -> np.ndarray:
        """Durations (ms) of the sc_decode_kernel launches of the last `count`
        decodes made with set_option(PQ_OPT_TIMING, 1): CUDA events on the
        launching stream right around the kernel (measurement only)."""
        out = np.zeros(count, np.float32)
        _lib.check(_lib.load().pq_decoder_kernel_times(self._h, out.ctypes.data, int(count)),
                   "pq_decoder_kernel_times")
        return out

    def alloc_words(self, frames: int):
        return torch.empty((frames, self.wpf), dtype=torch.int32, device=self.device)

    # -- decoding
    def decode(self, llr, frozen_u=None, u_hat=None, x_hat=None, want_u=True, want_x=False,
               stream=None):
        """llr: [F, N] float32 CUDA; frozen_u: [F, N/32] int32 words with the
        revealed u-values at frozen positions (None = all zero).  Returns
        (u_hat words, x_hat words), either None if not requested."""
        if not (llr.is_cuda and llr.dtype == torch.float32 and llr.is_contiguous() and llr.dim() == 2):
            raise ValueError("llr must be a contiguous [frames, N] float32 CUDA tensor")
        F = llr.shape[0]
        if llr.shape[1] != self.N:
            raise ValueError(f"llr length {llr.shape[1]} != N = {self.N}")
        u_hat, x_hat = self._outs(F, u_hat, x_hat, want_u, want_x)
        _check_words(frozen_u, F, self.wpf, "frozen_u")
        rc = _lib.load().pq_sc_decode_f32(self._h, _ptr(llr), _ptr(frozen_u), _ptr(u_hat), _ptr(x_hat),
                                          F, _stream_ptr(stream, self.device))
        _lib.check(rc, "pq_sc_decode_f32")
        return u_hat, x_hat

    def decode_q88(self, llr_q88, frozen_u=None, u_hat=None, x_hat=None, want_u=True, want_x=False,
                   stream=None):
        """SPEC.md:250 sc_decode_fixed on the device: llr_q88 is a contiguous
        [F, N] int16 CUDA tensor of saturating Q8.8 raw codes (quantize_q88);
        fixed-point decoders only."""
        if not (llr_q88.is_cuda and llr_q88.dtype == torch.int16 and llr_q88.is_contiguous()
                and llr_q88.dim() == 2):
            raise ValueError("llr_q88 must be a contiguous [frames, N] int16 CUDA tensor")
        F = llr_q88.shape[0]
        if llr_q88.shape[1] != self.N:
            raise ValueError(f"llr length {llr_q88.shape[1]} != N = {self.N}")
        u_hat, x_hat = self._outs(F, u_hat, x_hat, want_u, want_x)
        _check_words(frozen_u, F, self.wpf, "frozen_u")
        rc = _lib.load().pq_sc_decode_q88(self._h, _ptr(llr_q88), _ptr(frozen_u), _ptr(u_hat), _ptr(x_hat),
                                          F, _stream_ptr(stream, self.device))
        _lib.check(rc, "pq_sc_decode_q88")
        return u_hat, x_hat

    def decode_bsc(self, y_words, llr_mag: float, frozen_u=None, u_hat=None, x_hat=None,
                   want_u=True, want_x=False, frames=None, stream=None):
        """Fused BSC front end: y_words [F, N/32] int32 received bits."""
        F = y_words.shape[0] if frames is None else int(frames)
        _check_words(y_words, F, self.wpf, "y_words")
        _check_words(frozen_u, F, self.wpf, "frozen_u")
        u_hat, x_hat = self._outs(F, u_hat, x_hat, want_u, want_x)
        rc = _lib.load().pq_sc_decode_bsc(self._h, _ptr(y_words), ctypes.c_float(llr_mag), _ptr(frozen_u),
                                          _ptr(u_hat), _ptr(x_hat), F, _stream_ptr(stream, self.device))
        _lib.check(rc, "pq_sc_decode_bsc")
        return u_hat, x_hat

    def decode_dump(self, llr, frozen_u=None, stream=None):
        """Plain SC with every stage LLR: returns (u_hat, x_hat, dump[F, n+1, N])
        in the coset-shifted domain."""
        F = llr.shape[0]
        u_hat, x_hat = self._outs(F, None, None, True, True)
        dump = torch.zeros((F, self.n + 1, self.N), dtype=torch.float32, device=self.device)
        _check_words(frozen_u, F, self.wpf, "frozen_u")
        rc = _lib.load().pq_sc_decode_f32_dump(self._h, _ptr(llr), _ptr(frozen_u), _ptr(u_hat),
                                               _ptr(x_hat), _ptr(dump), F, _stream_ptr(stream, self.device))
        _lib.check(rc, "pq_sc_decode_f32_dump")
        return u_hat, x_hat, dump

    def _outs(self, F, u_hat, x_hat, want_u, want_x):
        if F > self.max_frames:
            raise ValueError(f"{F} frames > max_frames {self.max_frames}")
        if u_hat is None and want_u:
            u_hat = self.alloc_words(F)
        if x_hat is None and want_x:
            x_hat = self.alloc_words(F)
        _check_words(u_hat, F, self.wpf, "u_hat")
        _check_words(x_hat, F, self.wpf, "x_hat")
        return u_hat, x_hat

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().pq_decoder_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def f_device(a, b, f_mode: str = "exact"):
    """The decoder's signed f on device arrays (diagnostics / parity tests)."""
    _require_cuda()
    if not (a.is_cuda and b.is_cuda and a.dtype == torch.float32 and b.dtype == torch.float32):
        raise ValueError("a, b must be float32 CUDA tensors")
    a, b = a.contiguous(), b.contiguous()
    out = torch.empty_like(a)
    rc = _lib.load().pq_debug_fmag(F_MODES[f_mode], _ptr(a), _ptr(b), _ptr(out), a.numel(),
                                   _stream_ptr(None))
    _lib.check(rc, "pq_debug_fmag")
    return out


# --------------------------------------------------------------------------
# SPEC-named entry points

def polar_transform_words(words, n: int, out=None, stream=None):
    """x = u F^{(x)n} on packed device words [F, N/32] (int32)."""
    _require_cuda()
    F = words.shape[0] if words.dim() == 2 else 1
    wpf = words_per_frame(n)
    _check_words(words, F, wpf, "words")
    if out is None:
        out = torch.empty_like(words)
    rc = _lib.load().pq_polar_transform(_ptr(words), _ptr(out), n, F, _stream_ptr(stream, words.device))
    _lib.check(rc, "pq_polar_transform")
    return out


def hash_frames(x_words, n: int, key: int = 0, out=None, stream=None):
    """XXH64 (seed = key) of every frame's packed words on the device:
    [F, N/32] int32 -> [F] int64 (the uint64 hash bits)."""
    _require_cuda()
    F = x_words.shape[0] if x_words.dim() == 2 else 1
    _check_words(x_words, F, words_per_frame(n), "x_words")
    if out is None:
        out = torch.empty(F, dtype=torch.int64, device=x_words.device)
    rc = _lib.load().pq_hash_frames(_ptr(x_words), n, F, key & (2 ** 64 - 1), _ptr(out), _stream_ptr(stream, x_words.device))
    _lib.check(rc, "pq_hash_frames")
    return out


def verify_frames(x_words, n: int, expect, key: int = 0, verified=None, n_discarded=None, stream=None):
    """bob_decode's verification on the device: verified[f]
    = XXH64(x_hat[f], key) == expect[f] (uint8), and the discarded count is
    added to n_discarded (int32 [1] device tensor) when given."""
    _require_cuda()
    F = x_words.shape[0] if x_words.dim() == 2 else 1
    _check_words(x_words, F, words_per_frame(n), "x_words")
    if not (expect.is_cuda and expect.dtype == torch.int64 and expect.numel() >= F):
        raise ValueError("expect must be an int64 CUDA tensor of >= frames hashes")
    if verified is None:
        verified = torch.empty(F, dtype=torch.uint8, device=x_words.device)
    rc = _lib.load().pq_verify_frames(_ptr(x_words), n, F, key & (2 ** 64 - 1), _ptr(expect), _ptr(verified),
                                      _ptr(n_discarded) if n_discarded is not None else None,
                                      _stream_ptr(stream, x_words.device))
    _lib.check(rc, "pq_verify_frames")
    return verified


def block_hash_host(x_words: np.ndarray, key: int = 0) -> int:
    """The same XXH64 on the host (no GPU needed), over packed words."""
    data = np.ascontiguousarray(np.asarray(x_words, dtype="<u4")).tobytes()
    return int(_lib.load().pq_xxh64(data, len(data), key & (2 ** 64 - 1)))


def polar_transform(u) -> np.ndarray:
    """u (length 2^n bits, or [F, 2^n]) -> x, on the GPU."""
    dev = _require_cuda()
    u = np.asarray(u)
    N = u.shape[-1]
    if N < 1 or N & (N - 1):
        raise ValueError("polar_transform: length must be a power of two")
    if N == 1:
        return (u.astype(np.uint8) & 1).copy()
    n = N.bit_length() - 1
    words = torch.from_numpy(pack_bits(u.reshape(-1, N)).view(np.int32).copy()).to(dev)
    out = polar_transform_words(words, n)
    torch.cuda.current_stream().synchronize()
    x = unpack_bits(out.cpu().numpy().view(np.uint32), N)
    return x.reshape(u.shape).astype(np.uint8)


_DECODERS: dict = {}


def _cached_decoder(code: PolarCode, frames: int, f_mode: str) -> ScDecoder:
    key = (code.n, hashlib.blake2b(np.ascontiguousarray(code.frozen_mask, np.uint8).tobytes(),
                                   digest_size=16).digest(), f_mode, torch.cuda.current_device())
    dec = _DECODERS.get(key)
    if dec is None or dec.max_frames < frames:
        dec = ScDecoder(code, max_frames=max(frames, 1), f_mode=f_mode)
        _DECODERS[key] = dec
    return dec


def scatter_frozen_values(code: PolarCode, frozen_values) -> np.ndarray:
    """Compact |F| vector(s) in ascending frozen-index order
    -> full-length u-domain bits [.., N] with the values at frozen positions."""
    fv = np.asarray(frozen_values, dtype=np.uint8)
    fi = code.frozen_indices()
    if fv.shape[-1] != fi.size:
        raise ValueError(f"frozen_values has length {fv.shape[-1]}, code has {fi.size} frozen positions")
    full = np.zeros(fv.shape[:-1] + (code.block_size,), np.uint8)
    full[..., fi] = fv & 1
    return full


def quantize_q88(llrs) -> np.ndarray:
    """LLRs -> saturating Q8.8 raw codes (int16): sat(rint(256 * fp32(L))), the
    representation of SPEC.md:207-212 / :269 that sc_decode_fixed consumes."""
    l = np.asarray(llrs, dtype=np.float32)
    return np.clip(np.rint(l * np.float32(256.0)), -32767, 32767).astype(np.int16)


def sc_decode_fixed(code: PolarCode, llrs_fixed, frozen_values) -> np.ndarray:
    """SC decode of raw Q8.8 LLRs (int16 codes) with saturating
    fixed-point arithmetic and the table boxplus, on the GPU (bit-exact with
    the fixed-point oracle); the codes go to the device as int16."""
    raw = np.asarray(llrs_fixed)
    if raw.dtype.kind not in "iu":
        raise ValueError("llrs_fixed must be integer Q8.8 codes (see quantize_q88)")
    if raw.shape[-1] != code.block_size:
        raise ValueError(f"llrs length {raw.shape[-1]} != 2^n = {code.block_size}")
    dev = _require_cuda()
    batch = np.clip(raw.reshape(-1, code.block_size), -32767, 32767).astype(np.int16)
    full = scatter_frozen_values(code, frozen_values).reshape(-1, code.block_size)
    if full.shape[0] not in (1, batch.shape[0]):
        raise ValueError("frozen_values batch does not match llrs")
    if full.shape[0] == 1 and batch.shape[0] > 1:
        full = np.repeat(full, batch.shape[0], axis=0)
    dec = _cached_decoder(code, batch.shape[0], "fixed")
    u, _ = dec.decode_q88(torch.from_numpy(batch).to(dev),
                          torch.from_numpy(pack_bits(full).view(np.int32).copy()).to(dev))
    torch.cuda.current_stream().synchronize()
    out = unpack_bits(u.cpu().numpy().view(np.uint32), code.block_size)
    return out.reshape(raw.shape).astype(np.uint8)


def sc_decode(code: PolarCode, llrs, frozen_values, f_mode: str = "exact") -> np.ndarray:
    """float SC decode of one block (or a [F, N] batch) on the GPU.
    llrs are rounded to fp32 (the decoder's arithmetic type)."""
    dev = _require_cuda()
    l = np.asarray(llrs, dtype=np.float64)
    if l.shape[-1] != code.block_size:
        raise ValueError(f"llrs length {l.shape[-1]} != 2^n = {code.block_size}")
    batch = l.reshape(-1, code.block_size)
    full = scatter_frozen_values(code, frozen_values).reshape(-1, code.block_size)
    if full.shape[0] not in (1, batch.shape[0]):
        raise ValueError("frozen_values batch does not match llrs")
    if full.shape[0] == 1 and batch.shape[0] > 1:
        full = np.repeat(full, batch.shape[0], axis=0)
    F = batch.shape[0]
    dec = _cached_decoder(code, F, f_mode)
    llr_t = torch.from_numpy(batch.astype(np.float32)).to(dev)
    fz_t = torch.from_numpy(pack_bits(full).view(np.int32).copy()).to(dev)
    u, _ = dec.decode(llr_t, fz_t)
    torch.cuda.current_stream().synchronize()
    out = unpack_bits(u.cpu().numpy().view(np.uint32), code.block_size)
    return out.reshape(l.shape).astype(np.uint8)
