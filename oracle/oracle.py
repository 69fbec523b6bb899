"""TEST INFRASTRUCTURE ONLY -- Python face of the CPU oracle.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module; the product package never does.

Contents
--------
* ctypes bindings to ``oracle/liboracle.so`` (the C restatement of
  SPEC.md:202-285, see sc_oracle.c for the per-rule citations);
* ``sc_decode_recursive`` -- a second, independent restatement in plain
  numpy (textbook recursion), used to cross-check the C walk;
* ``sc_decode_naive`` -- the "straightforward non-recursive reference SC
  implementation" SPEC.md:248 asks for: each bit-channel LLR is obtained by
  brute-force marginalisation over the future bits,
  L_i = ln sum_{u>i} prod_j P(y_j|x_j(u<i,0,u>i)) - ln sum_{u>i} prod_j P(y_j|x_j(u<i,1,u>i)),
  which in exact arithmetic equals Arikan's recursion with the exact f; it pins
  both the recursion and the f formula (usable for N <= 16);
* ``polar_transform_bytes`` / ``phi`` / ``phi_table`` -- SPEC.md:220-238.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

F_EXACT, F_MINSUM = 0, 1

_lib = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no fast-math)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        L.orc_polar_transform.argtypes = [ctypes.c_int, u8p]
        L.orc_polar_transform.restype = None
        L.orc_sc_decode_f64.argtypes = [ctypes.c_int, u8p, f64p, u8p, ctypes.c_int, u8p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_sc_decode_f32.argtypes = [ctypes.c_int, u8p, f32p, u8p, ctypes.c_int, u8p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_sc_decode_batch.argtypes = [ctypes.c_int, u8p, ctypes.c_int, f32p, u8p,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p,
                                          ctypes.c_void_p]
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_fmag_f32.argtypes = [ctypes.c_float, ctypes.c_float]
        L.orc_fmag_f32.restype = ctypes.c_float
        L.orc_fmag_f64.argtypes = [ctypes.c_double, ctypes.c_double]
        L.orc_fmag_f64.restype = ctypes.c_double
        L.orc_fmag_f32_vec.argtypes = [f32p, f32p, f32p, ctypes.c_size_t]
        i16p = np.ctypeslib.ndpointer(np.int16, flags="C_CONTIGUOUS")
        L.orc_phi_table.argtypes = [i16p]
        L.orc_corr_table.argtypes = [i16p]
        L.orc_quantize.argtypes = [ctypes.c_float]
        L.orc_quantize.restype = ctypes.c_int16
        L.orc_sc_decode_fixed.argtypes = [ctypes.c_int, u8p, i16p, u8p, u8p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p]
        L.orc_fmag_f64_vec.argtypes = [f64p, f64p, f64p, ctypes.c_size_t]
        L.orc_xxh64.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_uint64]
        L.orc_xxh64.restype = ctypes.c_uint64
        _lib = L
    return _lib


# --------------------------------------------------------------------------
# verification hash (XXH64, seed-keyed; sc_oracle.c orc_xxh64)

def xxh64(data: bytes, seed: int = 0) -> int:
    return int(lib().orc_xxh64(bytes(data), len(data), seed & (2 ** 64 - 1)))


def block_hash_words(words, seed: int = 0) -> int:
    """XXH64 of one frame's packed uint32 words as little-endian bytes."""
    return xxh64(np.ascontiguousarray(np.asarray(words, dtype="<u4")).tobytes(), seed)


# --------------------------------------------------------------------------
# transform / phi

def polar_transform_bytes(u) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(u, dtype=np.uint8) & 1).copy()
    n = int(np.log2(v.size))
    if v.size != 1 << n:
        raise ValueError("length must be a power of two")
    lib().orc_polar_transform(n, v)
    return v


def polar_transform_numpy(u) -> np.ndarray:
    """Independent numpy restatement (recursive G_N = [[G, 0], [G, G]])."""
    v = np.asarray(u, dtype=np.uint8) & 1
    if v.size == 1:
        return v.copy()
    h = v.size // 2
    a, b = polar_transform_numpy(v[:h]), polar_transform_numpy(v[h:])
    return np.concatenate([a ^ b, b])


def phi(x):
    """phi(x) = -ln(tanh(x/2)), x > 0."""
    x = np.asarray(x, dtype=np.float64)
    if np.any(x <= 0):
        raise ValueError("phi requires x > 0")
    return -np.log(np.tanh(x / 2.0))


def fmag64(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.empty_like(a)
    lib().orc_fmag_f64_vec(a, b, out, a.size)
    return out


def fmag32(a, b):
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    out = np.empty_like(a)
    lib().orc_fmag_f32_vec(a, b, out, a.size)
    return out


# --------------------------------------------------------------------------
# SC decoders

def sc_decode(mask, llr, frozen_u, precision=64, fmode=F_EXACT, dump=False, leaf=False):
    """One frame.  mask: N uint8 (1 = frozen); llr: N LLRs (cast to the chosen
    precision); frozen_u: N uint8 revealed u-values (read at frozen positions).
    Returns (u_hat, x_hat[, stages][, leaf]) with stages[(n+1), N] if dump and
    the N decision LLRs if leaf."""
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    N = mask.size
    n = int(np.log2(N))
    fz = np.ascontiguousarray(frozen_u, dtype=np.uint8)
    u = np.empty(N, np.uint8)
    x = np.empty(N, np.uint8)
    if precision == 64:
        l = np.ascontiguousarray(llr, dtype=np.float64)
        st = np.zeros((n + 1, N), np.float64) if dump else None
        lf = np.zeros(N, np.float64) if leaf else None
        rc = lib().orc_sc_decode_f64(n, mask, l, fz, fmode, u, x.ctypes.data,
                                     st.ctypes.data if dump else None,
                                     lf.ctypes.data if leaf else None)
    else:
        l = np.ascontiguousarray(llr, dtype=np.float32)
        st = np.zeros((n + 1, N), np.float32) if dump else None
        lf = np.zeros(N, np.float32) if leaf else None
        rc = lib().orc_sc_decode_f32(n, mask, l, fz, fmode, u, x.ctypes.data,
                                     st.ctypes.data if dump else None,
                                     lf.ctypes.data if leaf else None)
    if rc != 0:
        raise MemoryError("oracle decode failed")
    out = (u, x)
    if dump:
        out += (st,)
    if leaf:
        out += (lf,)
    return out


def sc_decode_batch(mask, llr, frozen_u, precision=64, fmode=F_EXACT, threads=1, min_info=False):
    """[F][N] fp32 LLRs, [F][N] uint8 frozen u-values -> [F][N] uint8 u_hat
    (and, if min_info, [F] smallest |decision LLR| over information bits)."""
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    llr = np.ascontiguousarray(llr, dtype=np.float32)
    fz = np.ascontiguousarray(frozen_u, dtype=np.uint8)
    F, N = llr.shape
    out = np.empty((F, N), np.uint8)
    mi = np.full(F, np.inf) if min_info else None
    rc = lib().orc_sc_decode_batch(int(np.log2(N)), mask, F, llr, fz, fmode, precision,
                                   threads, out, mi.ctypes.data if min_info else None)
    if rc != 0:
        raise MemoryError("oracle batch decode failed")
    return (out, mi) if min_info else out


def corr_table_q88() -> np.ndarray:
    """The fixed-point f's table: CORR[k] = rint(256 ln(1 + e^(-k/256))), k = 0..4096."""
    out = np.zeros(4097, np.int16)
    lib().orc_corr_table(out)
    return out


def phi_table_q88() -> np.ndarray:
    """The oracle's Q8.8 phi table (4097 entries, index = raw magnitude code)."""
    out = np.zeros(4097, np.int16)
    lib().orc_phi_table(out)
    return out


def quantize_q88(llr) -> np.ndarray:
    """fp32 LLRs -> saturating Q8.8 raw int16 (rint(L * 256), |raw| <= 32767)."""
    l = np.asarray(llr, np.float32)
    r = np.rint(l * np.float32(256.0))
    return np.clip(r, -32767, 32767).astype(np.int16)


def sc_decode_fixed(mask, llr_raw, frozen_u, dump=False, leaf=False):
    """SPEC.md:250-258 fixed-point SC on raw Q8.8 LLRs.  Returns (u, x[, stages][, leaf])."""
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    N = mask.size
    n = int(np.log2(N))
    l = np.ascontiguousarray(llr_raw, dtype=np.int16)
    fz = np.ascontiguousarray(frozen_u, dtype=np.uint8)
    u = np.empty(N, np.uint8)
    x = np.empty(N, np.uint8)
    st = np.zeros((n + 1, N), np.int16) if dump else None
    lf = np.zeros(N, np.int16) if leaf else None
    rc = lib().orc_sc_decode_fixed(n, mask, l, fz, u, x.ctypes.data, st.ctypes.data if dump else None,
                                   lf.ctypes.data if leaf else None)
    if rc != 0:
        raise MemoryError("oracle decode failed")
    out = (u, x)
    if dump:
        out += (st,)
    if leaf:
        out += (lf,)
    return out


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _fmag_exact(a, b):
    # log((1 + e^-a e^-b) / (e^-a + e^-b)) in numpy float64
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    return np.log1p(-np.expm1(-lo) * -np.expm1(-hi) / (np.exp(-lo) + np.exp(-hi)))


def sc_decode_recursive(mask, llr, frozen_u, fmode=F_EXACT):
    """Textbook recursive SC in numpy float64 (independent of the C walk)."""
    mask = np.asarray(mask, np.uint8)
    fz = np.asarray(frozen_u, np.uint8)
    u_hat = np.zeros(mask.size, np.uint8)

    def f(a, b):
        mag = np.minimum(np.abs(a), np.abs(b)) if fmode == F_MINSUM else _fmag_exact(np.abs(a), np.abs(b))
        return np.where(np.signbit(a) != np.signbit(b), -mag, mag)

    def rec(L, off):
        W = L.size
        if W == 1:
            u = fz[off] if mask[off] else np.uint8(L[0] < 0)
            u_hat[off] = u
            return np.array([u], np.uint8)
        h = W // 2
        a, b = L[:h], L[h:]
        xl = rec(f(a, b), off)
        xr = rec(np.where(xl == 1, b - a, b + a), off + h)
        return np.concatenate([xl ^ xr, xr])

    x = rec(np.asarray(llr, np.float64), 0)
    return u_hat, x


def sc_decode_naive(mask, llr, frozen_u):
    """Brute-force bit-channel SC ("straightforward non-recursive
    reference SC"), exact likelihoods, N <= 16.  Returns (u_hat, leaf_llrs)."""
    mask = np.asarray(mask, np.uint8)
    fz = np.asarray(frozen_u, np.uint8)
    L = np.asarray(llr, np.float64)
    N = mask.size
    if N > 16:
        raise ValueError("naive SC is exponential; N <= 16")
    # generator rows of G_N = F^{(x)n}: row i is T(e_i)
    G = np.array([polar_transform_numpy(np.eye(N, dtype=np.uint8)[i]) for i in range(N)])
    u_hat = np.zeros(N, np.uint8)
    leaf = np.zeros(N)
    for i in range(N):
        nf = N - i - 1
        futures = ((np.arange(1 << nf)[:, None] >> np.arange(nf)) & 1).astype(np.uint8)
        ll = []
        for ui in (0, 1):
            U = np.zeros((futures.shape[0], N), np.uint8)
            U[:, :i] = u_hat[:i]
            U[:, i] = ui
            U[:, i + 1:] = futures
            X = (U.astype(np.int64) @ G) & 1
            # log P(y|x) up to a y-only constant: (1 - 2x) L / 2
            s = ((1 - 2 * X) * L[None, :] / 2.0).sum(axis=1)
            ll.append(np.logaddexp.reduce(s))
        d = ll[0] - ll[1]
        # exact ties (common on the BSC) come out as +-1e-16 from the two
        # log-sum-exps; snap them to 0 so the tie rule L < 0 applies as in SC
        leaf[i] = 0.0 if abs(d) < 1e-12 * (1.0 + abs(ll[0])) else d
        u_hat[i] = fz[i] if mask[i] else np.uint8(leaf[i] < 0)
    return u_hat, leaf


# --------------------------------------------------------------------------
# fixed-point phi table: 4096 entries uniform on (0, 16]

def phi_table() -> np.ndarray:
    """Entry k (k = 1..4096) is phi(k * 2^-8) rounded to Q8.8; entry 0 = phi(0+)
    saturated to the largest Q8.8 magnitude (the table index is the raw Q8.8
    magnitude code)."""
    k = np.arange(4097, dtype=np.float64)
    x = np.maximum(k, 1e-300) * 2.0 ** -8
    val = np.where(k == 0, np.inf, -np.log(np.tanh(x / 2.0)))
    q = np.minimum(np.round(val * 256.0), 32767)
    return q.astype(np.int16)
