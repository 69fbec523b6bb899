"""ctypes binding to the in-tree C-ABI library (include/polarsc.h).

There is deliberately no fallback: if libpolarsc.so is missing or no CUDA
device is present, every decode/transform call raises.  The CPU oracle under
oracle/ is test infrastructure and is never reachable from here.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PQ_LIB_PATH: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("PQ_LIB_PATH") or os.path.join(HERE, "libpolarsc.so")

PQ_F_EXACT = 0
PQ_F_MINSUM = 1
PQ_F_FAST = 2
PQ_F_FIXED = 3
PQ_OPT_SSC = 1
PQ_OPT_SUBTREE_LOG2 = 2
PQ_OPT_FMODE = 3
PQ_OPT_PROFILE = 4
PQ_OPT_WARP_LOG2 = 5
PQ_OPT_CLUSTER = 6
PQ_OPT_THREADS = 7
PQ_OPT_TIMING = 8
PQ_PROF_SLOTS = 16
PROF_NAMES = ("upper_f", "upper_g", "upper_other", "smem_f", "smem_g", "smem_other", "warp_subtrees",
              "type_staging", "rate1_block", "total", "n_warp_subtrees", "n_block_nodes",
              "w32_cycles", "w32_calls", "unused")

# every symbol include/polarsc.h declares (tests check the .so exports them)
EXPORTS = (
    "pq_decoder_create", "pq_decoder_set_frozen_mask", "pq_decoder_set_option",
    "pq_decoder_get_option", "pq_sc_decode_f32", "pq_sc_decode_f32_dump", "pq_sc_decode_bsc",
    "pq_polar_transform", "pq_decoder_workspace_bytes", "pq_decoder_last_launches",
    "pq_decoder_destroy", "pq_last_error", "pq_abi_version", "pq_decoder_read_profile",
    "pq_debug_fmag", "pq_decoder_last_ctas_per_frame", "pq_decoder_last_config", "pq_sc_decode_q88",
    "pq_decoder_kernel_times", "pq_read_code_table", "pq_blake2b64", "pq_hash_frames", "pq_verify_frames", "pq_xxh64", "pq_de_create", "pq_de_run", "pq_de_destroy",
    "pq_bsc_frames", "pq_pcg64_seed",
)

_lib = None


class PolarScError(RuntimeError):
    pass


def load():
    """Load libpolarsc.so (raises if it is absent -- build() first)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise PolarScError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i, u32p = ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p
    L.pq_decoder_create.argtypes = [ctypes.POINTER(vp), i, i, i, i]
    L.pq_decoder_set_frozen_mask.argtypes = [vp, ctypes.c_char_p]
    L.pq_decoder_set_option.argtypes = [vp, i, i]
    L.pq_decoder_get_option.argtypes = [vp, i]
    L.pq_sc_decode_f32.argtypes = [vp, vp, u32p, u32p, u32p, i, vp]
    L.pq_sc_decode_f32_dump.argtypes = [vp, vp, u32p, u32p, u32p, vp, i, vp]
    L.pq_sc_decode_q88.argtypes = [vp, vp, u32p, u32p, u32p, i, vp]
    L.pq_sc_decode_bsc.argtypes = [vp, u32p, ctypes.c_float, u32p, u32p, u32p, i, vp]
    L.pq_polar_transform.argtypes = [u32p, u32p, i, i, vp]
    L.pq_decoder_workspace_bytes.argtypes = [vp]
    L.pq_decoder_workspace_bytes.restype = ctypes.c_size_t
    L.pq_decoder_last_launches.argtypes = [vp]
    L.pq_decoder_last_ctas_per_frame.argtypes = [vp]
    L.pq_decoder_last_config.argtypes = [vp, vp, vp, vp]
    L.pq_decoder_destroy.argtypes = [vp]
    L.pq_decoder_read_profile.argtypes = [vp, vp, i]
    L.pq_decoder_kernel_times.argtypes = [vp, vp, i]
    L.pq_read_code_table.argtypes = [ctypes.c_char_p, vp, vp, vp, vp, vp, vp, ctypes.c_size_t]
    L.pq_blake2b64.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
    L.pq_blake2b64.restype = ctypes.c_uint64
    L.pq_debug_fmag.argtypes = [i, vp, vp, vp, i, vp]
    L.pq_hash_frames.argtypes = [u32p, i, i, ctypes.c_uint64, vp, vp]
    L.pq_verify_frames.argtypes = [u32p, i, i, ctypes.c_uint64, vp, vp, vp, vp]
    L.pq_xxh64.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_uint64]
    L.pq_xxh64.restype = ctypes.c_uint64
    dbl = ctypes.c_double
    L.pq_de_create.argtypes = [ctypes.POINTER(vp), i, dbl, vp, vp, vp, vp, i]
    L.pq_de_run.argtypes = [vp, vp, i, dbl, dbl, dbl, vp]
    L.pq_de_destroy.argtypes = [vp]
    L.pq_bsc_frames.argtypes = [i, ctypes.c_uint64, ctypes.c_uint64, i, dbl, u32p, u32p, vp]
    L.pq_pcg64_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64, vp]
    L.pq_last_error.restype = ctypes.c_char_p
    L.pq_abi_version.restype = ctypes.c_int
    for name in EXPORTS:
        getattr(L, name)
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    """Map C-ABI return codes onto the reference's error behaviour:
    negative -> ValueError (bad arguments, as the reference raises), positive
    -> PolarScError (CUDA failure)."""
    if rc == 0:
        return
    msg = load().pq_last_error().decode(errors="replace")
    if rc < 0:
        raise ValueError(f"{what}: {msg}")
    raise PolarScError(f"{what}: {msg} (rc={rc})")
