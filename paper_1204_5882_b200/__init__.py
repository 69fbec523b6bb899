"""B200-native successive-cancellation decoding of polar codes for QKD
reconciliation -- a drop-in for the decode path of the reference package
``polarqkd`` (see DESIGN.md and INTEGRATION.md).

The decode path runs as hand-written sm_100a CUDA kernels in the in-tree
``libpolarsc.so`` behind a C ABI (include/polarsc.h); this package is the
host-side mirror of the reference's Python interface for that path.
"""
from .channel import (LLR_CLAMP, BiAwgn, Bsc, ChannelModel, channel_llr, make_rng,
                      transmit)
from .codes import (CONFIGS, PolarCode, available_configs, code_table_checksum, load_config,
                    read_code_table, write_code_table)
from .polar_core import (ScDecoder, pack_bits, phi, polar_transform, polar_transform_words,
                         quantize_q88, sc_decode, sc_decode_fixed, unpack_bits, words_per_frame)
from .reconcile import alice_disclose, bob_decode

__version__ = "0.1.0"

__all__ = [
    "LLR_CLAMP", "BiAwgn", "Bsc", "ChannelModel", "channel_llr", "make_rng", "transmit",
    "CONFIGS", "PolarCode", "available_configs", "code_table_checksum", "load_config",
    "read_code_table", "write_code_table",
    "ScDecoder", "pack_bits", "phi", "polar_transform", "polar_transform_words", "quantize_q88",
    "sc_decode", "sc_decode_fixed",
    "unpack_bits", "words_per_frame", "alice_disclose", "bob_decode", "__version__",
]
