"""Golden fixtures for the GPU density evolution, generated
from the REFERENCE itself (run only in the build container; the tests read the
committed de_ref.npz):

  pe_<tag>        reference density_evolution(ch, n) pe (construction.py:313-391,
                  default grid and pruning) for small (channel, n) points
  f_idx_digest    blake2b-64 of the reference's _GridOps f_idx / f_whi /
  f_whi_digest    z_weights / i_loss tables (default grid), so the tests can
  zw_digest       check that the package's host tables are bit-identical
  il_digest       without the reference
  base_<tag>      the reference's _base_density for the same channels
"""
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from polarqkd import construction as RK  # noqa: E402
from polarqkd.channel import BiAwgn, Bsc  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
POINTS = [("bsc002_n10", Bsc(0.02), 10), ("awgn1_n10", BiAwgn(1.0), 10),
          ("awgn0161_n12", BiAwgn(0.161), 12), ("bsc003_n12", Bsc(0.03), 12)]


def digest(a):
    return np.uint64(int.from_bytes(hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=8).digest(),
                                    "little"))


def main():
    out = {}
    ops = RK._grid_ops(RK.DeGrid())
    out["f_idx_digest"] = digest(ops.f_idx.astype(np.int32))
    out["f_whi_digest"] = digest(ops.f_whi.astype(np.float64))
    out["zw_digest"] = digest(ops.z_weights)
    out["il_digest"] = digest(ops.i_loss)
    for tag, ch, n in POINTS:
        t0 = time.time()
        out["pe_" + tag] = RK.density_evolution(ch, n).pe
        out["base_" + tag] = RK._base_density(ch, ops)
        print(tag, f"{time.time() - t0:.1f}s")
    np.savez_compressed(os.path.join(HERE, "de_ref.npz"), **out)


if __name__ == "__main__":
    main()
