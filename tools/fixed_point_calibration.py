"""Calibration of the fixed-point decoder against SPEC.md:257 / acceptance
criterion 7 on the Table-1 row-1 code (codes/t1r1.pqct: BSC 2 %, N = 2^16,
FER-0.1 frozen set), 500 frames, seed 4242 (the frames of
tests/test_gpu_parity.py::test_fixed_spec_examples).

Prints, for the f64 float decoder (oracle), the shipped fixed-point form
(table boxplus, oracle precision 16) and the literal phi-table form
(tools/fixedpoint/phi_literal.c): FER and the fraction of frames whose outcome
(verified / discarded) agrees with the float decoder.  CPU only; ~1 minute.
Measured: float FER 0.098; table boxplus FER 0.100, agreement 0.994; literal
phi table FER 0.116, agreement 0.958.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1204_5882_b200 import channel as C  # noqa: E402
from paper_1204_5882_b200 import codes as K  # noqa: E402


def main(frames=500, seed=4242):
    code = K.read_code_table(os.path.join(ROOT, "codes", "t1r1.pqct"))
    ch, N = C.Bsc(0.02), code.block_size
    llr = np.empty((frames, N), np.float32)
    u = np.empty((frames, N), np.uint8)
    for j in range(frames):
        x, y = C.frame(ch, seed, j, N)
        llr[j] = C.channel_llr(ch, y)
        u[j] = O.polar_transform_bytes(x)
    th = O.max_threads()
    ok_f = np.all(O.sc_decode_batch(code.frozen_mask, llr, u, precision=64, threads=th) == u, axis=1)
    ok_q = np.all(O.sc_decode_batch(code.frozen_mask, llr, u, precision=16, threads=th) == u, axis=1)
    with tempfile.TemporaryDirectory() as td:
        exe = os.path.join(td, "phi_literal")
        subprocess.run(["gcc", "-O2", "-o", exe, os.path.join(ROOT, "tools", "fixedpoint", "phi_literal.c"), "-lm"],
                       check=True)
        paths = [os.path.join(td, f) for f in ("mask.bin", "llr.bin", "u.bin", "ok.bin")]
        code.frozen_mask.astype(np.uint8).tofile(paths[0])
        llr.tofile(paths[1])
        u.tofile(paths[2])
        subprocess.run([exe, str(code.n), str(frames), *paths], check=True)
        ok_p = np.fromfile(paths[3], np.uint8).astype(bool)
    print(f"float f64          FER {1 - ok_f.mean():.4f}")
    for name, ok in (("table boxplus", ok_q), ("literal phi table", ok_p)):
        print(f"{name:18s} FER {1 - ok.mean():.4f}  outcome agreement {np.mean(ok == ok_f):.4f}")


if __name__ == "__main__":
    main()
