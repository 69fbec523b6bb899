"""GPU density evolution vs the reference fixtures (tests/golden/de_ref.npz):
relative pe differences by pe band, frozen-set agreement, and timing of the
BASELINE configs' constructions."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1204_5882_b200 import channel as C  # noqa: E402
from paper_1204_5882_b200 import codes as K  # noqa: E402
from paper_1204_5882_b200 import construct as D  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "de_ref.npz"))
for tag, ch, n in [("bsc002_n10", C.Bsc(0.02), 10), ("awgn1_n10", C.BiAwgn(1.0), 10),
                   ("awgn0161_n12", C.BiAwgn(0.161), 12), ("bsc003_n12", C.Bsc(0.03), 12)]:
    ref = g["pe_" + tag]
    t0 = time.perf_counter()
    pe = D.density_evolution(ch, n).pe
    dt = time.perf_counter() - t0
    rel = np.abs(pe - ref) / np.maximum(ref, 1e-300)
    out = [f"{tag}: {dt:.2f}s"]
    for lo in (1e-2, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12):
        sel = ref >= lo
        out.append(f"pe>={lo:g}: {rel[sel].max():.2e}")
    print("  ".join(out))
for key in sys.argv[1:]:
    cfg = K.CONFIGS[key]
    code = K.load_config(key)
    t0 = time.perf_counter()
    res = D.density_evolution(cfg.channel, code.n)
    dt = time.perf_counter() - t0
    got = D.select_rate(res, cfg.rate)
    diff = int(np.count_nonzero(got.frozen_mask != code.frozen_mask))
    print(f"{key}: n={code.n} GPU DE {dt:.1f}s, frozen-set positions differing from the reference's: {diff}")
