"""Per-level cycle attribution of the single-warp band (needs a library built
with PQ_UBENCH_TIMING and the pq_debug_ub export; see tools/build_variant.sh):
python tools/ub_profile.py --config c3 --fmode fixed   (PQ_LIB_PATH=variants/vUB.so)
Slots: 0 dec8 generic, 1 dec32, 2 warp_walk, 3 dec16 generic, 4 dec8 pattern,
5 dec8 R1/REP/R0, 6 dec16 R1/REP/R0.  Cycles summed over frames (lane 0)."""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1204_5882_b200.channel import frames_batch  # noqa: E402
from paper_1204_5882_b200 import _lib, codes as K  # noqa: E402
from paper_1204_5882_b200.polar_core import ScDecoder, pack_bits, polar_transform_words  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--fmode", default="fixed")
ap.add_argument("--frames", type=int, default=0)
a = ap.parse_args()
cfg = K.CONFIGS[a.config]
code = K.load_config(a.config)
F = a.frames or cfg.frames_per_gpu
x, llr, _ = frames_batch(cfg.channel, cfg.seed, 0, F, code.block_size, want_y=False)
dev = torch.device("cuda", 0)
u = polar_transform_words(torch.from_numpy(pack_bits(x).view(np.int32).copy()).to(dev), code.n)
dec = ScDecoder(code, max_frames=F, f_mode=a.fmode)
l = torch.from_numpy(llr).to(dev)
L = _lib.load()
buf = (ctypes.c_ulonglong * 32)()
dec.decode(l, u)
L.pq_debug_ub(buf, 1)
dec.decode(l, u)
torch.cuda.synchronize()
L.pq_debug_ub(buf, 1)
names = ["dec8 generic", "dec32", "warp_walk", "dec16 generic", "dec8 pattern", "dec8 special", "dec16 special"]
for i, nm in enumerate(names):
    t, c = buf[i], buf[16 + i]
    print(f"{nm:16s} cycles/frame {t / F:14.0f}  calls/frame {c / F:9.1f}  cycles/call {t / max(c, 1):8.1f}")
