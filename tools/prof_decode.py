"""One warm decode of a config for profilers (ncu / compute-sanitizer).

python tools/prof_decode.py --config c2 --frames 148 [--reps 2] [--fmode exact] [--no-ssc]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1204_5882_b200.channel import frames_batch  # noqa: E402
from paper_1204_5882_b200 import codes as K  # noqa: E402
from paper_1204_5882_b200.polar_core import ScDecoder, pack_bits, polar_transform_words  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--frames", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--fmode", default="fast")
ap.add_argument("--no-ssc", action="store_true")
ap.add_argument("--subtree-log2", type=int, default=0)
a = ap.parse_args()
cfg = K.CONFIGS[a.config]
code = K.load_config(a.config)
F = a.frames or cfg.frames_per_gpu
x, llr, _ = frames_batch(cfg.channel, cfg.seed, 0, F, code.block_size, want_y=False)
dev = torch.device("cuda", 0)
u = polar_transform_words(torch.from_numpy(pack_bits(x).view(np.int32).copy()).to(dev), code.n)
dec = ScDecoder(code, max_frames=F, f_mode=a.fmode, ssc=not a.no_ssc, subtree_log2=a.subtree_log2)
l = torch.from_numpy(llr).to(dev)
for _ in range(a.reps):
    uh, _ = dec.decode(l, u)
torch.cuda.synchronize()
print("frame errors", int((uh != u).any(dim=1).sum()), "of", F)
