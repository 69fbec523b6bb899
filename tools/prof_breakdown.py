"""Per-step-class cycle breakdown of one decode (PQ_OPT_PROFILE)."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1204_5882_b200.channel import frames_batch  # noqa: E402
from paper_1204_5882_b200 import _lib  # noqa: E402
from paper_1204_5882_b200 import codes as K  # noqa: E402
from paper_1204_5882_b200.polar_core import ScDecoder, pack_bits, polar_transform_words  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["c1", "c2"])
ap.add_argument("--frames", type=int, default=0)
ap.add_argument("--subtree-log2", type=int, default=0)
ap.add_argument("--warp-log2", type=int, default=8)
ap.add_argument("--fmode", default="exact")
a = ap.parse_args()
dev = torch.device("cuda", 0)
for key in a.configs:
    cfg = K.CONFIGS[key]
    code = K.load_config(key)
    F = a.frames or cfg.frames_per_gpu
    x, llr, _ = frames_batch(cfg.channel, cfg.seed, 0, F, code.block_size, want_y=False)
    u = polar_transform_words(torch.from_numpy(pack_bits(x).view(np.int32).copy()).to(dev), code.n)
    dec = ScDecoder(code, max_frames=F, subtree_log2=a.subtree_log2, f_mode=a.fmode)
    dec.set_option(_lib.PQ_OPT_WARP_LOG2, a.warp_log2)
    l = torch.from_numpy(llr).to(dev)
    dec.decode(l, u)
    dec.set_option(_lib.PQ_OPT_PROFILE, 1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    dec.decode(l, u)
    e.record()
    torch.cuda.synchronize()
    pr = dec.read_profile(F).astype(np.float64)
    tot = pr[:, 9].mean()
    print(f"== {key}: F={F} N=2^{code.n}  batch {s.elapsed_time(e):.3f} ms (with profiling)  "
          f"mean frame cycles {tot:.0f} (max {pr[:, 9].max():.0f})")
    for q, name in enumerate(_lib.PROF_NAMES):
        if q in (9,):
            continue
        v = pr[:, q].mean()
        if q >= 10 and q != 12:
            print(f"   {name:16s} {v:12.0f}")
        else:
            print(f"   {name:16s} {v:12.0f} cycles  {100 * v / tot:5.1f}%")
