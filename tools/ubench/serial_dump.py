"""Real inputs of the single-warp band for tools/ubench/serial_bench.cu.

Decodes frames of a BASELINE config with the fixed-point oracle (all-zero
frozen values, so the textbook and the GPU's coset-shifted domains coincide),
takes the stage dump, and writes every node the warp band is handed -- the
visited non-rate-0 nodes of width WMAX (2048) -- in decode order.

File (little endian): header int32 n, wl, frames, nodes; then per frame and
node one record: int32 d0, uint32 j, int16 vals[W] (the node's Q8.8 LLRs),
uint32 expect[W/32] (T_W(u-hat of the node)), uint8 ty[2W] (the node's local
heap-order types, index (1 << e) + jj), uint32 fm[W/32] (frozen-mask words).
Output: tools/ubench/data/serial_<cfg>.bin

python tools/ubench/serial_dump.py [cfg=c3] [frames=2] [wmax_log2=11]
"""
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from oracle import oracle as O  # noqa: E402
from paper_1204_5882_b200 import channel as C  # noqa: E402
from paper_1204_5882_b200 import codes as K  # noqa: E402
from paper_1204_5882_b200.polar_core import pack_bits  # noqa: E402
from tree_stats import types, visited  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = int(sys.argv[3]) if len(sys.argv) > 3 else 11
cfg = K.CONFIGS[key]
code = K.load_config(key)
mask = code.frozen_mask.astype(np.uint8)
n, N = code.n, code.block_size
W = 1 << wl
d0 = n - wl
ty = types(mask)
vis = visited(ty)
nodes = [int(j) for j in np.nonzero(vis[d0])[0] if ty[d0][j] != 1]  # rate-0 nodes are zeroed by the block loop
local = {}
for j in nodes:
    t = np.zeros(2 * W, np.uint8)
    for e in range(wl + 1):
        t[(1 << e):(2 << e)] = ty[d0 + e][j << e:(j + 1) << e]
    local[j] = t.tobytes() + pack_bits(mask[j * W:(j + 1) * W]).tobytes()
rng = np.random.default_rng(77)
out = bytearray()
out += struct.pack("<iiii", n, wl, frames, len(nodes))
for f in range(frames):
    u = (rng.random(N) < 0.5).astype(np.uint8) * (1 - mask)
    x = O.polar_transform_bytes(u)
    if isinstance(cfg.channel, C.Bsc):
        y = x ^ (rng.random(N) < cfg.channel.p).astype(np.uint8)
    else:
        y = (1.0 - 2.0 * x) + rng.normal(0.0, np.sqrt(cfg.channel.sigma2), N)
    llr = C.channel_llr(cfg.channel, y).astype(np.float32)
    raw = O.quantize_q88(llr)
    uh, xh, st = O.sc_decode_fixed(mask, raw, np.zeros(N, np.uint8), dump=True)
    print(f"frame {f}: {'ok' if np.array_equal(uh, u) else 'decoding error'}; {len(nodes)} warp-band nodes of width {W}")
    for j in nodes:
        vals = st[d0, j * W:(j + 1) * W].astype(np.int16)
        xw = O.polar_transform_bytes(uh[j * W:(j + 1) * W])
        out += struct.pack("<iI", d0, j)
        out += vals.tobytes()
        out += pack_bits(xw).tobytes()
        out += local[j]
os.makedirs(os.path.join(ROOT, "tools", "ubench", "data"), exist_ok=True)
path = os.path.join(ROOT, "tools", "ubench", "data", f"serial_{key}.bin")
open(path, "wb").write(out)
print("->", path, len(out), "bytes")
