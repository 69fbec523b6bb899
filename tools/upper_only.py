"""Upper band in isolation: a code whose width-S blocks alternate rate-0 /
rate-1 keeps every level above S mixed (full HBM streaming) while the
shared-memory sub-trees cost almost nothing.  Prints the time per decode and
the algorithmic upper-band bandwidth (12.3125 N B per level).

python tools/upper_only.py [frames=256] [fmode=fixed] [--json out.json]
Under ncu (tools/capture_upper_only.sh) the 4th decode is the captured one."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1204_5882_b200 import channel as C  # noqa: E402
from paper_1204_5882_b200 import codes as K  # noqa: E402
from paper_1204_5882_b200.polar_core import ScDecoder  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n, F = 20, int(args[0]) if args else 256
fmode = args[1] if len(args) > 1 else "fixed"
N = 1 << n
log2S = 13
dev = torch.device("cuda", 0)
S = 1 << log2S
mask = np.zeros(N, np.uint8)
for b in range(N // S):
    if b % 2 == 0:
        mask[b * S:(b + 1) * S] = 1
code = K.PolarCode(n=n, frozen_mask=mask, channel=C.Bsc(0.02), target_fer=0.1)
dec = ScDecoder(code, max_frames=F, f_mode=fmode, subtree_log2=log2S)
g = torch.Generator(device=dev).manual_seed(5)
llr = (torch.rand(F, N, device=dev, generator=g) * 8 + 8) * torch.where(
    torch.rand(F, N, device=dev, generator=g) < 0.02, -1.0, 1.0)
fz = torch.zeros(F, N // 32, dtype=torch.int32, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
for _ in range(3):
    dec.decode(llr, fz)
ts = []
for i in range(5):
    flush.fill_(i)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dec.decode(llr, fz, want_u=False)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 1e3)
t = sorted(ts)[len(ts) // 2]
alg = 12.3125 * N * (n - log2S) * F
res = {"frames": F, "N": N, "subtree_log2": log2S, "fmode": fmode, "ms_per_decode": round(t * 1e3, 3),
       "alg_bytes_per_launch": alg, "alg_GBps": round(alg / t / 1e9, 1)}
print(json.dumps(res))
