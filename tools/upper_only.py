"""Upper band in isolation: a code whose width-S blocks alternate rate-0 /
rate-1 keeps every level above S mixed (full HBM streaming) while the
shared-memory sub-trees cost almost nothing.  Prints the time per decode and
the algorithmic upper-band bandwidth (12.3125 N B per level)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1204_5882_b200 import channel as C  # noqa: E402
from paper_1204_5882_b200 import codes as K  # noqa: E402
from paper_1204_5882_b200.polar_core import ScDecoder  # noqa: E402

n, F = 20, int(sys.argv[1]) if len(sys.argv) > 1 else 256
fmode = sys.argv[2] if len(sys.argv) > 2 else "fixed"
N = 1 << n
dev = torch.device("cuda", 0)
for log2S in (13,):
    S = 1 << log2S
    mask = np.zeros(N, np.uint8)
    for b in range(N // S):
        if b % 2 == 0:
            mask[b * S:(b + 1) * S] = 1
    code = K.PolarCode(n=n, frozen_mask=mask, channel=C.Bsc(0.02), target_fer=0.1)
    dec = ScDecoder(code, max_frames=F, f_mode=fmode, subtree_log2=log2S)
    llr = (torch.rand(F, N, device=dev) * 8 + 8) * torch.where(torch.rand(F, N, device=dev) < 0.02, -1.0, 1.0)
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
    print(f"F={F} S=2^{log2S} {fmode}: {t * 1e3:.3f} ms per decode, upper-band algorithmic {alg / t / 1e9:.0f} GB/s")
