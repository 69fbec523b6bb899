"""Small decodes at the production launch shapes, for compute-sanitizer
(tools/sanitize.sh): single-CTA 256 threads, 128-thread CTAs, clusters of 4
CTAs with 512 threads, clusters of 2 with 256; fixed point and exact f; the
fp32, Q8.8 and BSC inputs.  Each decode is checked against the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402  (the checker)
from paper_1204_5882_b200 import _lib  # noqa: E402
from paper_1204_5882_b200 import channel as C  # noqa: E402
from paper_1204_5882_b200 import codes as K  # noqa: E402
from paper_1204_5882_b200.polar_core import ScDecoder, pack_bits, unpack_bits  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(9)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 15
N = 1 << n
mask = (rng.random(N) < 0.45).astype(np.uint8)
mask[: N // 8] = 1
code = K.PolarCode(n=n, frozen_mask=mask, channel=C.Bsc(0.05), target_fer=0.1)
F = 3
x = rng.integers(0, 2, (F, N), dtype=np.uint8)
y = x ^ (rng.random((F, N)) < 0.05).astype(np.uint8)
llr = C.channel_llr(C.Bsc(0.05), y).astype(np.float32)
llr += rng.normal(0, 0.7, llr.shape).astype(np.float32)  # weak / strong mix: rate-1 guards pass and fail
u = np.array([O.polar_transform_bytes(xi) for xi in x])
uw = torch.from_numpy(pack_bits(u).view(np.int32).copy()).to(dev)
shapes = [(1, 256, 13), (1, 128, 12), (4, 0, 11), (2, 256, 11), (1, 64, 11)]
if os.environ.get("PQ_SHAPES"):  # "cluster,threads,log2S;..." (e.g. the fused / warp-release ring builds)
    shapes = [tuple(int(v) for v in t.split(",")) for t in os.environ["PQ_SHAPES"].split(";")]
modes = ("fixed",) if os.environ.get("PQ_FIXED_ONLY") else ("fixed", "exact")
bad = 0
for fmode in modes:
    prec = 16 if fmode == "fixed" else 32
    ref = O.sc_decode_batch(mask, llr, u, precision=prec, threads=8)
    for ncl, thr, lg in shapes:
        dec = ScDecoder(code, max_frames=F, f_mode=fmode, subtree_log2=lg)
        dec.set_option(_lib.PQ_OPT_CLUSTER, ncl)
        dec.set_option(_lib.PQ_OPT_THREADS, thr)
        uh, _ = dec.decode(torch.from_numpy(llr).to(dev), uw)
        got = unpack_bits(uh.cpu().numpy().view(np.uint32), N)
        cfg = dec.last_config
        ok = np.array_equal(got, ref)
        bad += not ok
        print(f"{fmode} cluster={ncl} threads={cfg['threads_per_cta']} S=2^{cfg['subtree_log2']} "
              f"K={cfg['ctas_per_frame']}: {'ok' if ok else 'MISMATCH'}", flush=True)
        if fmode == "fixed" and ncl == 1 and thr == 256:
            q = torch.from_numpy(O.quantize_q88(llr)).to(dev)
            u2, _ = dec.decode_q88(q, uw)
            yw = torch.from_numpy(pack_bits(y).view(np.int32).copy()).to(dev)
            u3, _ = dec.decode_bsc(yw, float(C.Bsc(0.05).llr_magnitude), uw)
            torch.cuda.synchronize()
            print("  q88 + bsc front ends ran", flush=True)
sys.exit(1 if bad else 0)
