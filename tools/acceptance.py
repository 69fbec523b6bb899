"""SPEC acceptance points on the GPU (run under gpurun; writes gpurun_out/acceptance.json
and the constructed code tables under gpurun_out/codes/):

 A. Table-1 BSC 2 % codes at target FER 0.1 built by GPU density evolution for
    n = 14..24: rate and beta = rate / (1 - h(p)) (acceptance 1-3).
 B. Monte-Carlo FER with the reference's seeded frame generators (run_trials,
    SPEC.md:382-390): n = 16, 500 trials -> [0.05, 0.14]; n = 20, 200 trials ->
    [0.05, 0.19]; n = 24, 32 trials -> [0, 0.25].
 C. Decode throughput against block size at fixed total bits (2^28 per decode, the
    c3 workload), BSC 2 %, fixed point: the N log N trend and the
    n = 16 -> 24 degradation (acceptance 8 at :505).
"""
from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1204_5882_b200 import channel as C  # noqa: E402
from paper_1204_5882_b200 import codes as K  # noqa: E402
from paper_1204_5882_b200 import construct as D  # noqa: E402
from paper_1204_5882_b200.polar_core import ScDecoder, polar_transform_words  # noqa: E402
from paper_1204_5882_b200.trials import run_trials  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")
P = 0.02


def h2(p):
    return -p * math.log2(p) - (1 - p) * math.log2(1 - p)


def build_codes(ns):
    ch = C.Bsc(P)
    os.makedirs(os.path.join(OUT, "codes"), exist_ok=True)
    rows, codes = [], {}
    for n in ns:
        t0 = time.perf_counter()
        res = D.density_evolution(ch, n)
        code = D.select_frozen(res, 0.1)
        dt = time.perf_counter() - t0
        path = os.path.join(OUT, "codes", f"bsc{P}_n{n}_fer0.1.pqct")
        K.write_code_table(code, path)
        order = np.lexsort((np.arange(res.pe.size), res.pe))
        k = code.block_size - code.frozen_count
        row = {"n": n, "rate": code.rate, "beta": code.rate / (1 - h2(P)), "K": k,
               "union_bound": float(res.pe[order[:k]].sum()), "de_seconds": round(dt, 2),
               "checksum": K.code_table_checksum(path)}
        if n == 16 and os.path.exists(os.path.join(K.CODES_DIR, "t1r1.pqct")):
            ref = K.read_code_table(os.path.join(K.CODES_DIR, "t1r1.pqct"))
            row["mask_diff_vs_reference_built"] = int(np.count_nonzero(ref.frozen_mask != code.frozen_mask))
        if n == 20 and os.path.exists(os.path.join(K.CODES_DIR, "t1r2.pqct")):
            ref = K.read_code_table(os.path.join(K.CODES_DIR, "t1r2.pqct"))
            row["mask_diff_vs_reference_built"] = int(np.count_nonzero(ref.frozen_mask != code.frozen_mask))
        rows.append(row)
        codes[n] = code
        print("code", row, flush=True)
    return rows, codes


def monte_carlo(codes):
    ch = C.Bsc(P)
    rows = []
    plan = [(16, 500, "fixed", 0.05, 0.14), (16, 500, "float", 0.05, 0.14),
            (20, 200, "fixed", 0.05, 0.19), (20, 200, "float", 0.05, 0.19), (24, 32, "fixed", 0.0, 0.25)]
    for n, trials, rep, lo, hi in plan:
        if n not in codes:
            continue
        r = run_trials(codes[n], ch, trials, seed=2012 + n, representation=rep, batch=min(trials, 256 if n <= 20 else 16))
        row = {"n": n, "trials": trials, "representation": rep, "fer_measured": r.fer_measured,
               "interval": [lo, hi], "inside": lo <= r.fer_measured <= hi,
               "throughput_mbps": round(r.throughput_mbps, 1), "wall_s": round(r.wall_time, 2), "seed": r.seed}
        rows.append(row)
        print("mc", row, flush=True)
    return rows


def throughput(codes, total_log2=28, extra=((24, 32),)):
    dev = torch.device("cuda", 0)
    rows = []
    shapes = [(n, 1 << (total_log2 - n)) for n in sorted(codes)] + [s for s in extra if s[0] in codes]
    g = torch.Generator(device=dev)
    for n, F in shapes:
        N = 1 << n
        code = codes[n]
        dec = ScDecoder(code, max_frames=F, f_mode="fixed", device=dev)
        g.manual_seed(1000 + n)
        x_w = torch.randint(-(1 << 31), (1 << 31) - 1, (F, N // 32), dtype=torch.int64, device=dev, generator=g).to(torch.int32)
        e_w = torch.zeros((F, N // 32), dtype=torch.int32, device=dev)
        sh = torch.arange(32, device=dev, dtype=torch.int64)
        step = max(1, (1 << 24) // N)
        for f0 in range(0, F, step):  # flips ~ Bernoulli(p), packed LSB-first, 2^24 bits at a time
            fl = (torch.rand((min(step, F - f0), N // 32, 32), device=dev, generator=g) < P).to(torch.int64)
            w = (fl << sh).sum(-1)
            e_w[f0:f0 + step] = torch.where(w >= (1 << 31), w - (1 << 32), w).to(torch.int32)
        y_w = x_w ^ e_w
        u_w = polar_transform_words(x_w, n)
        mag = float(np.float32(C.Bsc(P).llr_magnitude))
        xh = dec.alloc_words(F)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        ms = []
        for it in range(7):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dec.decode_bsc(y_w, mag, u_w, want_u=False, want_x=True, x_hat=xh, frames=F)
            b.record()
            torch.cuda.synchronize()
            if it >= 2:
                ms.append(a.elapsed_time(b))
        fer = float((xh != x_w).any(dim=1).float().mean().item())
        t = float(np.median(ms))
        row = {"n": n, "frames": F, "ms_per_decode": round(t, 3), "gbit_s": round(F * N / t / 1e6, 2),
               "ns_per_bit_per_level": round(t * 1e6 / (F * N * n), 5), "fer": fer, **dec.last_config}
        rows.append(row)
        print("tp", row, flush=True)
        dec.close()
        del dec, x_w, e_w, y_w, u_w, xh
        torch.cuda.empty_cache()
    return rows


if __name__ == "__main__":
    ns = [int(a) for a in sys.argv[1:]] or [14, 16, 18, 20, 22, 24]
    torch.cuda.set_device(0)
    out = {"channel": f"bsc({P})", "target_fer": 0.1}
    out["codes"], codes = build_codes(ns)
    out["throughput_fixed_total_bits"] = throughput(codes)
    by = {(r["n"], r["frames"]): r for r in out["throughput_fixed_total_bits"]}
    if (16, 1 << 12) in by and (24, 16) in by:
        out["degradation_n16_to_n24_equal_bits"] = round(by[(16, 1 << 12)]["gbit_s"] / by[(24, 16)]["gbit_s"], 3)
    if (16, 1 << 12) in by and (24, 32) in by:
        out["degradation_n16_to_n24_32frames"] = round(by[(16, 1 << 12)]["gbit_s"] / by[(24, 32)]["gbit_s"], 3)
    out["monte_carlo"] = monte_carlo(codes)
    with open(os.path.join(OUT, "acceptance.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))
