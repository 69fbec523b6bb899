"""SC-decode throughput bench (BASELINE.json metric: SC-decoded Mbit/s).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

A step = one batched decode of this rank's frames of the config (c3 by
default: BSC p=0.02, N=2^20, rate 0.83, 256 frames per GPU, the reference's
own frozen set).  Mbit/s = frames * N / seconds / 1e6 (block bits).

  value    device-resident fp32 LLRs (+ revealed frozen words) in HBM, u-hat
           written to HBM, CUDA events on the launching stream, L2 flushed
           (256 MiB write) between timed steps, max over ranks.
  e2e      the public API with host buffers: each step copies Bob's inputs from
           pinned host memory (BSC: received bits packed 1 bit/symbol, decoded
           by the fused front end; BIAWGN: fp32 LLRs) plus the revealed frozen
           words, decodes, and copies u-hat back.
Multi-GPU (torchrun): frames shard by index (rank r takes frames
[r*F, (r+1)*F)), no collective on the hot path; NCCL all-reduces the frame
error counts afterwards (scaling: weak).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_MBPS = {"c3": 9.5}  # BASELINE.md / PAPER.md:170: SC decode, BSC 2%, N=2^20, 1 core i5-670


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--frames", type=int, default=0, help="frames per GPU (default: the config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fmode", default="fixed", choices=["exact", "fast", "fixed", "min-sum"])
    ap.add_argument("--no-ssc", action="store_true")
    ap.add_argument("--threads", type=int, default=0, choices=[0, 64, 128, 256], help="threads per CTA (0 = auto)")
    ap.add_argument("--cluster", type=int, default=0, choices=[0, 1, 2, 4, 8], help="CTAs per frame (0 = auto)")
    ap.add_argument("--subtree-log2", type=int, default=0, help="log2 of the shared-memory sub-tree width S (0 = auto)")
    ap.add_argument("--warp-log2", type=int, default=0, help="widest node of the single-warp band, log2 (0 = default)")
    ap.add_argument("--cpu-sample-s", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def gen_frames(cfg, N, j0, F):
    """Bob's inputs for frames j0..j0+F-1 (seed convention of channel.frame)."""
    from paper_1204_5882_b200 import channel as C

    x = np.empty((F, N), np.uint8)
    llr = np.empty((F, N), np.float32)
    y_bits = np.empty((F, N), np.uint8) if isinstance(cfg.channel, C.Bsc) else None

    def one(i):
        xi, yi = C.frame(cfg.channel, cfg.seed, j0 + i, N)
        x[i] = xi
        llr[i] = C.channel_llr(cfg.channel, yi)
        if y_bits is not None:
            y_bits[i] = yi

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        list(ex.map(one, range(F)))
    return x, llr, y_bits


class ClockSampler:
    """nvidia-smi's clocks line, via NVML, sampled during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        rs = [name for bit, name in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max, "reasons": rs,
                "samples": len(self.samples)}


def oracle_precision(fmode):
    """The CPU decoder timed beside an f mode: the Q8.8 fixed-point port for
    --fmode fixed (the paper's Table-1 technique), else the
    f64 exact SC port."""
    return (16, "Q8.8 fixed-point SC (table boxplus)") if fmode == "fixed" else (64, "f64 exact SC")


def cpu_baseline(code, llr, u, sample_s, threads=1, precision=64):
    """The oracle port (SPEC restatement) on host cores: decode frames until
    ~sample_s of CPU work; Mbit/s of block bits."""
    from oracle import oracle as O

    N = code.block_size
    F = llr.shape[0]
    done, t0 = 0, time.perf_counter()
    while True:
        k = min(threads, F - (done % F))
        idx = [(done + i) % F for i in range(k)]
        O.sc_decode_batch(code.frozen_mask, llr[idx], u[idx], precision=precision, threads=threads)
        done += k
        el = time.perf_counter() - t0
        if el >= sample_s or done >= 64 * F:
            break
    return done * N / el / 1e6, done, el


def roofline_entry(code, frames, log2S, t_kernel_s, peaks, band_share=None, fmode="fast"):
    """Dominant kernel: sc_decode_kernel.  Algorithmic bytes per launch =
    SURVEY.md 8(d)'s 12.3125 N bytes per HBM-streamed level per frame x the
    levels this launch streams through the per-frame scratch (n - log2 S).
    (int16 stage storage for the fixed-point mode halves those bytes but
    measured slower: the per-frame streams are latency-bound, not byte-bound.)
    `achieved` divides them by the whole kernel time; `upper_band` divides
    them by the kernel time spent in the upper band (its share of the per-frame
    cycle profile, frames run concurrently), which is what the north star's
    ">= 50% of the binding roofline on the upper stages" refers to."""
    n = code.n
    L_up = max(0, n - log2S)
    eb = 4  # stage LLRs are fp32 in every f mode (Q8.8 codes are exact in fp32)
    alg = (3 * eb + 0.3125) * L_up * code.block_size * frames
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = alg / t_kernel_s / 1e9 if t_kernel_s > 0 else 0.0
    out = {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
           "frac": round(achieved / peak, 4), "traffic": None,
           "kernel": "sc_decode_kernel", "alg_bytes_per_launch": alg, "upper_levels": L_up, "stage_bytes_per_llr": eb,
           "peak_source": "MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback B200_PROFILING.md"}
    if band_share and band_share.get("upper", 0) > 0 and L_up > 0:
        t_up = band_share["upper"] * t_kernel_s
        up = alg / t_up / 1e9
        out["upper_band"] = {"time_share": round(band_share["upper"], 4), "achieved": round(up, 2),
                             "frac": round(up / peak, 4)}
        if up > peak:
            out["upper_band"]["note"] = (
                "algorithmic bytes above the HBM peak: part of the stage traffic is served from L2 "
                "(see traffic = ncu dram bytes per launch); the band is bound per CTA by its chunk work "
                "(tools/upper_only.py, DESIGN.md section 7), not by HBM")
        out["band_share"] = {k: round(v, 4) for k, v in band_share.items()}
    return out


def with_traffic(roof, args):
    """dram read+write bytes per launch from the committed ncu --set full capture
    of the same config/f mode (profiles/r01/ncu_full_<cfg>_<fmode>.json), if present."""
    path = os.path.join(ROOT, "profiles", "r01", f"ncu_full_{args.config}_{args.fmode}.json")
    try:
        with open(path) as fh:
            cap = json.load(fh)
        if cap.get("fmode") == args.fmode and not args.no_ssc:
            roof["traffic"] = cap["traffic_bytes_per_launch"]
            roof["traffic_source"] = os.path.relpath(path, ROOT)
    except Exception:
        pass
    return roof


def run_reference(args, rank, world):
    """--impl reference: the reference's decode path has no implementation
    (polar_core is SPEC-only), so the CPU oracle port -- the SPEC restatement --
    is timed on all host threads, one frame per thread per step."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_1204_5882_b200 import codes as K

    cfg = K.CONFIGS[args.config]
    code = K.load_config(args.config)
    N = code.block_size
    threads = max(1, len(os.sched_getaffinity(0)))
    F = threads
    x, llr, _ = gen_frames(cfg, N, 0, F)
    u = np.array([O.polar_transform_bytes(xi) for xi in x])
    prec, what = oracle_precision(args.fmode)
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.sc_decode_batch(code.frozen_mask, llr, u, precision=prec, threads=threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    tot = sum(times)
    v = F * N * len(times) / tot / 1e6
    line = {"metric": "SC-decoded Mbit/s", "value": round(v, 3), "unit": "Mbit/s", "n_gpus": args.gpus,
            "host_only": True,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(times), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "q8.8 (int16)" if prec == 16 else "f64",
            "data": "synthetic (reference channel model, seeded)", "impl": "reference",
            "config": {"workload": cfg.desc, "key": args.config, "frames_per_gpu": cfg.frames_per_gpu, "N": N,
                       "rate": cfg.rate, "f": args.fmode, "frames_per_step": F,
                       "parallelism": f"{threads} host threads on rank 0 (the reference's decoder is CPU-only)"},
            "cpu_baseline": {"value": round(v, 3), "unit": "Mbit/s", "cores": threads, "kind": "port",
                             "sample": f"{F} frames of {args.config} per step (one per thread), {what}"},
            "e2e": {"value": round(v, 3), "unit": "Mbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_1204_5882_b200 import codes as K
    from paper_1204_5882_b200.channel import Bsc
    from paper_1204_5882_b200.polar_core import ScDecoder, pack_bits, polar_transform_words

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = K.CONFIGS[args.config]
    code = K.load_config(args.config)
    N, n = code.block_size, code.n
    F = args.frames or cfg.frames_per_gpu
    is_bsc = isinstance(cfg.channel, Bsc)

    from paper_1204_5882_b200 import dist as D
    idx = D.shard(F, rank)  # weak scaling: rank r owns frames [rF, (r+1)F)
    x, llr, y_bits = gen_frames(cfg, N, idx.start, F)
    x_w = torch.from_numpy(pack_bits(x).view(np.int32).copy()).to(dev)
    u_w = polar_transform_words(x_w, n)  # Alice: u = T(x); the decoder reads u at frozen positions
    llr_d = torch.from_numpy(llr).to(dev)
    dec = ScDecoder(code, max_frames=F, f_mode=args.fmode, ssc=not args.no_ssc, subtree_log2=args.subtree_log2)
    from paper_1204_5882_b200 import _lib
    if args.threads:
        dec.set_option(_lib.PQ_OPT_THREADS, args.threads)
    if args.cluster:
        dec.set_option(_lib.PQ_OPT_CLUSTER, args.cluster)
    if args.warp_log2:
        dec.set_option(_lib.PQ_OPT_WARP_LOG2, args.warp_log2)
    uh = dec.alloc_words(F)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)  # 256 MiB > L2
    stream = torch.cuda.current_stream()

    def step():
        dec.decode(llr_d, u_w, u_hat=uh, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    errors = int((uh != u_w).any(dim=1).sum().item())
    launches = dec.last_launches
    launch_cfg = dec.last_config
    log2S = launch_cfg["subtree_log2"]

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    t_wall = time.perf_counter()
    with sampler:
        for i in range(args.steps):
            flush.fill_(i)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    t_dev = sum(a.elapsed_time(b) for a, b in ev) / 1e3
    t_max = torch.tensor([t_dev], device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_max = float(t_max.item())
    ms_step = 1e3 * t_max / args.steps
    value = world * F * N * args.steps / t_max / 1e6

    # kernel-only time of the dominant kernel on the same stream
    kt = []
    for i in range(min(args.steps, 5)):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dec.decode(llr_d, None, u_hat=None, want_u=False, stream=stream)
        b.record(stream)
        kt.append((a, b))
    torch.cuda.synchronize()
    t_kernel = statistics.median(a.elapsed_time(b) for a, b in kt) / 1e3

    # per-band split of the kernel (one extra, untimed decode with the cycle profile)
    from paper_1204_5882_b200 import _lib
    dec.set_option(_lib.PQ_OPT_PROFILE, 1)
    dec.decode(llr_d, u_w, u_hat=uh, stream=stream)
    torch.cuda.synchronize()
    prof = dec.read_profile(F).astype(np.float64)
    dec.set_option(_lib.PQ_OPT_PROFILE, 0)
    band_share = {
        "upper": float((prof[:, 0] + prof[:, 1] + prof[:, 2]).sum() / prof[:, 9].sum()),
        "shared": float((prof[:, 3] + prof[:, 4] + prof[:, 5] + prof[:, 7] + prof[:, 8]).sum() / prof[:, 9].sum()),
        "warp": float(prof[:, 6].sum() / prof[:, 9].sum()),
    }

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        q88 = not is_bsc and args.fmode == "fixed"
        if is_bsc:
            h_in = torch.from_numpy(pack_bits(y_bits).view(np.int32).copy()).pin_memory()
        elif q88:  # the fixed-point decoder's own input format: Q8.8 int16 codes
            h_in = torch.from_numpy(np.clip(np.rint(llr * np.float32(256.0)), -32767, 32767)
                                    .astype(np.int16)).pin_memory()
        else:
            h_in = torch.from_numpy(llr).pin_memory()
        h_fz = u_w.cpu().pin_memory()
        h_out = [torch.empty((F, dec.wpf), dtype=torch.int32).pin_memory() for _ in range(2)]
        mag = cfg.channel.llr_magnitude if is_bsc else None
        # the public streaming API: batch k's H2D, k-1's decode and k-2's D2H overlap
        from paper_1204_5882_b200.pipeline import PipelinedDecoder
        pipe = PipelinedDecoder(dec, F, bsc_llr_mag=mag, q88=q88)

        for q in range(2):
            pipe.submit(h_in, h_fz, h_out[q & 1])
        pipe.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(pipe.s_h2d)
        for q in range(args.steps):
            pipe.submit(h_in, h_fz, h_out[q & 1])
        b.record(pipe.last_stream)
        pipe.synchronize()
        torch.cuda.synchronize()
        te = torch.tensor([a.elapsed_time(b) / 1e3], device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        te = float(te.item())
        hb = h_in.numel() * h_in.element_size() + h_fz.numel() * 4
        e2e = {"value": round(world * F * N * args.steps / te / 1e6, 2), "unit": "Mbit/s",
               "h2d_bytes_per_step": int(hb), "d2h_bytes_per_step": int(h_out[0].numel() * 4),
               "input": ("received bits, fused BSC front end" if is_bsc else
                         "Q8.8 int16 LLR codes (sc_decode_fixed input)" if q88 else "fp32 LLRs"),
               "pipeline": "PipelinedDecoder: H2D / decode / D2H on 3 streams, 2 buffer sets"}
        last = h_out[(args.steps - 1) & 1].to(dev)
        err2 = int((last != u_w).any(dim=1).sum().item())
        assert err2 == errors, "e2e path decoded differently from the device path"

    # statistics off the hot path (NCCL all-reduce of frame errors), and the
    # decoded bits gathered over NVLink; both untimed
    stats = D.reduce_stats(torch.tensor([errors, F], dtype=torch.int64, device=dev))
    gather = None
    if world > 1:
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        allu = D.gather_words(uh)
        g1.record()
        torch.cuda.synchronize()
        assert allu.shape[0] == world * F
        gather = {"collective": "all_gather (NCCL)", "bytes_per_rank": int(uh.numel() * 4),
                  "ms": round(g0.elapsed_time(g1), 3)}

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
                peaks = json.load(fh)
        except Exception:
            pass
        cpu = None
        if not args.no_cpu_baseline:
            from oracle import oracle as O
            u_np = np.array([O.polar_transform_bytes(xi) for xi in x[:8]])
            prec, what = oracle_precision(args.fmode)
            v, nfr, el = cpu_baseline(code, llr[:8], u_np, args.cpu_sample_s, threads=1, precision=prec)
            cpu = {"value": round(v, 3), "unit": "Mbit/s", "cores": 1, "kind": "port",
                   "sample": f"{nfr} frames of {args.config} (N=2^{n}) in {el:.1f} s, {what}, 1 thread"}
        line = {
            "metric": "SC-decoded Mbit/s", "value": round(value, 2), "unit": "Mbit/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": round(value / PAPER_MBPS[args.config], 1) if args.config in PAPER_MBPS else None,
            "dtype": {"exact": "f32", "fast": "f32 (SFU transcendentals)", "fixed": "q8.8 (saturating int16 semantics)", "min-sum": "f32-minsum"}[args.fmode],
            "data": "synthetic: reference channel model, seeded (SURVEY 8(d)); reference-constructed frozen set",
            "config": {"workload": cfg.desc, "key": args.config, "frames_per_gpu": F, "N": N,
                       "rate": cfg.rate, "f": args.fmode, "ssc": not args.no_ssc, "subtree_log2": log2S, "threads_per_cta": launch_cfg["threads_per_cta"],
                       "ctas_per_frame": launch_cfg["ctas_per_frame"],
                       "parallelism": f"frames sharded over {world} GPU(s)", "l2": "256 MiB flush between steps"},
            "fer": round(int(stats[0]) / int(stats[1]), 4), "frames_total": int(stats[1]),
            "e2e": e2e, "gpu_launches": launches * args.steps, "gather_u_hat": gather,
            "roofline": with_traffic(roofline_entry(code, F, log2S, t_kernel, peaks, band_share, args.fmode), args),
            "kernel_ms": round(1e3 * t_kernel, 3),
            "cpu_baseline": cpu, "clocks": sampler.summary(), "wall_s_timed": round(t_wall, 3),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
