"""SC-decode throughput bench (BASELINE.json metric: SC-decoded Mbit/s).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

A step = one batched decode of this rank's frames of the config (c3 by
default: BSC p=0.02, N=2^20, rate 0.83, 256 frames per GPU, the reference's
own frozen set).  Mbit/s = frames * N / seconds / 1e6 (block bits).

  value    device-resident LLRs (+ revealed frozen words) in HBM, u-hat
           written to HBM, CUDA events on the launching stream, L2 flushed
           (256 MiB write) between timed steps, max over ranks.
  e2e      the public streaming API with host buffers: each step copies Bob's
           inputs from pinned host memory (BSC: received bits packed 1
           bit/symbol, decoded by the fused front end; BIAWGN + fixed point:
           Q8.8 int16 codes) plus the revealed frozen words, decodes, and
           copies u-hat back.
  parity   after the timed region every timed frame's u-hat is compared with
           the CPU oracle (the integer Q8.8 oracle for --fmode fixed, the fp32
           mirror for exact) on all host threads -- the bench checks itself.
  roofline kernel_ms = CUDA events bracketing the sc_decode_kernel launch
           itself inside every timed step (PQ_OPT_TIMING), so kernel_ms <=
           ms_per_step by construction.
The default c3 run adds the N = 2^20 BIAWGN (c4), the N = 2^24 (c5) and the
fp32-exact c3 numbers as `configs` sub-objects (--no-extras skips them).

Multi-GPU: `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks (one per GPU); under torchrun WORLD_SIZE
must equal --gpus.  Frames shard by index (rank r takes frames
[r*F, (r+1)*F)), no collective on the hot path; NCCL all-reduces the frame
error counts and all-gathers u-hat afterwards (scaling: weak).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_MBPS = {"c3": 9.5}  # BASELINE.md / PAPER.md:170: SC decode, BSC 2%, N=2^20, 1 core i5-670
EXTRAS = (("c4", "fixed"), ("c5", "fixed"), ("c3", "exact"))


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
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the c4 / c5 / c3-exact sub-objects")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_respawn(args) -> None:
    """`--gpus N` outside torchrun: run this script under torch.distributed.run
    with N ranks and exit with its status.  Inside torchrun: WORLD_SIZE must
    equal --gpus (fail loudly otherwise)."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch one rank per GPU)")
        return
    if args.gpus <= 1:
        return
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} requested, {have} CUDA device(s) visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    print(f"[bench] spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    sys.exit(subprocess.call(cmd))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


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
    """The CPU decoder beside an f mode: the Q8.8 fixed-point port for --fmode
    fixed (the paper's Table-1 technique), the fp32 mirror
    for exact (bit-exact reference of the GPU's IEEE-only f), else f64."""
    return {"fixed": (16, "Q8.8 fixed-point SC (table boxplus), plain recursion: every node visited, "
                          "none of the GPU path's decision-exact sub-tree shortcuts"),
            "exact": (32, "fp32 exact SC (IEEE-only boxplus mirror), plain recursion")}.get(
                fmode, (64, "f64 exact SC, plain recursion"))


def cpu_baseline(code, llr, u, sample_s, threads=1, precision=16):
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


def load_json(*parts):
    try:
        with open(os.path.join(ROOT, *parts)) as fh:
            return json.load(fh)
    except Exception:
        return None


def roofline_entry(code, frames, log2S, t_kernel_s, peaks, key, fmode, ssc=True):
    """Dominant kernel: sc_decode_kernel.  Algorithmic bytes per launch =
    SURVEY.md 8(d)'s 12.3125 N bytes per HBM-streamed level per frame x the
    levels this launch streams through the per-frame scratch (n - log2 S),
    x frames; achieved = that / the kernel's mean launch duration (CUDA events
    around the launch inside the timed steps).  `traffic` = ncu
    dram__bytes_read + write of the same launch from the committed capture;
    `upper_band` = the upper band measured in isolation by ncu
    (tools/upper_only.py: every level above S streams, the sub-trees are
    trivial), from the committed capture."""
    n = code.n
    L_up = max(0, n - log2S)
    alg = 12.3125 * L_up * code.block_size * frames
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = alg / t_kernel_s / 1e9 if t_kernel_s > 0 else 0.0
    out = {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
           "frac": round(achieved / peak, 4), "traffic": None,
           "kernel": "sc_decode_kernel", "alg_bytes_per_launch": alg, "upper_levels": L_up,
           "alg_bytes_per_unit": "12.3125 N per streamed level per frame (SURVEY 8(d))",
           "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback B200_PROFILING.md"}
    for rnd in ("r02", "r01"):
        cap = load_json("profiles", rnd, f"ncu_full_{key}_{fmode}.json")
        if cap and cap.get("fmode") == fmode and ssc:
            out["traffic"] = cap["traffic_bytes_per_launch"]
            out["traffic_source"] = f"profiles/{rnd}/ncu_full_{key}_{fmode}.json"
            break
    up = load_json("profiles", "r02", "ncu_upper_only.json")
    if up and key in ("c3", "c4") and fmode == up.get("fmode"):
        a = up["alg_bytes_per_launch"] / (up["gpu__time_duration_ms"] / 1e3) / 1e9
        out["upper_band"] = {"achieved": round(a, 2), "frac": round(a / peak, 4),
                             "dram_bytes_per_launch": up["traffic_bytes_per_launch"],
                             "source": "profiles/r02/ncu_upper_only.json (ncu, tools/upper_only.py, 256 frames, N=2^20)"}
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's decode path has no implementation
    (polar_core is SPEC-only), so the CPU oracle port -- the SPEC restatement --
    is timed on all host threads, one frame per thread per step."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_1204_5882_b200 import channel as C
    from paper_1204_5882_b200 import codes as K

    cfg = K.CONFIGS[args.config]
    code = K.load_config(args.config)
    N = code.block_size
    threads = host_threads()
    F = threads
    x, llr, _ = C.frames_batch(cfg.channel, cfg.seed, 0, F, N, want_y=False)
    u = np.array([O.polar_transform_bytes(xi) for xi in x])
    # the reference's LlrBlock is Float64 or Q8.8 fixed point
    prec, what = oracle_precision(args.fmode) if args.fmode == "fixed" else (64, "f64 exact SC")
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
            "dtype": {16: "q8.8 (int16)", 32: "f32"}.get(prec, "f64"),
            "data": "synthetic (reference channel model, seeded)", "impl": "reference",
            "config": {"workload": cfg.desc, "key": args.config, "frames_per_gpu": cfg.frames_per_gpu, "N": N,
                       "rate": cfg.rate, "f": args.fmode, "frames_per_step": F,
                       "parallelism": f"{threads} host threads on rank 0 (the reference's decoder is CPU-only)"},
            "cpu_baseline": {"value": round(v, 3), "unit": "Mbit/s", "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(),
                             "sample": f"{F} frames of {args.config} per step (one per thread), {what}"},
            "e2e": {"value": round(v, 3), "unit": "Mbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


class Ctx:
    """Per-rank state shared by the measurements."""

    def __init__(self, args, rank, world, local, dev):
        import torch
        self.args, self.rank, self.world, self.local, self.dev = args, rank, world, local, dev
        self.flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)  # 256 MiB > L2
        self.peaks = load_json("MEASURED_PEAKS.json") or {}


def measure(ctx: Ctx, key: str, fmode: str, frames: int = 0, headline: bool = False) -> dict:
    """Time one config on this rank's frames; rank 0 returns the result dict."""
    import torch
    import torch.distributed as dist

    from paper_1204_5882_b200 import _lib
    from paper_1204_5882_b200 import channel as C
    from paper_1204_5882_b200 import codes as K
    from paper_1204_5882_b200 import dist as D
    from paper_1204_5882_b200.pipeline import PipelinedDecoder
    from paper_1204_5882_b200.polar_core import ScDecoder, pack_bits, polar_transform_words, unpack_bits

    args, rank, world, dev = ctx.args, ctx.rank, ctx.world, ctx.dev
    cfg = K.CONFIGS[key]
    code = K.load_config(key)
    N, n = code.block_size, code.n
    F = frames or cfg.frames_per_gpu
    is_bsc = isinstance(cfg.channel, C.Bsc)
    idx = D.shard(F, rank)  # weak scaling: rank r owns frames [rF, (r+1)F)
    t_gen = time.perf_counter()
    x, llr, y_bits = C.frames_batch(cfg.channel, cfg.seed, idx.start, F, N)
    t_gen = time.perf_counter() - t_gen
    x_w = torch.from_numpy(pack_bits(x).view(np.int32).copy()).to(dev)
    u_w = polar_transform_words(x_w, n)  # Alice: u = T(x); the decoder reads u at frozen positions
    llr_d = torch.from_numpy(llr).to(dev)
    dec = ScDecoder(code, max_frames=F, f_mode=fmode, ssc=not args.no_ssc,
                    subtree_log2=args.subtree_log2 if headline else 0)
    if headline:
        if args.threads:
            dec.set_option(_lib.PQ_OPT_THREADS, args.threads)
        if args.cluster:
            dec.set_option(_lib.PQ_OPT_CLUSTER, args.cluster)
        if args.warp_log2:
            dec.set_option(_lib.PQ_OPT_WARP_LOG2, args.warp_log2)
    uh = dec.alloc_words(F)
    stream = torch.cuda.current_stream(dev)

    def step():
        dec.decode(llr_d, u_w, u_hat=uh, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    errors = int((uh != u_w).any(dim=1).sum().item())
    launches = dec.last_launches
    launch_cfg = dec.last_config
    log2S = launch_cfg["subtree_log2"]

    # ---- timed region: K steps, events on the launching stream, L2 flushed between steps;
    # the decoder brackets its sc_decode_kernel launch with its own events (kernel_ms)
    dec.set_option(_lib.PQ_OPT_TIMING, 1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(ctx.local)
    t_wall = time.perf_counter()
    with sampler:
        for i in range(args.steps):
            ctx.flush.fill_(i)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    t_dev = sum(a.elapsed_time(b) for a, b in ev) / 1e3
    t_max = D.max_over_ranks(t_dev, dev)
    ms_step = 1e3 * t_max / args.steps
    value = world * F * N * args.steps / t_max / 1e6
    kt = dec.kernel_times(min(args.steps, 64)).astype(np.float64)
    dec.set_option(_lib.PQ_OPT_TIMING, 0)
    t_kernel = D.max_over_ranks(float(kt.mean()) / 1e3, dev)

    # per-band split of one extra, untimed decode (diagnostic cycle profile)
    dec.set_option(_lib.PQ_OPT_PROFILE, 1)
    uh_prof = dec.alloc_words(F)
    dec.decode(llr_d, u_w, u_hat=uh_prof, stream=stream)
    torch.cuda.synchronize()
    prof = dec.read_profile(F).astype(np.float64)
    dec.set_option(_lib.PQ_OPT_PROFILE, 0)
    tot = prof[:, 9].sum()
    band_share = {"upper": float((prof[:, 0] + prof[:, 1] + prof[:, 2]).sum() / tot),
                  "shared": float((prof[:, 3] + prof[:, 4] + prof[:, 5] + prof[:, 7] + prof[:, 8]).sum() / tot),
                  "warp": float(prof[:, 6].sum() / tot)}
    assert torch.equal(uh_prof, uh), "profiling instantiation decoded differently"
    del uh_prof

    # ---- end to end through the public streaming API with host buffers
    e2e = None
    if not args.no_e2e:
        q88 = not is_bsc and fmode == "fixed"
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
        del llr_d
        torch.cuda.empty_cache()
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
        te = D.max_over_ranks(a.elapsed_time(b) / 1e3, dev)
        hb = h_in.numel() * h_in.element_size() + h_fz.numel() * 4
        e2e = {"value": round(world * F * N * args.steps / te / 1e6, 2), "unit": "Mbit/s",
               "h2d_bytes_per_step": int(hb), "d2h_bytes_per_step": int(h_out[0].numel() * 4),
               "input": ("received bits, fused BSC front end" if is_bsc else
                         "Q8.8 int16 LLR codes (sc_decode_fixed input)" if q88 else "fp32 LLRs"),
               "pipeline": "PipelinedDecoder: H2D / decode / D2H on 3 streams, 2 buffer sets"}
        last = h_out[(args.steps - 1) & 1].to(dev)
        assert torch.equal(last, uh), "e2e path decoded differently from the device path"
        del pipe, h_in, h_out

    # ---- statistics and the decoded bits gathered over NVLink (off the hot path, untimed)
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
        del allu

    out = None
    if rank == 0:
        parity = None
        if not args.no_parity:
            from oracle import oracle as O
            prec, what = oracle_precision(fmode)
            got = unpack_bits(uh.cpu().numpy().view(np.uint32), N)
            u = unpack_bits(u_w.cpu().numpy().view(np.uint32), N)
            t0 = time.perf_counter()
            if prec == 64:  # SFU f: the north star's tolerance rule against f64
                ref, mi = O.sc_decode_batch(code.frozen_mask, llr, u, precision=64, threads=host_threads(),
                                            min_info=True)
                clean = mi >= 1e-4
                bad = int(np.sum(np.any(got[clean] != ref[clean], axis=1)))
            else:
                ref = O.sc_decode_batch(code.frozen_mask, llr, u, precision=prec, threads=host_threads())
                bad = int(np.sum(np.any(got != ref, axis=1)))
            parity = {"frames": F, "mismatches": bad, "oracle": what,
                      "fer_oracle": round(float(np.mean(np.any(ref != u, axis=1))), 4),
                      "fer_gpu": round(float(np.mean(np.any(got != u, axis=1))), 4),
                      "oracle_s": round(time.perf_counter() - t0, 1), "threads": host_threads(),
                      "scope": "every timed frame of rank 0"}
        out = {
            "value": round(value, 2), "ms_per_step": round(ms_step, 3), "kernel_ms": round(1e3 * t_kernel, 3),
            "fer": round(int(stats[0]) / int(stats[1]), 4), "frames_total": int(stats[1]),
            "e2e": e2e, "parity": parity, "gpu_launches": launches * args.steps, "gather_u_hat": gather,
            "roofline": roofline_entry(code, F, log2S, t_kernel, ctx.peaks, key, fmode, not args.no_ssc),
            "band_share": {k: round(v, 4) for k, v in band_share.items()},
            "config": {"workload": cfg.desc, "key": key, "frames_per_gpu": F, "N": N, "rate": cfg.rate,
                       "f": fmode, "ssc": not args.no_ssc, "subtree_log2": log2S,
                       "threads_per_cta": launch_cfg["threads_per_cta"],
                       "ctas_per_frame": launch_cfg["ctas_per_frame"],
                       "parallelism": f"frames sharded over {world} GPU(s)", "l2": "256 MiB flush between steps"},
            "clocks": sampler.summary(), "wall_s_timed": round(t_wall, 3), "host_gen_s": round(t_gen, 2),
        }
        if headline and not args.no_cpu_baseline:
            from oracle import oracle as O
            u_np = np.array([O.polar_transform_bytes(xi) for xi in x[:8]])
            prec, what = oracle_precision(fmode)
            v, nfr, el = cpu_baseline(code, llr[:8], u_np, args.cpu_sample_s, threads=1, precision=prec)
            out["cpu_baseline"] = {"value": round(v, 3), "unit": "Mbit/s", "cores": 1, "kind": "port",
                                   "cpu_model": cpu_model(),
                                   "sample": f"{nfr} frames of {key} (N=2^{n}) in {el:.1f} s, {what}, 1 thread"}
    del dec, uh, u_w, x_w
    torch.cuda.empty_cache()
    return out


DTYPES = {"exact": "f32", "fast": "f32 (SFU transcendentals)", "fixed": "q8.8 (saturating int16 semantics)",
          "min-sum": "f32-minsum"}


def main():
    args = parse()
    maybe_respawn(args)
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        probe = torch.ones(1, device=dev)
        dist.all_reduce(probe)  # the NCCL communicator is up on every rank
        print(f"[bench] rank {rank}/{world}: NCCL communicator initialised on cuda:{local} "
              f"({torch.cuda.get_device_name(dev)}), all_reduce probe = {int(probe.item())}",
              file=sys.stderr, flush=True)
    ctx = Ctx(args, rank, world, local, dev)
    head = measure(ctx, args.config, args.fmode, args.frames, headline=True)
    extras = {}
    if not args.no_extras and args.config == "c3" and not args.frames:
        for key, fm in EXTRAS:
            if key == args.config and fm == args.fmode:
                continue
            sub = measure(ctx, key, fm)
            if rank == 0:
                extras[f"{key}_{fm}"] = sub

    if rank == 0:
        line = {
            "metric": "SC-decoded Mbit/s", "value": head["value"], "unit": "Mbit/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": round(head["value"] / PAPER_MBPS[args.config], 1) if args.config in PAPER_MBPS else None,
            "dtype": DTYPES[args.fmode],
            "data": "synthetic: reference channel model, seeded (SURVEY 8(d)); reference-constructed frozen set",
        }
        line.update({k: v for k, v in head.items() if k not in ("value", "ms_per_step")})
        if extras:
            line["configs"] = {k: {kk: v[kk] for kk in ("value", "ms_per_step", "kernel_ms", "fer", "e2e", "parity",
                                                          "gpu_launches", "config", "clocks")}
                               | {"roofline": {kk: v["roofline"].get(kk) for kk in
                                               ("achieved", "frac", "peak", "traffic", "alg_bytes_per_launch",
                                                "upper_levels")},
                                  "dtype": DTYPES[k.split("_", 1)[1]]}
                               for k, v in extras.items()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
