"""Monte-Carlo FER / throughput trials -- SPEC.md's ``bench.run_trials``
(SPEC.md:374-390, :417-420), on the GPU decoder.

run_trials(code, ch, trials, seed, representation) -> BenchRow
  for each trial: draw random x, transmit, disclose (u = T(x) at the frozen
  positions), decode, verify; fer_measured = discarded / trials; throughput =
  trials * N / decode time (block bits), decode time only
  (construction and channel sampling excluded, one warm-up decode discarded,
  SPEC.md:419).  Trial t uses make_rng(seed, 2t) for x and stream 2t+1 for the
  channel noise (the same frames whatever the batch size).

BSC frames are drawn on the device (the reference's numpy sequence, bit for
bit: csrc/frames.cu); BIAWGN frames on host threads, one batch ahead of the
decode.  Frames are decoded in batches on one GPU; verification compares x_hat with
x on the device (equivalent to SPEC.md:318's hash check without the 2^-64
collision term).  CSV output (``emit_csv``) follows SPEC.md:402-410.
"""
from __future__ import annotations

import csv
import io
import time
from dataclasses import asdict, dataclass

import numpy as np

from . import channel as C
from .codes import PolarCode, code_table_checksum
from .polar_core import ScDecoder, pack_bits, polar_transform_words

REPRESENTATIONS = {"float": "exact", "fast": "fast", "fixed": "fixed"}


@dataclass
class BenchRow:
    channel: str
    n: int
    rate: float
    fer_measured: float
    trials: int
    throughput_mbps: float
    wall_time: float
    seed: int
    representation: str
    code_checksum: int | None = None


def _channel_name(ch) -> str:
    return f"bsc({ch.p})" if isinstance(ch, C.Bsc) else f"biawgn({ch.snr})"


def run_trials(code: PolarCode, ch, trials: int, seed: int, representation: str = "fixed",
               batch: int = 256, device=None, code_path=None) -> BenchRow:
    """SPEC.md:382-390 on the GPU.  ``representation``: "fixed" (Q8.8, the
    reference's default decode path), "float" (exact fp32) or
    "fast" (fp32, SFU transcendentals)."""
    import torch

    if trials < 1:
        raise ValueError("trials must be >= 1")
    if representation not in REPRESENTATIONS:
        raise ValueError(f"representation must be one of {sorted(REPRESENTATIONS)}")
    if type(ch) is not type(code.channel):
        raise ValueError("channel family must match the code's design channel")
    N, n = code.block_size, code.n
    batch = max(1, min(batch, trials))
    dec = ScDecoder(code, max_frames=batch, f_mode=REPRESENTATIONS[representation], device=device)
    dev = dec.device
    is_bsc = isinstance(ch, C.Bsc)
    mag = np.float32(ch.llr_magnitude) if is_bsc else None
    failures, decode_s = 0, 0.0
    t_wall = time.perf_counter()
    warm = True
    done = 0
    from concurrent.futures import ThreadPoolExecutor

    def host_batch(j0, F):
        # BIAWGN: threaded host generation of the next batch (channel.frames_batch),
        # overlapped with the device decode of the current one
        x, llr, _ = C.frames_batch(ch, seed, j0, F, N, want_y=False)
        return x, llr

    gen = None if is_bsc else ThreadPoolExecutor(max_workers=1)
    nxt = None if is_bsc else gen.submit(host_batch, 0, min(batch, trials))
    while done < trials:
        F = min(batch, trials - done)
        if is_bsc:
            # BSC: the same numpy-seeded frames drawn on the device (csrc/frames.cu)
            x_w, d_in = C.bsc_frames_device(ch, seed, done, F, n, device=dev)
        else:
            x, inp = nxt.result()
            if done + F < trials:
                nxt = gen.submit(host_batch, done + F, min(batch, trials - done - F))
            x_w = torch.from_numpy(pack_bits(x).view(np.int32).copy()).to(dev)
            d_in = torch.from_numpy(inp).to(dev)
        u_w = polar_transform_words(x_w, n)  # Alice's disclosure: u = T(x)

        def decode():
            if is_bsc:
                return dec.decode_bsc(d_in, mag, u_w, want_u=False, want_x=True, frames=F)[1]
            return dec.decode(d_in, u_w, want_u=False, want_x=True)[1]

        if warm:  # one discarded warm-up decode
            decode()
            warm = False
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        x_hat = decode()
        b.record()
        torch.cuda.synchronize(dev)
        decode_s += a.elapsed_time(b) / 1e3
        failures += int((x_hat[:F] != x_w).any(dim=1).sum().item())
        done += F
    if gen is not None:
        gen.shutdown()
    wall = time.perf_counter() - t_wall
    return BenchRow(channel=_channel_name(ch), n=n, rate=code.rate, fer_measured=failures / trials,
                    trials=trials, throughput_mbps=trials * N / decode_s / 1e6, wall_time=wall, seed=seed,
                    representation=representation,
                    code_checksum=code_table_checksum(code_path) if code_path else None)


def emit_csv(rows, path=None) -> str:
    """One header line then one row per entry, RFC-4180 quoting, fields in
    BenchRow order; byte-identical for identical rows."""
    rows = list(rows)
    if not rows:
        raise ValueError("empty report")
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    fields = list(asdict(rows[0]).keys())
    w.writerow(fields)
    for r in rows:
        d = asdict(r)
        w.writerow([d[f] for f in fields])
    text = buf.getvalue()
    if path is not None:
        with open(path, "w", newline="") as fh:
            fh.write(text)
    return text
