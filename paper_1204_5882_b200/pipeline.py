"""Streaming decode of host batches with the PCIe copies overlapped.

A reconciliation service decodes a continuous stream of blocks whose inputs
arrive in host memory (Bob's received bits or LLRs, Alice's revealed frozen
values).  ``PipelinedDecoder`` keeps two device buffer sets
and three CUDA streams so that, in steady state, batch k's host-to-device
copy, batch k-1's decode and batch k-2's device-to-host copy of u-hat run
concurrently: the throughput is max(copies, decode) instead of their sum.
Every batch still makes the full round trip (pinned host in -> device ->
pinned host out); nothing is cached between batches.
"""
from __future__ import annotations

import torch

from .polar_core import ScDecoder


class PipelinedDecoder:
    """Double-buffered host-batch decoding on one device.

    dec: an ScDecoder sized for ``frames`` frames.  ``bsc_llr_mag`` given ->
    inputs are packed received bits ([F, N/32] int32, fused BSC front end);
    ``q88`` -> Q8.8 int16 LLR codes ([F, N], fixed-point decoders); otherwise
    fp32 LLRs ([F, N]).  ``submit`` enqueues one batch and returns
    immediately; ``synchronize`` waits for everything submitted.  Host tensors
    must be pinned and must not be modified until the batch has completed.
    """

    def __init__(self, dec: ScDecoder, frames: int, bsc_llr_mag: float | None = None, q88: bool = False):
        self.dec, self.F = dec, int(frames)
        self.mag, self.q88 = bsc_llr_mag, q88
        dev = dec.device
        N, wpf = dec.N, dec.wpf
        if q88:  # Q8.8 int16 codes (SPEC.md:250's fixed-point input; fixed-point decoders)
            self.d_in = [torch.empty((frames, N), dtype=torch.int16, device=dev) for _ in range(2)]
        elif bsc_llr_mag is None:
            self.d_in = [torch.empty((frames, N), dtype=torch.float32, device=dev) for _ in range(2)]
        else:
            self.d_in = [torch.empty((frames, wpf), dtype=torch.int32, device=dev) for _ in range(2)]
        self.d_fz = [torch.empty((frames, wpf), dtype=torch.int32, device=dev) for _ in range(2)]
        self.d_u = [torch.empty((frames, wpf), dtype=torch.int32, device=dev) for _ in range(2)]
        self.s_h2d = torch.cuda.Stream(dev)
        self.s_dec = torch.cuda.Stream(dev)
        self.s_d2h = torch.cuda.Stream(dev)
        self.ev_in = [torch.cuda.Event() for _ in range(2)]     # inputs landed
        self.ev_dec = [torch.cuda.Event() for _ in range(2)]    # decode done (inputs free, u-hat ready)
        self.ev_out = [torch.cuda.Event() for _ in range(2)]    # u-hat copied out (buffer free)
        self.k = 0

    def submit(self, h_in: torch.Tensor, h_fz: torch.Tensor, h_out: torch.Tensor) -> None:
        i = self.k & 1
        if self.k >= 2:
            self.s_h2d.wait_event(self.ev_dec[i])   # decode k-2 has read d_in[i]
        with torch.cuda.stream(self.s_h2d):
            self.d_in[i].copy_(h_in, non_blocking=True)
            self.d_fz[i].copy_(h_fz, non_blocking=True)
            self.ev_in[i].record(self.s_h2d)
        self.s_dec.wait_event(self.ev_in[i])
        if self.k >= 2:
            self.s_dec.wait_event(self.ev_out[i])   # u-hat of k-2 is out of d_u[i]
        if self.q88:
            self.dec.decode_q88(self.d_in[i], self.d_fz[i], u_hat=self.d_u[i], stream=self.s_dec)
        elif self.mag is None:
            self.dec.decode(self.d_in[i], self.d_fz[i], u_hat=self.d_u[i], stream=self.s_dec)
        else:
            self.dec.decode_bsc(self.d_in[i], self.mag, self.d_fz[i], u_hat=self.d_u[i], stream=self.s_dec)
        self.ev_dec[i].record(self.s_dec)
        self.s_d2h.wait_event(self.ev_dec[i])
        with torch.cuda.stream(self.s_d2h):
            h_out.copy_(self.d_u[i], non_blocking=True)
            self.ev_out[i].record(self.s_d2h)
        self.k += 1

    @property
    def last_stream(self) -> torch.cuda.Stream:
        """The stream the last submitted batch finishes on (its u-hat D2H)."""
        return self.s_d2h

    def synchronize(self) -> None:
        for s in (self.s_h2d, self.s_dec, self.s_d2h):
            s.synchronize()
