"""Multi-GPU plumbing for the decode path.

Frames are independent ("embarrassingly parallel"), so the hot
path has no collective: rank r decodes the frames [r*F, (r+1)*F) of the global
seed sequence (weak scaling).  The only exchanges happen after decoding:
``reduce_stats`` sums frame/bit error counters and ``gather_words`` collects
packed u-hat words on every rank (NCCL over NVLink on the GPU box; gloo in the
CPU tests).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard(frames_per_rank: int, rank: int) -> range:
    """Global frame indices decoded by `rank` (weak scaling)."""
    return range(rank * frames_per_rank, (rank + 1) * frames_per_rank)


def shard_total(total_frames: int, rank: int, world: int) -> range:
    """Strong-scaling split of a fixed total: contiguous, sizes differ by <= 1."""
    base, extra = divmod(total_frames, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def reduce_stats(counters: torch.Tensor, group=None) -> torch.Tensor:
    """Sum int64 counters (e.g. [frame_errors, frames, bit_errors]) over ranks."""
    out = counters.clone()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def max_over_ranks(value: float, device) -> float:
    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_words(words: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather equal-shaped [F, W] word tensors -> [world*F, W] in rank order."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return words
    parts = [torch.empty_like(words) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, words.contiguous(), group=group)
    return torch.cat(parts, dim=0)
