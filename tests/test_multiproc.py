"""World-size-2 gloo tests of the multi-GPU plumbing (CPU; the decode itself is
the oracle here, standing in for each rank's GPU decode)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1204_5882_b200 import channel as C
from paper_1204_5882_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frames(cfg_seed, idx, N, ch):
    xs, ls = [], []
    for j in idx:
        x, y = C.frame(ch, cfg_seed, j, N)
        xs.append(x)
        ls.append(C.channel_llr(ch, y).astype(np.float32))
    return np.array(xs), np.array(ls)


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_1204_5882_b200.polar_core import pack_bits
        N, F, ch, seed = 256, 3, C.Bsc(0.06), 77
        mask = (np.random.default_rng(5).random(N) < 0.5).astype(np.uint8)
        idx = D.shard(F, rank)
        x, llr = _frames(seed, idx, N, ch)
        u = np.array([O.polar_transform_bytes(xi) for xi in x])
        uh = O.sc_decode_batch(mask, llr, u, precision=32)
        err = int(np.any(uh != u, axis=1).sum())
        stats = D.reduce_stats(torch.tensor([err, F], dtype=torch.int64))
        words = torch.from_numpy(pack_bits(uh).view(np.int32).copy())
        allw = D.gather_words(words)
        tmax = D.max_over_ranks(float(rank + 1), "cpu")
        if rank == 0:
            result_q.put((stats.tolist(), allw.numpy(), tmax))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_shard_reduce_gather():
    from oracle import oracle as O
    from paper_1204_5882_b200.polar_core import pack_bits
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    stats, allw, tmax = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    # single-process reference over the union of the shards
    N, F, ch, seed = 256, 3, C.Bsc(0.06), 77
    mask = (np.random.default_rng(5).random(N) < 0.5).astype(np.uint8)
    x, llr = _frames(seed, range(2 * F), N, ch)
    u = np.array([O.polar_transform_bytes(xi) for xi in x])
    uh = O.sc_decode_batch(mask, llr, u, precision=32)
    assert stats == [int(np.any(uh != u, axis=1).sum()), 2 * F]
    assert np.array_equal(allw, pack_bits(uh).view(np.int32))
    assert tmax == 2.0


def test_shard_ranges():
    assert list(D.shard(4, 0)) == [0, 1, 2, 3] and list(D.shard(4, 3)) == [12, 13, 14, 15]
    parts = [D.shard_total(10, r, 4) for r in range(4)]
    assert [len(p) for p in parts] == [3, 3, 2, 2]
    assert sum((list(p) for p in parts), []) == list(range(10))
