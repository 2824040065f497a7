"""N > 1 host path on CPU: world_size-2 gloo ranks run the frame sharding and the final
statistics reduction of paper_1008_0502_b200/shard.py (the only collective of the path,
SURVEY.md §8(e)); the result must equal the single-process statistics of the whole batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1008_0502_b200 import shard

N_PER_RANK = 5
H, W = 6, 7


def fake_results(t0, n):
    """Deterministic per-frame (F, mask) as a solved shard would return them (frame 3 failed)."""
    rng = np.random.default_rng(1234)
    F = rng.integers(0, 10**9, size=64)
    M = rng.integers(0, 2, size=(64, H, W)).astype(np.uint8)
    F[3] = -1
    M[3] = 0
    return torch.from_numpy(F[t0:t0 + n].copy()), torch.from_numpy(M[t0:t0 + n].copy())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t0, n = shard.frame_range(rank, world, N_PER_RANK)
        flow, mask = fake_results(t0, n)
        stats, per = shard.frame_stats(flow, mask)
        stats, per = shard.reduce_stats(stats, per, world)
        ms = shard.max_over_ranks(10.0 + rank, torch.device("cpu"), world)
        if rank == 0:
            out.put((stats.tolist(), per.tolist(), ms))
    finally:
        dist.destroy_process_group()


def test_frame_range():
    assert shard.frame_range(0, 2, 5) == (0, 5)
    assert shard.frame_range(1, 2, 5) == (5, 5)
    with pytest.raises(ValueError):
        shard.frame_range(2, 2, 5)


def test_two_rank_gloo_reduction():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    stats, per, ms = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    flow, mask = fake_results(0, world * N_PER_RANK)
    ref_stats, ref_per = shard.frame_stats(flow, mask)
    assert stats == ref_stats.tolist()
    assert per == ref_per.tolist()
    assert stats[2] == 1  # the failed frame (F = -1) is counted, not summed
    assert ms == 11.0     # timing = max over ranks
