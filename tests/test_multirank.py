"""N > 1 host path on CPU: world_size-2 gloo ranks run the frame sharding, the final
statistics reduction and the cross-rank check of paper_1008_0502_b200/shard.py (the only
collectives of the path); the result must equal the single-process
statistics of the whole batch.  The ranks are started both by torch.multiprocessing and by
shard.launch_local_ranks (the self-launch path of `python bench.py --gpus N`)."""
import json
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1008_0502_b200 import shard

N_PER_RANK = 5


def fake_digest(t0, n):
    """Deterministic per-frame digests (F, popcount, hash, 0) as gc_frame_digest returns them
    for a solved shard (frame 3 failed: F = -1, empty mask)."""
    rng = np.random.default_rng(1234)
    D = np.zeros((64, 4), np.int64)
    D[:, 0] = rng.integers(0, 10**9, size=64)
    D[:, 1] = rng.integers(0, 5000, size=64)
    D[:, 2] = rng.integers(-(1 << 62), 1 << 62, size=64)
    D[3, :3] = (-1, 0, 0)
    return torch.from_numpy(D[t0:t0 + n].copy())


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t0, n = shard.frame_range(rank, world, N_PER_RANK)
        stats, per = shard.reduce_stats(*shard.frame_stats(fake_digest(t0, n)), world)
        ms = shard.max_over_ranks(10.0 + rank, torch.device("cpu"), world)
        # a rank that re-solved its peer's frames differently is caught
        nxt, _ = shard.frame_range((rank + 1) % world, world, N_PER_RANK)
        chk = fake_digest(nxt, 2)[:, [0, 2]].clone()
        if rank == 1:
            chk[1, 1] += 1
        bad = shard.cross_rank_mismatches(fake_digest(t0, 2)[:, [0, 2]], chk, world, rank)
        if rank == 0:
            out.put((stats.tolist(), per.tolist(), ms, bad))
    finally:
        dist.destroy_process_group()


def test_frame_range():
    assert shard.frame_range(0, 2, 5) == (0, 5)
    assert shard.frame_range(1, 2, 5) == (5, 5)
    with pytest.raises(ValueError):
        shard.frame_range(2, 2, 5)


def test_frame_stats_counts_failures():
    stats, per = shard.frame_stats(fake_digest(0, 6), torch.arange(12).reshape(6, 2))
    D = fake_digest(0, 6).numpy()
    assert stats.tolist() == [int(D[D[:, 0] >= 0, 0].sum()), int(D[:, 1].sum()), 1]
    assert per.shape == (6, 5) and per[:, :3].tolist() == D[:, :3].tolist()


def test_two_rank_gloo_reduction():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = shard.free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    stats, per, ms, bad = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_stats, ref_per = shard.frame_stats(fake_digest(0, world * N_PER_RANK))
    assert stats == ref_stats.tolist()
    assert per == ref_per.tolist()
    assert stats[2] == 1  # the failed frame (F = -1) is counted, not summed
    assert ms == 11.0     # timing = max over ranks
    assert bad == 1       # the one corrupted cross-rank re-solve is found


def test_self_launch_two_ranks(tmp_path):
    """shard.launch_local_ranks -- what `python bench.py --gpus 2` does without torchrun --
    starts two rank processes with RANK/LOCAL_RANK/WORLD_SIZE/MASTER_* set; they rendezvous
    over gloo on 127.0.0.1 and reduce their shards."""
    out = tmp_path / "r0.json"
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_rank_worker.py")
    rc = shard.launch_local_ranks(2, [worker, str(out)], timeout=180)
    assert rc == 0
    res = json.load(open(out))
    ref_stats, ref_per = shard.frame_stats(fake_digest(0, 2 * N_PER_RANK))
    assert res["world"] == 2 and res["stats"] == ref_stats.tolist() and res["per"] == ref_per.tolist()
    assert res["bad"] == 0 and res["ms"] == 6.0


def test_self_launch_reports_failure(tmp_path):
    rc = shard.launch_local_ranks(2, ["-c", "import os,sys; sys.exit(3 if os.environ['RANK']=='1' else 0)"],
                                  timeout=60)
    assert rc == 3
