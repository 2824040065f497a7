"""Rank process for tests/test_multirank.py::test_self_launch_two_ranks: started by
shard.launch_local_ranks (the path `python bench.py --gpus N` takes), it reads its rank from
the environment, joins a gloo group on 127.0.0.1 and runs the statistics reduction and the
cross-rank check of shard.py on deterministic fake shard results; rank 0 writes them."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1008_0502_b200 import shard  # noqa: E402
from test_multirank import N_PER_RANK, fake_digest  # noqa: E402


def main(out_path):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert os.environ["LOCAL_RANK"] == str(rank) and os.environ["MASTER_ADDR"] == "127.0.0.1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t0, n = shard.frame_range(rank, world, N_PER_RANK)
        dg = fake_digest(t0, n)
        stats, per = shard.reduce_stats(*shard.frame_stats(dg), world)
        nxt, _ = shard.frame_range((rank + 1) % world, world, N_PER_RANK)
        bad = shard.cross_rank_mismatches(dg[:2, [0, 2]], fake_digest(nxt, 2)[:, [0, 2]], world, rank)
        ms = shard.max_over_ranks(3.0 * (rank + 1), torch.device("cpu"), world)
        if rank == 0:
            json.dump({"stats": stats.tolist(), "per": per.tolist(), "bad": bad, "ms": ms, "world": world},
                      open(out_path, "w"))
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
