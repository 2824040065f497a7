"""Multi-GPU plumbing of the batched solve.

Frames are independent problems (each is its own graph), so N ranks -- one
process per GPU -- take contiguous frame shards and solve whole frames with no data-path
collective ("weak" scaling).  The only collective is the final statistics reduction:
one all_reduce of the per-rank sums and one all_gather of the per-frame digests
(F, popcount, 64-bit mask hash; computed on the device by gc_frame_digest), which makes
rank-count invariance checkable.  The functions take whatever process group
torch.distributed was initialised with (NCCL on the GPU box; gloo in the CPU tests), so
the same code is tested on CPU.  ``launch_local_ranks`` starts one process per GPU when a
script is run without a launcher (``python bench.py --gpus N``).
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import torch


def frame_range(rank: int, world: int, frames_per_rank: int) -> tuple[int, int]:
    """(first frame index, frame count) of `rank`'s shard: contiguous, frames_per_rank each."""
    if not (0 <= rank < world) or frames_per_rank < 0:
        raise ValueError(f"bad shard rank={rank} world={world} frames_per_rank={frames_per_rank}")
    return rank * frames_per_rank, frames_per_rank


def frame_stats(digest: torch.Tensor, counters: torch.Tensor | None = None):
    """Per-rank statistics of a solved shard from its per-frame digest [n, 4] int64
    (F, popcount, mask hash, 0 -- gc_frame_digest) and optional per-frame solver counters
    [n, c] (stats_out: push tasks, global relabels, ...).  Returns ([sum F over solved frames,
    sum popcount, failed frames] int64, per-frame [n, 3 + c] int64 of (F, popcount, hash,
    counters...)).  Failed frames carry F = -1 (gc.h)."""
    digest = digest.to(torch.int64)
    flow, pop = digest[:, 0], digest[:, 1]
    ok = flow >= 0
    stats = torch.stack([torch.where(ok, flow, torch.zeros_like(flow)).sum(), pop.sum(),
                         (~ok).sum().to(torch.int64)])
    per = digest[:, :3]
    if counters is not None:
        per = torch.cat([per, counters.to(torch.int64).reshape(per.shape[0], -1)], dim=1)
    return stats, per.contiguous()


def reduce_stats(stats: torch.Tensor, per_frame: torch.Tensor, world: int):
    """The one collective of the path: sums over ranks and the per-frame table of all ranks
    (rank order = frame order).  world == 1 returns the inputs."""
    if world <= 1:
        return stats, per_frame
    import torch.distributed as dist
    stats = stats.clone()
    dist.all_reduce(stats)
    gathered = [torch.empty_like(per_frame) for _ in range(world)]
    dist.all_gather(gathered, per_frame.contiguous())
    return stats, torch.cat(gathered)


def cross_rank_mismatches(own: torch.Tensor, peer_check: torch.Tensor, world: int, rank: int) -> int:
    """Rank-count invariance: every rank re-solves the first m frames of the next rank's shard
    and reports their (F, hash) in `peer_check` [m, 2]; `own` [m, 2] is this rank's (F, hash) of
    its own first m frames.  Gathers both and counts frames where the two solves disagree
    (frames solved on different GPUs / in different launches must be identical)."""
    if world <= 1:
        return int((own != peer_check).any(dim=1).sum().item())
    import torch.distributed as dist
    g_own = [torch.empty_like(own) for _ in range(world)]
    g_chk = [torch.empty_like(peer_check) for _ in range(world)]
    dist.all_gather(g_own, own.contiguous())
    dist.all_gather(g_chk, peer_check.contiguous())
    bad = 0
    for r in range(world):  # rank r checked rank (r + 1) % world
        bad += int((g_chk[r] != g_own[(r + 1) % world]).any(dim=1).sum().item())
    return bad


def max_over_ranks(ms: float, device, world: int) -> float:
    """Timing of a multi-GPU step: the slowest rank's device time."""
    if world <= 1:
        return ms
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_local_ranks(world: int, argv: list[str], env: dict | None = None, timeout: float | None = None) -> int:
    """Run `python argv...` as ranks 0..world-1 of one node (one process per GPU): each gets
    RANK = LOCAL_RANK = r, WORLD_SIZE, LOCAL_WORLD_SIZE, MASTER_ADDR = 127.0.0.1 and a free
    MASTER_PORT, and inherits stdout/stderr.  Returns the worst exit code (0 if all succeed);
    if one rank fails the others are terminated."""
    port = free_port()
    procs = []
    for r in range(world):
        e = dict(os.environ)
        e.update(env or {})
        e.update({"RANK": str(r), "LOCAL_RANK": str(r), "WORLD_SIZE": str(world), "LOCAL_WORLD_SIZE": str(world),
                  "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
        procs.append(subprocess.Popen([sys.executable] + list(argv), env=e))
    rc = 0
    try:
        pending = list(procs)
        import time
        t0 = time.time()
        while pending:
            for p in list(pending):
                c = p.poll()
                if c is None:
                    continue
                pending.remove(p)
                if c != 0:
                    rc = rc or c
                    for q in pending:
                        q.terminate()
            if timeout is not None and time.time() - t0 > timeout:
                for q in pending:
                    q.terminate()
                rc = rc or 124
                break
            time.sleep(0.05)
    finally:
        for p in procs:
            try:
                p.wait(timeout=30)
            except Exception:
                p.kill()
    return rc
