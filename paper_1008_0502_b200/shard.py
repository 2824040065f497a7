"""Multi-GPU plumbing of the batched solve.

Frames are independent problems (each is its own graph), so N ranks -- one
process per GPU -- take contiguous frame shards and solve whole frames with no data-path
collective ("weak" scaling).  The only collective is the final statistics reduction:
one all_reduce of the per-rank sums and one all_gather of the per-frame (F, popcount)
pairs.  The functions take whatever process group torch.distributed was initialised
with (NCCL on the GPU box; gloo in the CPU tests), so the same code is tested on CPU.
"""
from __future__ import annotations

import torch


def frame_range(rank: int, world: int, frames_per_rank: int) -> tuple[int, int]:
    """(first frame index, frame count) of `rank`'s shard: contiguous, frames_per_rank each."""
    if not (0 <= rank < world) or frames_per_rank < 0:
        raise ValueError(f"bad shard rank={rank} world={world} frames_per_rank={frames_per_rank}")
    return rank * frames_per_rank, frames_per_rank


def frame_stats(flow: torch.Tensor, mask: torch.Tensor):
    """Per-rank statistics of a solved shard: ([sum F, sum popcount, failed frames] int64,
    per-frame [n, 2] int64 of (F, popcount)).  Failed frames carry F = -1 (gc.h)."""
    n = flow.shape[0]
    pop = mask.reshape(n, -1).sum(dim=1, dtype=torch.int64)
    flow = flow.to(torch.int64)
    ok = flow >= 0
    stats = torch.stack([torch.where(ok, flow, torch.zeros_like(flow)).sum(), pop.sum(),
                         (~ok).sum().to(torch.int64)])
    return stats, torch.stack([flow, pop], dim=1)


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


def max_over_ranks(ms: float, device, world: int) -> float:
    """Timing of a multi-GPU step: the slowest rank's device time."""
    if world <= 1:
        return ms
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
