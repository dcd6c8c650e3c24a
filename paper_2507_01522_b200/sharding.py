"""Env sharding across GPUs (one process per GPU, torch.distributed).

The step has no exchange: env i depends only on (its seed, its episode, its
actions) (engine.py:1-8).  A G-GPU job therefore partitions the global env
index range into contiguous shards; GPU g seeds its envs with
split_seed(master, global_i) and binds the device RandomPolicy to the same
global rows, so the union of the shards is bit-identical to one big batch
(the multi-GPU form of the reference's worker-count invariance,
tests/test_engine.py:78-86).  The only collective is the reduction of
rollout statistics (episode returns, counts) — NCCL over NVLink on the GPU
box, gloo in the CPU tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    offset: int  # first global env index
    count: int


def plan(global_envs: int, world: int) -> list[Shard]:
    """Contiguous balanced shards (the reference splits workers the same way, engine.py:449)."""
    if global_envs < world:
        raise ValueError("need at least one env per rank")
    cuts = [global_envs * r // world for r in range(world + 1)]
    return [Shard(r, world, cuts[r], cuts[r + 1] - cuts[r]) for r in range(world)]


def local_shard(global_envs: int) -> Shard:
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    return plan(global_envs, world)[rank]


def reduce_rollout_stats(stats: torch.Tensor) -> torch.Tensor:
    """Sum per-shard statistics across ranks in place (no-op single-process)."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM)
    return stats


def episode_stats_summary(ep_stats: torch.Tensor, done: torch.Tensor) -> torch.Tensor:
    """[count, sum profit, sum reward, sum energy] over envs that just finished
    (ep_stats is the feature-major [8, B] block written at episode end)."""
    m = done.to(torch.float64)
    return torch.stack([m.sum(), (ep_stats[0] * m).sum(), (ep_stats[1] * m).sum(), (ep_stats[5] * m).sum()])
