"""Multi-GPU environment sharding (the B200 counterpart of the reference's
`ShardedScene`, parallel.py:79-155).

Environments are disjoint constraint islands, so a global batch partitions
across ranks with no data-path communication: rank r owns the contiguous
global env range `shard_range(total, world, r)` (the reference's
`np.linspace` bounds, parallel.py:102-112), builds its scene with
`env_offset = lo` / `total_envs = total`, and every env-dependent quantity
(origins on the global grid, reset / randomisation RNG keys) uses the global
env id -- per-env results are identical whatever the partition.  NCCL is
only used for scalar rollout statistics (and, in a trainer, the PPO gradient
allreduce), never inside the step.
"""

from __future__ import annotations

import os

import numpy as np


def shard_bounds(total_envs: int, world: int):
    """Contiguous partition of [0, total_envs) into `world` ranges."""
    if world < 1 or total_envs < 0:
        raise ValueError("world must be >= 1 and total_envs >= 0")
    return np.linspace(0, total_envs, world + 1).astype(int)


def shard_range(total_envs: int, world: int, rank: int):
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    b = shard_bounds(total_envs, world)
    return int(b[rank]), int(b[rank + 1])


def dist_env():
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def make_sharded_env(name, total_envs, rank=None, world=None, **overrides):
    """This rank's shard of a `total_envs` batch of task `name` on its GPU."""
    from .envs import make_env
    r, w, local = dist_env()
    rank = r if rank is None else rank
    world = w if world is None else world
    lo, hi = shard_range(total_envs, world, rank)
    overrides.setdefault("device", f"cuda:{local}")
    return make_env(name, num_envs=hi - lo, env_offset=lo, total_envs=total_envs, **overrides)


def rollout_stats(reward, done, group=None):
    """Global (mean reward, finished episodes, env count) over all ranks:
    one small allreduce (the only collective next to the hot path)."""
    import torch
    import torch.distributed as dist
    t = torch.stack([reward.double().sum(), done.double().sum(),
                     torch.tensor(float(reward.numel()), dtype=torch.float64, device=reward.device)])
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, group=group)
    return float(t[0] / t[2]), int(t[1]), int(t[2])
