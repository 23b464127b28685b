"""Multi-GPU layout: one process per GPU, members sharded across ranks.

The GL history sum is pointwise in space and members of an ensemble never
interact, so an ensemble (BASELINE c5) shards by member with no
data-path collective at all: rank r owns a contiguous block of members, streams
only its own history slices, and the only collective is the max-over-ranks of
the device-timed loop for reporting.  A single-member workload (c2) runs one
independently seeded member per rank — the same weak-scaling layout.
(Spatial slab sharding with a per-step halo exchange is the next item.)
"""

from __future__ import annotations

import os
from dataclasses import replace

import numpy as np


def dist_env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults 0, 1, 0)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def member_range(n_members: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced block of members owned by ``rank`` (sizes differ by ≤ 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(int(n_members), world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_config(cfg, rank: int, world: int):
    """This rank's share of a ``FieldConfig``: a member block of an ensemble."""
    if world == 1:
        return cfg
    if not cfg.batched:
        raise ValueError("only batched (ensemble) configs shard by member; use replica_config")
    lo, hi = member_range(cfg.members(), rank, world)
    idx = np.arange(lo, hi)
    return replace(cfg, initial=np.asarray(cfg.initial)[idx],
                   gamma=np.broadcast_to(np.asarray(cfg.gamma, dtype=np.float64), (cfg.members(),))[idx],
                   dt=np.broadcast_to(np.asarray(cfg.dt, dtype=np.float64), (cfg.members(),))[idx])


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (loop time) over the process group, if any."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
