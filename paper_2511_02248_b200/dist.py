"""Multi-GPU planning: candidate-range sharding + one MIN all-reduce.

Every window's candidate space [0, prod m_i) is split into contiguous
shards, one per rank (opsc_compose_argmin's `shard / n_shards`). Each rank
min-reduces its shard to a packed key (objective << 40 | lexicographic
index); since the key embeds the global lexicographic index, the MIN
all-reduce over ranks (NCCL over NVLink on GPUs, gloo in the CPU tests)
returns exactly the single-GPU decision for any world size. Menus are cheap
(~1 us per window) and are rebuilt on every rank, so the all-reduce of
[W] int64 keys is the only data-path exchange.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import abi


def merge_keys(keys: torch.Tensor, group=None) -> torch.Tensor:
    """In-place MIN all-reduce of per-window packed keys (int64)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
    return keys


def rank_shard(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def plan_windows_sharded(planner, group=None):
    """Run one DevicePlanner step with this rank's shard and the NCCL merge;
    every rank ends with the full decisions of every window."""
    rank, world = rank_shard(group)
    planner.step(rank, world, allreduce=lambda k: merge_keys(k, group))
    return planner


def plan_windows_host_sharded(planner, host_windows, host_out, group=None):
    """Host buffers in, decisions out, on N ranks: H2D of the window SoA,
    this rank's candidate shard, the MIN merge, decode + materialise, D2H.
    `host_out` (tables.DecisionArrays) ends with the full decisions on every
    rank."""
    planner.load_windows(host_windows)
    plan_windows_sharded(planner, group)
    return planner.fetch(host_out)


def infeasible_keys(n, device="cpu"):
    return torch.full((n,), abi.KEY_INFEASIBLE, dtype=torch.int64, device=device)
