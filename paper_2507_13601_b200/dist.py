"""Multi-GPU sharding of independent FAR instances.

Instances never communicate: rank r solves a contiguous shard with far_solve_many and the only
collective is an all_gather of the per-instance int32 makespans (4 B per instance) and, on request,
of the packed per-task schedules (far_task_slot, 8 B per task) — NCCL over NVLink/NVSwitch on GPUs;
the same code runs over gloo on CPU tensors in the tests.
"""
from __future__ import annotations


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of ceil(total/world) instances for `rank` (the last may be short)."""
    per = -(-total // world) if world > 0 else 0
    lo = min(total, rank * per)
    hi = min(total, lo + per)
    return lo, hi


def padded_shard(total: int, world: int) -> int:
    return -(-total // world) if world > 0 else 0


def gather_makespans(local_ms, total: int, group=None):
    """All-gather the int32 makespans of every rank's shard (padded to equal size) and return
    the [total] tensor of the whole job on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    per = padded_shard(total, world)
    buf = torch.full((per,), -1, dtype=local_ms.dtype, device=local_ms.device)
    buf[: local_ms.numel()] = local_ms
    out = torch.empty(per * world, dtype=local_ms.dtype, device=local_ms.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out[:total]


def gather_schedules(local_sched, total: int, group=None):
    """All-gather the per-task schedules of every rank's shard: local_sched is the uint8
    [shard][n][8] tensor far_solve_many writes (far_task_slot), padded to equal shards; returns
    the [total][n][8] tensor of the whole job on every rank (8 B per task, one collective)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    per = padded_shard(total, world)
    row = tuple(local_sched.shape[1:])
    buf = torch.zeros((per,) + row, dtype=torch.uint8, device=local_sched.device)
    buf[: local_sched.shape[0]] = local_sched
    out = torch.empty((per * world,) + row, dtype=torch.uint8, device=local_sched.device)
    dist.all_gather_into_tensor(out.view(-1), buf.view(-1), group=group)
    return out[:total]
