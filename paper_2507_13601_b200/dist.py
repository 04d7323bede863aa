"""Multi-GPU sharding of independent FAR instances.

Instances never communicate: rank r solves a contiguous shard with far_solve_many and the only
collective is an all_gather of the per-instance int32 makespans (4 B per instance) — NCCL over
NVLink/NVSwitch on GPUs; the same code runs over gloo on CPU tensors in the tests.
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
