"""Head sharding across GPUs.

Heads are independent end to end in the reference (one head per cmd_run call,
proj/tools/main.cpp:276-300; per-head plans and masks), so rank g of P owns the
contiguous heads [g*H/P, (g+1)*H/P): its own Q/K/V slice, orders and masks, and
no data crosses GPUs on the hot path. The only collective is an all-gather
that reassembles the layer output [H, N, d] where a caller needs it (tests),
run outside the timed region.
"""
from __future__ import annotations

from typing import List, Sequence


def shard_heads(heads: int, world: int, rank: int) -> List[int]:
    """Heads owned by `rank` (contiguous block; every config's H divides 1/2/4/8)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of world {world}")
    if heads % world:
        raise ValueError(f"{heads} heads do not split evenly over {world} ranks")
    per = heads // world
    return list(range(rank * per, (rank + 1) * per))


def shard_orders(orders: Sequence[str], world: int, rank: int) -> List[str]:
    return [orders[h] for h in shard_heads(len(orders), world, rank)]


def gather_layer(local, group=None):
    """all_gather of each rank's [H/P, N, d] output into [H, N, d] (rank order
    == head order). Works with NCCL (CUDA tensors) and gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, dim=0)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """The slowest rank's time (multi-GPU numbers are max over ranks)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
