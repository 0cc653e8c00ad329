"""Multi-GPU plumbing for the O(|V|) rebuild.

A node's exact recompute reads only its own memory row and its ring (the
frozen payloads of its top-L entries, copied at insertion), so a full
rebuild partitions by node-id range with no communication during the
recompute. Replicas that each hold the full state split the node range,
recompute their shard, and all-gather the layer-cache rows so every
replica ends bit-identical to a single-GPU rebuild. One process per GPU,
torch.distributed (NCCL on B200s; gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous node-id range [lo, hi) of `rank`; sizes differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_rows(rows, n: int, group=None):
    """All-gather per-rank row blocks (rank r holds rows shard_range(n, W, r))
    into one [n, ...] tensor on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(n, world, rank)
    if rows.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {rows.shape[0]} rows, expected {hi - lo}")
    cap = -(-n // world)  # equal-size buffers for all_gather
    send = torch.zeros((cap,) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
    send[:hi - lo] = rows
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    parts = []
    for r in range(world):
        a, b = shard_range(n, world, r)
        parts.append(recv[r][:b - a])
    return torch.cat(parts, dim=0)


def sharded_rebuild(recompute, n: int, group=None):
    """Distributed full rebuild: `recompute(lo, hi)` returns this rank's
    recomputed rows for node ids [lo, hi); the result is every row on every
    rank. With the CUDA engine, recompute = engine.rebuild_range."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(n, world, rank)
    return gather_rows(recompute(lo, hi), n, group)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (timings are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def replica_seeds(base_seed: int, world: int) -> np.ndarray:
    """Stream seeds of the weak-scaling replicas (rank r streams seed base+r)."""
    return base_seed + np.arange(world)
