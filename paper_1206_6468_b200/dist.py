"""Multi-GPU plumbing: one process per GPU, independent mixtures sharded across ranks.

There is no collective on the data path: each rank generates and processes only its own mixtures.
torch.distributed (NCCL on GPUs, gloo in the CPU tests) is used only after the timed region: the MAX
of the per-rank device times and gathers of per-mixture results (free-energy traces, posteriors).
"""
from __future__ import annotations

import os

import numpy as np


def env():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def shard(M: int, world: int, rank: int) -> list[int]:
    """Contiguous block of mixtures owned by `rank`: [rank*M//world, (rank+1)*M//world)."""
    if not (0 <= rank < world) or M < 0:
        raise ValueError("bad shard request")
    return list(range(rank * M // world, (rank + 1) * M // world))


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_mixtures(local: np.ndarray, M: int, device=None):
    """Gather per-mixture rows (local: [len(shard)][...]) from all ranks into [M][...] on every rank,
    ordered by global mixture index.  Shards differ in size by at most one; rows are padded for the
    collective and stripped afterwards."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return np.asarray(local)
    world, rank = dist.get_world_size(), dist.get_rank()
    rows = max(len(shard(M, world, r)) for r in range(world))
    tail = tuple(np.asarray(local).shape[1:])
    buf = torch.zeros((rows,) + tail, dtype=torch.float64, device=device)
    if len(local):
        buf[: len(local)] = torch.as_tensor(np.asarray(local, dtype=np.float64), device=device)
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    parts = [out[r][: len(shard(M, world, r))].cpu().numpy() for r in range(world)]
    return np.concatenate(parts, axis=0)
