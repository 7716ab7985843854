"""Batch partition across the GPUs of one box.

Chains are independent, so a batch of B problems is split into G contiguous
slices of ceil(B/G); each rank (one process per GPU) solves its slice with no
collective on the hot path. Results are bit-identical for any G because each
chain's arithmetic does not depend on the partition. The optional final
gather of qddot to rank 0 is a single torch.distributed gather (NCCL over
NVLink on GPUs, gloo on CPU), timed separately from the solves.
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np


def shard_bounds(total: int, world: int, rank: int) -> Tuple[int, int]:
    """[begin, end) of rank's contiguous slice; slices of ceil(total/world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    per = -(-total // world)
    b = min(total, rank * per)
    return b, min(total, b + per)


def gather_rows(local: np.ndarray, total: int, world: int, rank: int, group=None) -> Optional[np.ndarray]:
    """Gathers each rank's (rows_r, n) float64 slice into a (total, n) array on
    rank 0 (None elsewhere). Uses a padded dist.gather so every rank sends the
    same shape."""
    import torch
    import torch.distributed as dist

    per = -(-total // world)
    n = local.shape[1]
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros((per, n), dtype=torch.float64, device=device)
    buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local)).to(device)
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, parts, dst=0, group=group)
    if rank != 0:
        return None
    out = np.empty((total, n))
    for r in range(world):
        b, e = shard_bounds(total, world, r)
        out[b:e] = parts[r][: e - b].cpu().numpy()
    return out
