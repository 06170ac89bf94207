"""Multi-GPU plumbing: trajectories sharded over ranks, map replicated,
one all_gather of (score, global index) for the global argmax (a7).

Trajectory k of the global set lives on rank k mod W (interleaved: feasible/infeasible and
early-exit costs vary ~10x per trajectory, contiguous blocks would be unbalanced).  Every
rank scores its shard with the C ABI (rtg_score + rtg_best), then all ranks exchange a
16-byte (score, index) pair; the global best is the maximum score, ties to the lowest global
index (SPEC S:419 reading, Q11), -1 / -inf when no trajectory is feasible.
Works with the "nccl" backend (CUDA tensors, NVLink/NVSwitch) and "gloo" (CPU, tests).
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np


def shard_indices(K: int, rank: int, world: int) -> np.ndarray:
    """Global trajectory indices owned by `rank`: k = rank, rank + W, rank + 2W, ..."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return np.arange(rank, K, world, dtype=np.int64)


def local_to_global(idx: int, rank: int, world: int) -> int:
    return -1 if idx < 0 else rank + idx * world


def reduce_best(pairs: np.ndarray) -> Tuple[float, int]:
    """pairs [W, 2] of (score, global index) -> (max score, lowest index among ties)."""
    best_s, best_i = -math.inf, -1
    for s, i in pairs:
        i = int(i)
        if i < 0:
            continue
        if s > best_s or (s == best_s and (best_i < 0 or i < best_i)):
            best_s, best_i = float(s), i
    return best_s, best_i


def global_best(score: float, local_idx: int, rank: int, world: int, device=None) -> Tuple[float, int]:
    """All-gather this rank's (score, global index) and return the global best on every rank."""
    import torch
    import torch.distributed as dist
    gidx = local_to_global(local_idx, rank, world)
    if world == 1:
        return (score if gidx >= 0 else -math.inf), gidx
    dev = device if device is not None else torch.device("cpu")
    mine = torch.tensor([score if gidx >= 0 else -math.inf, float(gidx)], dtype=torch.float64, device=dev)
    out = torch.empty(2 * world, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, mine)
    return reduce_best(out.view(world, 2).cpu().numpy())
