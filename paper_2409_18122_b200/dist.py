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


# ---- alternative single-op exchange: all_reduce(MAX) on a packed 64-bit key.
# Valid only when every feasible utility is an integer in [-2^31, 2^31) (the XI variant with an
# integer lambda_xi, e.g. the paper's lambda_xi = 1) and K < 2^32 - 1.  The key
#     key = xi * 2^32 + (2^32 - 1 - k)      (signed int64; none feasible -> INT64_MIN)
# orders by xi first and, among equal xi, by the LOWEST global index k -- the same rule as
# reduce_best -- so one MAX reduction yields the global best on every rank.
_KEY_NONE = -(1 << 63)


def pack_key(score: float, gidx: int) -> int:
    if gidx < 0 or not math.isfinite(score):
        return _KEY_NONE
    if score != math.floor(score) or not (-(1 << 31) <= score < (1 << 31)):
        raise ValueError("packed key needs an integer utility in [-2^31, 2^31)")
    if not (0 <= gidx < (1 << 32) - 1):      # k = 2^32-1 with xi = -2^31 would be INT64_MIN
        raise ValueError("packed key needs a global index in [0, 2^32 - 1)")
    return int(score) * (1 << 32) + ((1 << 32) - 1 - gidx)


def unpack_key(key: int) -> Tuple[float, int]:
    if key == _KEY_NONE:
        return -math.inf, -1
    xi, low = key >> 32, key & 0xFFFFFFFF      # arithmetic shift: floor division for negative xi
    return float(xi), (1 << 32) - 1 - low


def global_best_packed(score: float, local_idx: int, rank: int, world: int, device=None) -> Tuple[float, int]:
    """Like global_best, with one all_reduce(MAX) of a 16-byte (key, invalid) pair instead of an
    all_gather.  A rank whose local best cannot be packed (not an integer utility, or an index
    beyond 2^32 - 2) does not raise before the collective -- that would leave the other ranks
    blocked in it -- but sets `invalid`; when any rank did, every rank falls back to global_best."""
    import torch
    import torch.distributed as dist
    gidx = local_to_global(local_idx, rank, world)
    try:
        key, invalid = pack_key(score, gidx), 0
    except ValueError:
        if world == 1:
            raise
        key, invalid = _KEY_NONE, 1
    if world == 1:
        return unpack_key(key)
    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([key, invalid], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if int(t[1].item()):
        return global_best(score, local_idx, rank, world, device=device)
    return unpack_key(int(t[0].item()))


def gather_outputs(first_col, feasible, gain, utility, K: int, rank: int, world: int, device=None):
    """Optional exchange: all_gather every rank's per-trajectory outputs and return
    them in GLOBAL trajectory order on every rank, as numpy arrays (int32, uint8, float64,
    float64).  Inputs are this rank's shard outputs (length len(shard_indices(K, rank, world)),
    torch tensors or numpy arrays, any device).  One all_gather of [4, ceil(K/W)] float64 per
    rank (first_col and feasible are exact in float64); padding columns are dropped."""
    import torch
    import torch.distributed as dist
    n_loc = len(shard_indices(K, rank, world))
    kmax = -(-K // world) if K > 0 else 0
    dev = device if device is not None else torch.device("cpu")
    buf = torch.zeros((4, kmax), dtype=torch.float64, device=dev)
    for row, a in enumerate((first_col, feasible, gain, utility)):
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        if t.numel() != n_loc:
            raise ValueError("shard output length does not match shard_indices(K, rank, world)")
        buf[row, :n_loc] = t.to(device=dev, dtype=torch.float64)
    if world == 1:
        allb = buf.view(1, 4, kmax)
    else:
        out = torch.empty((world * 4 * kmax,), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(out, buf.reshape(-1))
        allb = out.view(world, 4, kmax)
    allb = allb.cpu().numpy()
    res = np.empty((4, K), dtype=np.float64)
    for r in range(world):
        idx = shard_indices(K, r, world)
        res[:, idx] = allb[r, :, :len(idx)]
    return (res[0].astype(np.int32), res[1].astype(np.uint8), res[2].copy(), res[3].copy())
