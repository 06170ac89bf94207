"""Multi-rank host logic on CPU (gloo, world_size 2): sharding and the global argmax exchange."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_18122_b200 import dist as D


def test_shards_partition_all_trajectories():
    for K, W in ((10, 3), (16384, 8), (5, 8), (1, 1)):
        parts = [D.shard_indices(K, r, W) for r in range(W)]
        allk = np.sort(np.concatenate(parts))
        assert np.array_equal(allk, np.arange(K))
        for r, p in enumerate(parts):
            assert all(D.local_to_global(j, r, W) == k for j, k in enumerate(p))


def test_reduce_best_ties_and_none():
    assert D.reduce_best(np.array([[3.0, 7], [5.0, 9], [5.0, 2]])) == (5.0, 2)
    assert D.reduce_best(np.array([[-math.inf, -1], [-math.inf, -1]])) == (-math.inf, -1)
    assert D.reduce_best(np.array([[-math.inf, -1], [-2.0, 4]])) == (-2.0, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rtg_best_shaped(local):
    """This rank's local best exactly as rtg.best() returns it from rtg_best (include/rtg.h): the
    (score, LOCAL index) pair of the oracle's O7 rule (max, ties -> lowest index),
    which rtg_best is parity-tested against on the GPU, and (-inf, -1) with RTG_ERR_NO_FEASIBLE."""
    from oracle import oracle as O
    j = O.best(np.asarray(local, np.float64))
    return (float(local[j]), j) if j >= 0 else (-math.inf, -1)


def _worker(rank, world, port, utility, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        idx = D.shard_indices(len(utility), rank, world)
        s, j = _rtg_best_shaped(utility[idx])
        q.put((rank, D.global_best(s, j, rank, world)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["random", "ties_across_ranks", "none_feasible"])
def test_global_best_gloo_world2(case):
    rng = np.random.default_rng(3)
    u = rng.normal(size=101)
    u[rng.random(101) < 0.4] = -np.inf
    if case == "ties_across_ranks":
        u[:] = -np.inf
        u[[7, 4, 10]] = 2.5            # 4 -> rank 0, 7 -> rank 1, 10 -> rank 0
    if case == "none_feasible":
        u[:] = -np.inf
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, u, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if np.all(np.isneginf(u)):
        expect = (-math.inf, -1)
    else:
        k = int(np.argmax(u))
        expect = (float(u[k]), k)
    assert res[0] == res[1] == expect


def test_packed_key_orders_like_reduce_best():
    rng = np.random.default_rng(11)
    for _ in range(200):
        W = int(rng.integers(1, 6))
        pairs = []
        for r in range(W):
            if rng.random() < 0.2:
                pairs.append((-math.inf, -1))
            else:
                pairs.append((float(rng.integers(-5, 5)), int(rng.integers(0, (1 << 32) - 1))))
        keys = [D.pack_key(s, i) for s, i in pairs]
        assert D.unpack_key(max(keys)) == D.reduce_best(np.array(pairs, dtype=object))
    for s, i in ((0.0, 0), (-(2.0 ** 31), (1 << 32) - 2), (2.0 ** 31 - 1, 5), (-1.0, 3)):
        assert D.unpack_key(D.pack_key(s, i)) == (s, i)
    with pytest.raises(ValueError):
        D.pack_key(1.5, 0)
    with pytest.raises(ValueError):
        D.pack_key(2.0 ** 31, 0)
    with pytest.raises(ValueError):
        D.pack_key(-(2.0 ** 31), (1 << 32) - 1)


def _worker_outputs(rank, world, port, fc, fe, g, u, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K = len(u)
        idx = D.shard_indices(K, rank, world)
        out = D.gather_outputs(torch.from_numpy(fc[idx]), fe[idx], g[idx], torch.from_numpy(u[idx]), K, rank, world)
        s, j = _rtg_best_shaped(u[idx])
        q.put((rank, out, D.global_best_packed(s, j, rank, world)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("K", [101, 1, 0])
def test_gather_outputs_and_packed_best_gloo_world2(K):
    rng = np.random.default_rng(5)
    fc = rng.integers(-1, 100, size=K).astype(np.int32)
    fe = (fc < 0).astype(np.uint8)
    g = rng.normal(size=K)
    g[fe == 0] = np.nan
    u = np.where(fe == 1, rng.integers(-3, 4, size=K).astype(np.float64), -np.inf)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_outputs, args=(r, world, port, fc, fe, g, u, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: (o, b) for r, o, b in (q.get(timeout=120) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if K == 0 or np.all(np.isneginf(u)):
        expect_best = (-math.inf, -1)
    else:
        expect_best = (float(u.max()), int(np.argmax(u)))
    for r in range(world):
        o, b = res[r]
        assert np.array_equal(o[0], fc) and np.array_equal(o[1], fe)
        assert np.array_equal(o[2], g, equal_nan=True) and np.array_equal(o[3], u)
        assert b == expect_best


def _worker_packed_invalid(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank 1's best is not an integer utility (e.g. the SUM variant): it must not raise before
        # the collective (rank 0 would block in it); every rank falls back to the all_gather
        s, j = (3.0, 0) if rank == 0 else (3.5, 2)
        q.put((rank, D.global_best_packed(s, j, rank, world)))
    finally:
        dist.destroy_process_group()


def test_packed_best_falls_back_on_every_rank_when_one_is_invalid():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_packed_invalid, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1] == (3.5, 1 + 2 * 2)     # rank 1, local 2 -> global 5
