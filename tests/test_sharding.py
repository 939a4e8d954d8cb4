"""Multi-GPU plumbing on CPU: ownership function and the ordered gather over
gloo with world_size 2 (the N>1 path; the GPU box has a single device)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_17084_b200 import sharding


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_owner_partition_is_deterministic_and_balanced():
    rng = np.random.default_rng(0)
    keys = rng.integers(-5000, 5000, (200000, 3))
    for world in (2, 4, 8):
        own = sharding.owner_of(keys, world)
        assert own.min() >= 0 and own.max() < world
        np.testing.assert_array_equal(own, sharding.owner_of(keys, world))
        frac = np.bincount(own, minlength=world) / len(own)
        assert np.all(np.abs(frac - 1 / world) < 0.01)
    # spatially adjacent voxels spread over shards
    line = np.stack([np.arange(64), np.zeros(64), np.zeros(64)], axis=1)
    assert len(set(sharding.owner_of(line, 8))) == 8


def test_pack_keys_matches_device_layout():
    k = np.array([[0, 0, 0], [-1, 2, -3], [(1 << 20) - 1, -(1 << 20), 5]])
    p = sharding.pack_keys(k)
    bias = 1 << 20
    for row, v in zip(k, p):
        a, b, c = (int(x) + bias for x in row)
        assert int(v) == (a << 42) | (b << 21) | c
    with pytest.raises(ValueError):
        sharding.pack_keys([[1 << 20, 0, 0]])


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # records of a global stream split by owner; each rank holds its subset in
        # local (ascending order-key) order, as the device engine emits them
        rng = np.random.default_rng(7)
        n = 301
        order = np.sort(rng.choice(10 ** 6, n, replace=False)).astype(np.int64)
        owner = rng.integers(0, world, n)
        mine = owner == rank
        rec = {"position": torch.from_numpy(np.arange(n * 3, dtype=np.float64).reshape(n, 3)[mine]),
               "source_key": torch.from_numpy(np.arange(n * 3, dtype=np.int64).reshape(n, 3)[mine])}
        out = sharding.gather_records(rec, torch.from_numpy(order[mine]), dst=0)
        if rank == 0:
            q.put((out["position"].numpy(), out["source_key"].numpy()))
    finally:
        dist.destroy_process_group()


def test_ordered_gather_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    pos, keys = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 301
    np.testing.assert_array_equal(pos, np.arange(n * 3, dtype=np.float64).reshape(n, 3))
    np.testing.assert_array_equal(keys, np.arange(n * 3, dtype=np.int64).reshape(n, 3))


def _worker_v(rank, world, port, q, empty_rank):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # a frame's predictions split by owner (81-point blocks per voxel), one
        # rank owning nothing: gather-v of unequal, possibly empty row sets
        rng = np.random.default_rng(11)
        n, m = 157, 81
        order = np.sort(rng.choice(1 << 40, n, replace=False)).astype(np.int64)
        owner = rng.integers(0, world, n)
        owner[owner == empty_rank] = (empty_rank + 1) % world
        mine = owner == rank
        pos = np.arange(n * m * 3, dtype=np.float64).reshape(n, m, 3)
        var = np.arange(n * m, dtype=np.float64).reshape(n, m) * 0.5
        keys = np.arange(n * 3, dtype=np.int64).reshape(n, 3) - 7
        out = sharding.gather_v({"positions": torch.from_numpy(pos[mine]),
                                 "variances": torch.from_numpy(var[mine]),
                                 "keys": torch.from_numpy(keys[mine])},
                                torch.from_numpy(order[mine]), dst=world - 1)
        if rank == world - 1:
            q.put({k: v.numpy() for k, v in out.items()})
        else:
            assert out is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,empty_rank", [(2, 0), (3, 1)])
def test_gather_v_unequal_counts_and_empty_rank(world, empty_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_v, args=(r, world, port, q, empty_rank))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, m = 157, 81
    rng = np.random.default_rng(11)
    order = np.sort(rng.choice(1 << 40, n, replace=False)).astype(np.int64)
    np.testing.assert_array_equal(out["order"], order)
    np.testing.assert_array_equal(out["positions"],
                                  np.arange(n * m * 3, dtype=np.float64).reshape(n, m, 3))
    np.testing.assert_array_equal(out["variances"],
                                  np.arange(n * m, dtype=np.float64).reshape(n, m) * 0.5)
    np.testing.assert_array_equal(out["keys"], np.arange(n * 3, dtype=np.int64).reshape(n, 3) - 7)
