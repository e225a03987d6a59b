"""Multi-process (gloo, world_size 2, CPU) tests of the data-parallel host logic."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_09767_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.full((1000,), float(rank + 1))
        parallel.allreduce_mean_(g)
        # identical Adam-state trajectory requires bitwise-identical grads on every rank
        gathered = [torch.empty_like(g) for _ in range(world)]
        dist.all_gather(gathered, g)
        out[rank] = (float(g[0]), all(torch.equal(gathered[0], x) for x in gathered),
                     [parallel.shard_index(s, rank, world) for s in range(3)])
    finally:
        dist.destroy_process_group()


def test_allreduce_mean_and_sharding_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        mean, same, shards = out[r]
        assert mean == pytest.approx(1.5)
        assert same
        assert shards == [0 * world + r, 1 * world + r, 2 * world + r]
    # every sequence index is used exactly once across ranks
    all_idx = sorted(i for r in range(world) for i in out[r][2])
    assert all_idx == list(range(3 * world))


def test_allreduce_is_noop_without_process_group():
    g = torch.arange(4.0)
    assert torch.equal(parallel.allreduce_mean_(g.clone()), g)
