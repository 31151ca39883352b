"""Sharded (distributed-sort) transform with the real device kernels.

World 1, and world 2 over gloo with both ranks on the one GPU of the box:
every collective goes through host copies and no kernel waits on a peer, so
the ranks only share the device; the numbers are not a scaling measurement.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu


def worker(rank, world, port, shards, delta, ne, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1909_09825_b200 import cf_soe, fold
    from paper_1909_09825_b200.sharded import sharded_transform
    x, y, a = (torch.from_numpy(v).cuda() for v in shards[rank])
    u = sharded_transform(x, y, a, delta, fold(cf_soe(2 * ne)))
    torch.cuda.synchronize()
    q.put((rank, u.cpu().numpy()))
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2])
def test_sharded_transform_on_device(world):
    from paper_1909_09825_b200.transform import uniform_points_array as up
    n, m, delta, ne = 200003, 150001, 1e-4, 6
    x, y = up(n, 21, 3), up(m, 21, 0)
    y[100:400] = x[50]  # equal coordinates across sets
    a = 2.0 * up(m, 21, 1) - 1.0
    xs, ys, as_ = np.array_split(x, world), np.array_split(y, world), np.array_split(a, world)
    shards = [(xs[r], ys[r], as_[r]) for r in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, shards, delta, ne, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u = np.concatenate([res[r] for r in range(world)])
    ref = oracle.transform(x, y, a, delta, ne=ne, mode=0)
    assert np.max(np.abs(u - ref)) <= 1e-12 * np.sum(np.abs(a))
