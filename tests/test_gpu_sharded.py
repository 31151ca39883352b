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


def worker(rank, world, port, shards, delta, ne, q, backend="gloo"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if backend == "nccl":
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", 0))
    else:
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


@pytest.mark.parametrize("world,backend", [(1, "gloo"), (2, "gloo"), (1, "nccl")])
def test_sharded_transform_on_device(world, backend):
    """(1, "nccl"): the NCCL data plane itself -- all_gather / all_to_all_single /
    all_reduce on device tensors, no host copies -- on the one GPU of the box."""
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
    procs = [ctx.Process(target=worker, args=(r, world, port, shards, delta, ne, q, backend))
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


def test_device_permutation_helpers():
    # fgt_gather_device / fgt_scatter_device / fgt_merge_runs_device (the
    # sharded path's device data movement) against numpy
    from paper_1909_09825_b200.sharded import DeviceOps
    from paper_1909_09825_b200.transform import uniform_points_array as up
    ops = DeviceOps("cuda:0")
    rng = np.random.default_rng(4)
    v = up(100_003, 31, 0)
    perm = rng.permutation(v.size).astype(np.int32)
    vd, pd = torch.from_numpy(v).cuda(), torch.from_numpy(perm).cuda()
    assert np.array_equal(ops.gather(vd, pd).cpu().numpy(), v[perm])
    sc = np.empty_like(v)
    sc[perm] = v
    assert np.array_equal(ops.scatter(vd, pd).cpu().numpy(), sc)
    for counts in ([5, 0, 17, 100_000], [100_003], [0, 0, 3, 0, 100_000], [1] * 7 + [99_996]):
        runs, o = [], 0
        for c in counts:
            r = np.sort(rng.choice(np.round(v[:2000], 3), size=c)) if c else np.empty(0)
            runs.append(r)
            o += c
        cat = np.concatenate(runs)
        m, p = ops.merge_runs(torch.from_numpy(cat).cuda(), counts)
        ref_p = np.argsort(cat, kind="stable")  # ties in run order
        assert np.array_equal(p.cpu().numpy(), ref_p)
        assert np.array_equal(m.cpu().numpy(), cat[ref_p])


@pytest.mark.parametrize("world", [3])
def test_sharded_transform_unsorted_ragged_three_ranks(world):
    from paper_1909_09825_b200.transform import uniform_points_array as up
    n, m, delta, ne = 120001, 90001, 1e-5, 5
    x, y = up(n, 22, 3), up(m, 22, 0)
    a = up(m, 22, 1)
    cuts_x, cuts_y = [1000, 100000], [0, 89000]  # ragged; rank 0 holds no sources
    shards = [(s_x, s_y, s_a) for s_x, s_y, s_a in
              zip(np.split(x, cuts_x), np.split(y, cuts_y), np.split(a, cuts_y))]
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
