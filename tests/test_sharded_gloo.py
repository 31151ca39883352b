"""Multi-rank test of the sharded (distributed-sort) transform host path on CPU
over gloo, world sizes 2 and 3.

The ranks run paper_1909_09825_b200.sharded.sharded_transform for real:
sampling, splitter agreement, all_to_all exchanges, z_prev / has_prev
bookkeeping, the aggregate all_gather, the C-ABI carry algebra
(fgt_chunk_carries) and the inverse exchange.  Only the per-rank device work
(sort, chunk aggregate / finish) is replaced by a numpy emulation (no GPU
here); the GPU suite runs the same path with the real kernels.  The result
must equal the single-process oracle on the union of the shards.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from chunk_emul import chunk_aggregate, chunk_finish, merged


class EmulatedOps:
    """Per-rank device work in numpy (test infrastructure only)."""

    def sort(self, v):
        vn = v.numpy()
        p = np.argsort(vn, kind="stable")
        return torch.from_numpy(vn[p].copy()), torch.from_numpy(p.astype(np.int32))

    def gather(self, src, perm):
        return src[perm.long()]

    def scatter(self, src, perm):
        out = torch.empty(perm.numel(), dtype=torch.float64)
        out[perm.long()] = src
        return out

    def merge_runs(self, v, counts):
        # a stable sort of the concatenated sorted runs is their stable merge
        return self.sort(v)

    def chunk(self, xs, ys, bs, z_prev, has_prev, delta, soe_args, ne, gather_aggs):
        t, mw = oracle.folded_table(2 * ne)
        s_all = t / np.sqrt(delta)
        z, b, kind = merged(xs.numpy(), ys.numpy(), bs.numpy())
        zp = z_prev if has_prev else (z[0] if z.size else 0.0)
        agg = np.zeros(3 * ne, complex)
        for k in range(ne):
            agg[k], agg[ne + k], agg[2 * ne + k] = chunk_aggregate(z, b, zp, s_all[k])
        flat = np.zeros(6 * ne + 1)
        flat[0:6 * ne:2], flat[1:6 * ne:2] = agg.real, agg.imag
        allagg, rank = gather_aggs(torch.from_numpy(flat))
        allagg = np.ascontiguousarray(allagg.numpy()[:, :6 * ne])
        assert allagg.shape[0] >= 1
        from paper_1909_09825_b200 import _capi
        import ctypes
        PD = ctypes.POINTER(ctypes.c_double)
        world = allagg.shape[0]
        carries = np.empty(world * 4 * ne)
        _capi.check(_capi.lib().fgt_chunk_carries(allagg.ctypes.data_as(PD), world, ne,
                                                  carries.ctypes.data_as(PD)))
        c = carries[rank * 4 * ne:(rank + 1) * 4 * ne]
        c = c[0::2] + 1j * c[1::2]
        u = np.zeros(xs.numel())
        for k in range(ne):
            u += chunk_finish(z, b, kind, zp, s_all[k], mw[k], c[k], c[ne + k])
        return torch.from_numpy(u)


def worker(rank, world, port, shards, delta, ne, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1909_09825_b200 import cf_soe, fold
    from paper_1909_09825_b200.sharded import sharded_transform
    x, y, a = (torch.from_numpy(v) for v in shards[rank])
    u = sharded_transform(x, y, a, delta, fold(cf_soe(2 * ne)), ops=EmulatedOps())
    q.put((rank, u.numpy()))
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run(world, shards, delta, ne):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, shards, delta, ne, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [res[r] for r in range(world)]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_unsorted_shards_match_single_process(world):
    from paper_1909_09825_b200.transform import uniform_points_array as up
    rng = np.random.default_rng(world)
    n, m, delta, ne = 700, 500, 1e-3, 4
    x, y = up(n, 9, 3), up(m, 9, 0)
    x[5] = x[6]      # tied targets
    y[7] = x[8]      # a source exactly on a target
    y[9:40] = 0.25   # a block of equal source coordinates (never split)
    a = 2.0 * up(m, 9, 1) - 1.0
    # ragged, unsorted shards; the last rank holds no sources
    cx = np.sort(rng.choice(np.arange(1, n), world - 1, replace=False))
    cy = np.sort(rng.choice(np.arange(1, m), world - 2, replace=False)) if world > 2 else []
    xs = np.split(x, cx)
    ys = np.split(y, list(cy) + [m])
    as_ = np.split(a, list(cy) + [m])
    shards = [(xs[r], ys[r], as_[r]) for r in range(world)]
    parts = run(world, shards, delta, ne)
    u = np.concatenate(parts)
    ref = oracle.transform(x, y, a, delta, ne=ne, mode=0)
    assert u.shape == ref.shape
    assert np.max(np.abs(u - ref)) <= 1e-12 * np.sum(np.abs(a))


def test_splitters_are_monotone_and_balanced():
    from paper_1909_09825_b200.sharded import splitters
    z = np.linspace(0.0, 1.0, 1000)
    c = splitters(z, np.ones_like(z), 4)
    assert np.all(np.diff(c) >= 0)
    assert np.allclose(c, [0.25, 0.5, 0.75], atol=2e-3)
    # zero-weight padding is ignored; all-empty gives +inf (everything on rank 0..)
    assert np.all(np.isinf(splitters(np.zeros(8), np.zeros(8), 3)))


def nan_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1909_09825_b200 import cf_soe, fold
    from paper_1909_09825_b200.sharded import sharded_transform
    from paper_1909_09825_b200.transform import uniform_points_array as up
    x = torch.from_numpy(up(50, rank, 3))
    y = torch.from_numpy(up(40, rank, 0))
    a = torch.from_numpy(up(40, rank, 1))
    if rank == world - 1:
        y[7] = float("nan")  # one bad source on one rank only
    try:
        sharded_transform(x, y, a, 1e-3, fold(cf_soe(8)), ops=EmulatedOps())
        q.put((rank, "no error"))
    except ValueError as e:
        q.put((rank, str(e)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_non_finite_on_one_rank_raises_on_all(world):
    # a domain error on one rank must not leave the others
    # waiting in a collective
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=nan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all("source coordinates must be finite" in res[r] for r in range(world)), res
