"""World-size-2 CPU test of the multi-GPU host path over gloo.

The per-chunk device work (fgt_apply_chunk_aggregate / _finish) is emulated
here in numpy with the same chunk semantics, so that the host-side pieces the
ranks actually run are exercised for real: merge-path partition
(bench.merge_split), all_gather of the chunk aggregates through
torch.distributed, the shared carry algebra (fgt_chunk_carries in the C ABI),
and the recombination.  The result must equal the single-process oracle.
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

PD = ctypes.POINTER(ctypes.c_double)


from chunk_emul import chunk_aggregate, chunk_finish, merged  # noqa: E402


def worker(rank, world, port, x, y, a, delta, ne, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1909_09825_b200 import _capi
    t, mw = oracle.folded_table(2 * ne)
    s_all = t / np.sqrt(delta)
    tot = x.size + y.size
    d0, d1 = tot * rank // world, tot * (rank + 1) // world
    i0, i1 = bench.merge_split(x, y, d0), bench.merge_split(x, y, d1)
    j0, j1 = d0 - i0, d1 - i1
    z, b, kind = merged(x[i0:i1], y[j0:j1], a[j0:j1])
    if d0 > 0:
        zprev = max(x[i0 - 1] if i0 > 0 else -np.inf, y[j0 - 1] if j0 > 0 else -np.inf)
    else:
        zprev = z[0]
    agg = np.zeros(3 * ne, complex)
    for k in range(ne):
        agg[k], agg[ne + k], agg[2 * ne + k] = chunk_aggregate(z, b, zprev, s_all[k])
    flat = np.empty(6 * ne)
    flat[0::2], flat[1::2] = agg.real, agg.imag
    buf = [torch.zeros(6 * ne, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(buf, torch.from_numpy(flat))
    allagg = torch.cat(buf).numpy().copy()
    carries = np.empty(world * 4 * ne)
    _capi.check(_capi.lib().fgt_chunk_carries(allagg.ctypes.data_as(PD), world, ne,
                                              carries.ctypes.data_as(PD)))
    c = carries[rank * 4 * ne:(rank + 1) * 4 * ne]
    c = c[0::2] + 1j * c[1::2]
    u = np.zeros(i1 - i0)
    for k in range(ne):
        u += chunk_finish(z, b, kind, zprev, s_all[k], mw[k], c[k], c[ne + k])
    q.put((rank, i0, u))
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_chunked_carry_exchange_matches_single_process(world):
    from paper_1909_09825_b200.transform import uniform_points_array as up
    n, m, delta, ne = 301, 257, 1e-3, 4
    x, y = np.sort(up(n, 5, 3)), np.sort(up(m, 5, 0))
    x[10] = x[11]  # a tie among targets
    y[20] = x[30]  # a source exactly on a target
    a = 2.0 * up(m, 5, 1) - 1.0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, x, y, a, delta, ne, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u = np.zeros(n)
    for _r, i0, part in res:
        u[i0:i0 + part.size] = part
    ref = oracle.transform(x, y, a, delta, ne=ne, mode=0)
    assert np.max(np.abs(u - ref)) <= 1e-12 * np.sum(np.abs(a))
