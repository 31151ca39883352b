"""Multi-GPU transform: one process per GPU over torch.distributed.

Every rank holds an arbitrary shard of the targets, sources and strengths
(unsorted, ragged, possibly empty).  ``sharded_transform`` is collective over
the process group:

1. each rank sorts its shard on its GPU (``fgt_sort_device``: stable radix
   sort + permutation);
2. the ranks agree on G-1 splitter coordinates from regular samples of every
   sorted shard (all_gather), so that rank p owns the coordinates in
   (c_{p-1}, c_p]: a contiguous chunk of the global merged stream.  Equal
   coordinates never straddle two ranks, so the reference's merged order
   (sources before targets at ties, transform.cpp:138-147) is preserved;
3. points move with ``all_to_all_single`` (targets; sources + strengths);
4. each rank sorts what it received and runs the chunk scan:
   ``fgt_plan_create_chunk`` (z_prev = last coordinate of the nearest
   non-empty lower rank), ``fgt_apply_chunk_aggregate`` -> all_gather of the
   3 n_e complex chunk aggregates -> ``fgt_chunk_carries`` (same inputs, same
   order on every rank) -> ``fgt_apply_chunk_finish``;
5. the potentials go back to their owners with the inverse all_to_all and
   are scattered to the shard's original target order.

The only data-path collectives are the point exchange (a distributed sort
needs one) and the 288-byte aggregate all_gather; with NCCL they run on device
tensors, with gloo on host copies.  Device work goes through the C ABI
(libfgt1d_b200.so); there is no CPU path.
"""
import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _capi
from .soe import SoeForm, fold

_PD = ctypes.POINTER(ctypes.c_double)
_PU8 = ctypes.POINTER(ctypes.c_uint8)

SAMPLES_PER_SET = 64  # regular samples per rank and point set for the splitters


class DeviceOps:
    """This rank's device work through the C ABI."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.L = _capi.lib()

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def sort(self, v):
        """Stable sort of a float64 device tensor -> (sorted, int64 permutation)."""
        n = v.numel()
        out = torch.empty_like(v)
        perm = torch.empty(n, dtype=torch.int32, device=v.device)
        if n:
            _capi.check(self.L.fgt_sort_device(ctypes.c_void_p(v.data_ptr()), n,
                                               ctypes.c_void_p(out.data_ptr()),
                                               ctypes.c_void_p(perm.data_ptr()), self._stream()))
        return out, perm.long()

    def chunk(self, xs, ys, bs, z_prev, has_prev, delta, soe_args, ne, gather_aggs):
        """Chunk scan of this rank's sorted (xs, ys, bs); gather_aggs maps this
        rank's 6 ne aggregate doubles to the (G, 6 ne) array of all ranks'
        and returns this rank's index.  Returns the potentials (sorted order)."""
        fl = _capi.FGT_DEVICE_PTRS | _capi.FGT_BORROW
        st = self._stream()
        u = torch.empty(max(xs.numel(), 1), dtype=torch.float64, device=xs.device)
        h = ctypes.c_void_p()
        _capi.check(self.L.fgt_plan_create_chunk(
            ctypes.cast(xs.data_ptr(), _PD), xs.numel(), ctypes.cast(ys.data_ptr(), _PD),
            ys.numel(), float(z_prev), int(has_prev), float(delta), *soe_args, fl,
            self.device.index or 0, st, ctypes.byref(h)))
        try:
            agg = np.empty(6 * ne)
            _capi.check(self.L.fgt_apply_chunk_aggregate(h, ctypes.cast(bs.data_ptr(), _PD),
                                                         agg.ctypes.data_as(_PD), fl, st))
            allagg, rank = gather_aggs(agg)
            allagg = np.ascontiguousarray(allagg, dtype=np.float64)
            world = allagg.shape[0]
            carries = np.empty(world * 4 * ne)
            _capi.check(self.L.fgt_chunk_carries(allagg.ctypes.data_as(_PD), world, ne,
                                                 carries.ctypes.data_as(_PD)))
            mine = np.ascontiguousarray(carries[rank * 4 * ne:(rank + 1) * 4 * ne])
            _capi.check(self.L.fgt_apply_chunk_finish(h, ctypes.cast(bs.data_ptr(), _PD),
                                                      mine.ctypes.data_as(_PD),
                                                      ctypes.cast(u.data_ptr(), _PD), fl, st))
        finally:
            self.L.fgt_plan_destroy(h)
        return u[:xs.numel()]


def _soe_args(soe):
    folded = soe if soe.form == SoeForm.FOLDED else fold(soe)
    tr, ti, wr, wi, sc = folded.arrays()
    keep = (tr, ti, wr, wi, sc)
    args = (tr.ctypes.data_as(_PD), ti.ctypes.data_as(_PD), wr.ctypes.data_as(_PD),
            wi.ctypes.data_as(_PD), sc.ctypes.data_as(_PU8), len(folded), int(SoeForm.FOLDED))
    return keep, args, len(folded)


class _Comm:
    """Collectives on device tensors (NCCL) or host copies (gloo)."""

    def __init__(self, group, device):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.host = dist.get_backend(group) != "nccl"
        self.device = device

    def _out(self, t):
        return t.cpu() if self.host else t

    def _in(self, t):
        return t.to(self.device) if self.host else t

    def all_gather(self, t):
        t = self._out(t.contiguous())
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t, group=self.group)
        return self._in(torch.stack(parts))

    def all_to_all(self, t, send_counts, recv_counts):
        t = self._out(t.contiguous())
        out = torch.empty((int(sum(recv_counts)),) + tuple(t.shape[1:]), dtype=t.dtype,
                          device=t.device)
        dist.all_to_all_single(out, t, output_split_sizes=[int(c) for c in recv_counts],
                               input_split_sizes=[int(c) for c in send_counts], group=self.group)
        return self._in(out)


def splitters(sample_z, sample_w, world):
    """G-1 splitter coordinates from the gathered weighted samples: c_p is the
    first sample coordinate at which the cumulative weight reaches p/G of the
    total (deterministic: every rank computes the same values)."""
    z = np.asarray(sample_z, dtype=np.float64).reshape(-1)
    w = np.asarray(sample_w, dtype=np.float64).reshape(-1)
    keep = w > 0
    z, w = z[keep], w[keep]
    if z.size == 0:
        return np.full(world - 1, np.inf)
    order = np.argsort(z, kind="stable")
    z, cw = z[order], np.cumsum(w[order])
    total = cw[-1]
    out = np.empty(world - 1)
    for p in range(1, world):
        i = int(np.searchsorted(cw, p * total / world, side="left"))
        out[p - 1] = z[min(i, z.size - 1)]
    return np.maximum.accumulate(out)


def _samples(v_sorted, k):
    """k regular samples of a sorted vector with weight n/k each (padded)."""
    n = v_sorted.numel()
    z = torch.zeros(k, dtype=torch.float64, device=v_sorted.device)
    w = torch.zeros(k, dtype=torch.float64, device=v_sorted.device)
    if n:
        m = min(k, n)
        idx = (torch.arange(m, device=v_sorted.device, dtype=torch.float64) + 0.5) * (n / m)
        z[:m] = v_sorted[idx.long().clamp(max=n - 1)]
        w[:m] = n / m
    return z, w


def _split_counts(v_sorted, cuts):
    """Elements of a sorted vector per destination rank: (c_{p-1}, c_p]."""
    n = v_sorted.numel()
    if cuts.numel() == 0:
        return [n]
    b = torch.searchsorted(v_sorted, cuts, right=True).cpu().tolist() if n else [0] * cuts.numel()
    edges = [0] + b + [n]
    return [edges[i + 1] - edges[i] for i in range(len(edges) - 1)]


def sharded_transform(targets, sources, strengths, delta, soe, group=None, ops=None):
    """u_i = sum_j exp(-(x_i - y_j)^2 / (4 delta)) alpha_j over the UNION of all
    ranks' shards, returned for this rank's targets in their given order.

    targets / sources / strengths: this rank's float64 tensors on its GPU (any
    order, ragged, possibly empty).  Collective over ``group`` (default: the
    world group).  ``ops`` is the device-work object (default DeviceOps on the
    targets' device)."""
    if not dist.is_initialized():
        raise RuntimeError("sharded_transform needs an initialised torch.distributed group")
    if not (float(delta) > 0.0 and np.isfinite(float(delta))):
        raise ValueError("delta must be positive and finite")
    x = targets.reshape(-1).to(torch.float64)
    y = sources.reshape(-1).to(torch.float64)
    a = strengths.reshape(-1).to(torch.float64)
    if a.numel() != y.numel():
        raise ValueError("one strength per source required")
    device = x.device
    ops = ops or DeviceOps(device)
    comm = _Comm(group, device)
    world, rank = comm.world, comm.rank
    keep, soe_args, ne = _soe_args(soe)

    # 1. local sort
    xs, xp = ops.sort(x)
    ys, yp = ops.sort(y)
    bs = a[yp] if a.numel() else a

    # 2. splitters from regular samples of every rank's sorted shard
    zx, wx = _samples(xs, SAMPLES_PER_SET)
    zy, wy = _samples(ys, SAMPLES_PER_SET)
    smp = comm.all_gather(torch.stack([torch.cat([zx, zy]), torch.cat([wx, wy])]))
    smp = smp.cpu().numpy()  # (world, 2, 2k)
    cuts_np = splitters(smp[:, 0, :], smp[:, 1, :], world)
    cuts = torch.from_numpy(cuts_np).to(device)

    # 3. exchange
    sx = _split_counts(xs, cuts)
    sy = _split_counts(ys, cuts)
    cnt = comm.all_to_all(torch.tensor([[c, d] for c, d in zip(sx, sy)], dtype=torch.int64,
                                       device=device), [1] * world, [1] * world).cpu()
    rx, ry = cnt[:, 0].tolist(), cnt[:, 1].tolist()
    x_recv = comm.all_to_all(xs, sx, rx)
    yb_recv = comm.all_to_all(torch.stack([ys, bs], dim=1) if ys.numel() else
                              torch.empty((0, 2), dtype=torch.float64, device=device), sy, ry)

    # 4. local chunk: sort the received runs, chunk scan with the carry exchange
    xc, xcp = ops.sort(x_recv)
    yc, ycp = ops.sort(yb_recv[:, 0].contiguous())
    bc = yb_recv[:, 1][ycp].contiguous() if yc.numel() else yb_recv[:, 1].contiguous()
    nonempty = xc.numel() + yc.numel() > 0
    last = max(float(xc[-1]) if xc.numel() else -np.inf, float(yc[-1]) if yc.numel() else -np.inf)
    info = comm.all_gather(torch.tensor([1.0 if nonempty else 0.0, last], dtype=torch.float64,
                                        device=device)).cpu().numpy()
    prev = [info[r, 1] for r in range(rank) if info[r, 0] > 0]
    has_prev = len(prev) > 0
    z_prev = prev[-1] if has_prev else 0.0

    def gather_aggs(agg):
        allagg = comm.all_gather(torch.from_numpy(np.ascontiguousarray(agg)).to(device))
        return allagg.cpu().numpy(), rank

    u_sorted = ops.chunk(xc, yc, bc, z_prev, has_prev, delta, soe_args, ne, gather_aggs)
    del keep

    # 5. back to the owners: received order, inverse exchange, original order
    u_recv = torch.empty_like(x_recv)
    if x_recv.numel():
        u_recv[xcp] = u_sorted
    back = comm.all_to_all(u_recv, rx, sx)
    u = torch.empty_like(x)
    if x.numel():
        u[xp] = back
    return u
