"""Multi-GPU transform: one process per GPU over torch.distributed.

Every rank holds an arbitrary shard of the targets, sources and strengths
(unsorted, ragged, possibly empty).  ``sharded_transform`` is collective over
the process group:

0. the ranks agree that every coordinate is finite (one all_reduce of two
   flags) before any data moves, so a bad value on one rank raises the same
   error on all of them (check_points, transform.cpp:21-25, targets first);
1. each rank sorts its shard on its GPU (``fgt_sort_device``: stable radix
   sort + permutation) and gathers its strengths into sorted-source order
   (``fgt_gather_device``);
2. the ranks agree on G-1 splitter coordinates from regular samples of every
   sorted shard (all_gather), so that rank p owns the coordinates in
   (c_{p-1}, c_p]: a contiguous chunk of the global merged stream.  Equal
   coordinates never straddle two ranks, so the reference's merged order
   (sources before targets at ties, transform.cpp:138-147) is preserved.  One
   more all_gather carries every rank's send counts and its largest
   coordinate at or below each splitter; its single host read gives the
   exchange sizes and every rank's chunk predecessor z_prev;
3. points move with ``all_to_all_single`` (targets; sources + strengths);
4. each rank merges the G sorted runs it received (``fgt_merge_runs_device``,
   merge path, stable in rank order) and runs the chunk scan on the device:
   ``fgt_plan_create_chunk``, ``fgt_apply_chunk_aggregate`` into a device
   array, all_gather of the 3 n_e complex chunk aggregates (+ a status
   word), ``fgt_chunk_carries_device``, ``fgt_apply_chunk_finish``;
5. the potentials go back to their owners with the inverse all_to_all and
   are scattered to the shard's original target order (``fgt_scatter_device``).

The data-path collectives are the point exchange (a distributed sort needs
one) and the aggregate all_gather; with NCCL they run on device tensors,
with gloo on host copies.  Device work goes through the C ABI
(libfgt1d_b200.so); there is no CPU path.
"""
import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _capi
from .soe import SoeForm, fold

_PD = ctypes.POINTER(ctypes.c_double)
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PU8 = ctypes.POINTER(ctypes.c_uint8)

SAMPLES_PER_SET = 64  # regular samples per rank and point set for the splitters


def _vp(t):
    return ctypes.c_void_p(t.data_ptr())


class DeviceOps:
    """This rank's device work through the C ABI (stream-ordered on the
    current torch stream of the device)."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.L = _capi.lib()

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def sort(self, v):
        """Stable sort of a float64 device tensor -> (sorted, int32 permutation)."""
        n = v.numel()
        out = torch.empty_like(v)
        perm = torch.empty(n, dtype=torch.int32, device=v.device)
        if n:
            _capi.check(self.L.fgt_sort_device(_vp(v), n, _vp(out), _vp(perm), self._stream()))
        return out, perm

    def gather(self, src, perm):
        """out[i] = src[perm[i]]."""
        out = torch.empty(perm.numel(), dtype=torch.float64, device=src.device)
        if perm.numel():
            _capi.check(self.L.fgt_gather_device(_vp(src), _vp(perm), perm.numel(), _vp(out),
                                                 self._stream()))
        return out

    def scatter(self, src, perm):
        """out[perm[i]] = src[i]."""
        out = torch.empty(perm.numel(), dtype=torch.float64, device=src.device)
        if perm.numel():
            _capi.check(self.L.fgt_scatter_device(_vp(src), _vp(perm), perm.numel(), _vp(out),
                                                  self._stream()))
        return out

    def merge_runs(self, v, counts):
        """Stable merge of the sorted runs of v (lengths counts, in order) ->
        (merged, int32 permutation merged[i] == v[perm[i]])."""
        off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        out = torch.empty_like(v)
        perm = torch.empty(v.numel(), dtype=torch.int32, device=v.device)
        if v.numel():
            _capi.check(self.L.fgt_merge_runs_device(_vp(v), off.ctypes.data_as(_PI64), len(counts),
                                                     _vp(out), _vp(perm), self._stream()))
        return out, perm

    def chunk(self, xs, ys, bs, z_prev, has_prev, delta, soe_args, ne, gather_aggs):
        """Chunk scan of this rank's sorted (xs, ys, bs).  gather_aggs maps this
        rank's device tensor of 6 ne aggregate doubles + 1 status word to the
        device tensor of all ranks' (G x (6 ne + 1)) and this rank's index; a
        rank that failed before the exchange still takes part (status 1) so
        that every rank raises instead of waiting.  Returns the potentials
        (sorted order)."""
        fl = _capi.FGT_DEVICE_PTRS | _capi.FGT_BORROW | _capi.FGT_DEVICE_AGGS
        st = self._stream()
        dev = xs.device
        u = torch.empty(max(xs.numel(), 1), dtype=torch.float64, device=dev)
        agg = torch.zeros(6 * ne + 1, dtype=torch.float64, device=dev)
        h = ctypes.c_void_p()
        err = None
        try:
            _capi.check(self.L.fgt_plan_create_chunk(
                ctypes.cast(xs.data_ptr(), _PD), xs.numel(), ctypes.cast(ys.data_ptr(), _PD),
                ys.numel(), float(z_prev), int(has_prev), float(delta), *soe_args, fl,
                dev.index or 0, st, ctypes.byref(h)))
            _capi.check(self.L.fgt_apply_chunk_aggregate(h, ctypes.cast(bs.data_ptr(), _PD),
                                                         ctypes.cast(agg.data_ptr(), _PD), fl, st))
        except Exception as e:  # noqa: BLE001 -- re-raised after the collective
            err = e
            agg[-1] = 1.0
        try:
            allagg, rank = gather_aggs(agg)
            if float(allagg[:, -1].max()) != 0.0:
                raise err if err is not None else RuntimeError(
                    "sharded_transform: the chunk scan failed on another rank")
            world = allagg.shape[0]
            aggs = allagg[:, :6 * ne].contiguous()
            car = torch.empty(4 * ne, dtype=torch.float64, device=dev)
            _capi.check(self.L.fgt_chunk_carries_device(_vp(aggs), world, ne, rank, _vp(car), st))
            _capi.check(self.L.fgt_apply_chunk_finish(h, ctypes.cast(bs.data_ptr(), _PD),
                                                      ctypes.cast(car.data_ptr(), _PD),
                                                      ctypes.cast(u.data_ptr(), _PD), fl, st))
        finally:
            if h.value:
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

    def all_reduce_max(self, t):
        t = self._out(t.contiguous()).clone()
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return self._in(t)

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


def _split(v_sorted, cuts):
    """Per destination rank: element counts of (c_{p-1}, c_p] and, per
    splitter, the largest element <= c_q (-inf if none), on the device."""
    n = v_sorted.numel()
    g1 = cuts.numel()
    if g1 == 0:
        return (torch.tensor([n], dtype=torch.float64, device=v_sorted.device),
                torch.empty(0, dtype=torch.float64, device=v_sorted.device))
    if n == 0:
        return (torch.zeros(g1 + 1, dtype=torch.float64, device=v_sorted.device),
                torch.full((g1,), -np.inf, dtype=torch.float64, device=v_sorted.device))
    b = torch.searchsorted(v_sorted, cuts, right=True)
    edges = torch.cat([torch.zeros(1, dtype=b.dtype, device=b.device), b,
                       torch.full((1,), n, dtype=b.dtype, device=b.device)])
    counts = (edges[1:] - edges[:-1]).to(torch.float64)
    last = torch.where(b > 0, v_sorted[(b - 1).clamp(min=0)],
                       torch.full_like(cuts, -np.inf))
    return counts, last


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
    device = x.device
    ops = ops or DeviceOps(device)
    comm = _Comm(group, device)
    world, rank = comm.world, comm.rank
    keep, soe_args, ne = _soe_args(soe)

    # 0. every rank learns whether any coordinate anywhere is non-finite and
    # whether any shard's strength count is off (one collective, then the
    # same exception everywhere, in the reference's order)
    bad = torch.stack([(~torch.isfinite(x)).any(), (~torch.isfinite(y)).any(),
                       torch.tensor(a.numel() != y.numel(), device=device)]).to(torch.float64)
    bad = comm.all_reduce_max(bad).cpu().numpy()
    if bad[0]:
        raise ValueError("target coordinates must be finite")
    if bad[1]:
        raise ValueError("source coordinates must be finite")
    if bad[2]:
        raise ValueError("one strength per source required")

    # 1. local sort; strengths in sorted-source order
    xs, xp = ops.sort(x)
    ys, yp = ops.sort(y)
    bs = ops.gather(a, yp)

    # 2. splitters from regular samples of every rank's sorted shard
    zx, wx = _samples(xs, SAMPLES_PER_SET)
    zy, wy = _samples(ys, SAMPLES_PER_SET)
    smp = comm.all_gather(torch.stack([torch.cat([zx, zy]), torch.cat([wx, wy])]))
    smp = smp.cpu().numpy()  # (world, 2, 2k)
    cuts = torch.from_numpy(splitters(smp[:, 0, :], smp[:, 1, :], world)).to(device)
    # send counts and the largest coordinate at or below each splitter, all
    # ranks' in one gather (the only host read after splitter agreement)
    cxn, lx = _split(xs, cuts)
    cyn, ly = _split(ys, cuts)
    info = comm.all_gather(torch.cat([cxn, cyn, torch.maximum(lx, ly)])).cpu().numpy()
    sx = info[rank, :world].astype(np.int64).tolist()
    sy = info[rank, world:2 * world].astype(np.int64).tolist()
    rx = info[:, rank].astype(np.int64).tolist()
    ry = info[:, world + rank].astype(np.int64).tolist()
    z_prev = float(info[:, 2 * world + rank - 1].max()) if rank > 0 else -np.inf
    has_prev = bool(np.isfinite(z_prev))

    # 3. exchange
    x_recv = comm.all_to_all(xs, sx, rx)
    yb_recv = comm.all_to_all(torch.stack([ys, bs], dim=1) if ys.numel() else
                              torch.empty((0, 2), dtype=torch.float64, device=device), sy, ry)

    # 4. merge the received sorted runs; chunk scan with the carry exchange
    xc, xcp = ops.merge_runs(x_recv, rx)
    yc, ycp = ops.merge_runs(yb_recv[:, 0].contiguous(), ry)
    bc = ops.gather(yb_recv[:, 1].contiguous(), ycp)

    def gather_aggs(agg):
        return comm.all_gather(agg), rank

    u_sorted = ops.chunk(xc, yc, bc, z_prev if has_prev else 0.0, has_prev, delta, soe_args, ne,
                         gather_aggs)
    del keep

    # 5. back to the owners: received order, inverse exchange, original order
    u_recv = ops.scatter(u_sorted, xcp)
    back = comm.all_to_all(u_recv, rx, sx)
    return ops.scatter(back, xp)
