#!/usr/bin/env python3
"""Measurements of the other BASELINE.json configs on one GPU (the headline
cfg 3 line is bench.py).  Same timing rules: device-resident inputs, W warm-up
steps, K timed steps between CUDA events on the launching stream, inputs
larger than L2.  One step = plan (checks, device sort when unsorted,
partition, segment metadata) + apply + destroy.

  cfg2: N=M=1e7 uniform, UNSORTED, alpha ~ N(0,1) (Box-Muller, streams 1/4),
        delta=1e-4, tol 1e-6 -> n_e=4
  cfg4: M=2^25 / N=2^27 16-component mixture (sigma 1e-3; SURVEY 8(d) recipe),
        unsorted, alpha ~ U[0,1), delta=1e-6, tol 1e-8 -> n_e=5  (1 GPU; the
        8-GPU partition needs 8 GPUs)
  cfg5: 4096 transforms of N=M=65536, presorted uniform, alpha=2u-1,
        delta_b log-uniform in [1e-6, 1e-1] (stream 9), tol in {1e-3, 1e-6, 1e-10};
        under torchrun the transforms are split over the ranks

Prints one JSON line per config.
"""
import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1909_09825_b200 import _capi  # noqa: E402
from paper_1909_09825_b200.soe import soe_for_tolerance  # noqa: E402
from paper_1909_09825_b200.transform import uniform_points_array as up  # noqa: E402

PD = ctypes.POINTER(ctypes.c_double)
PI64 = ctypes.POINTER(ctypes.c_int64)
L = _capi.lib()
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count()))
torch.cuda.set_device(dev)
stream = torch.cuda.current_stream()
sh = ctypes.c_void_p(stream.cuda_stream)


def soe_args(tol):
    soe = soe_for_tolerance(tol)
    tr, ti, wr, wi, sc = soe.arrays()
    keep = (tr, ti, wr, wi, sc)
    return keep, (tr.ctypes.data_as(PD), ti.ctypes.data_as(PD), wr.ctypes.data_as(PD),
                  wi.ctypes.data_as(PD), sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                  len(soe), 1)


def normal(n, seed, s1, s2):
    u1, u2 = up(n, seed, s1), up(n, seed, s2)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def timed(step, steps, warmup):
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def kernel_ms(fn, reps=3):
    """Average K1/K2/K3 durations (profiling events on the launching stream)."""
    L.fgt_profile_enable(1)
    L.fgt_profile_read(None, None, 3)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    kms = np.zeros(3)
    kcnt = (ctypes.c_longlong * 3)()
    L.fgt_profile_read(kms.ctypes.data_as(PD), kcnt, 3)
    L.fgt_profile_enable(0)
    return {k: kms[i] / max(1, kcnt[i]) for i, k in enumerate(("K1", "K2", "K3"))}


EMIT = print  # bench.py --config replaces this to add the bench-contract keys


def single_config(name, x, y, a, delta, tol, steps, warmup, extra):
    keep, sp = soe_args(tol)
    M, N = x.numel(), y.numel()
    u = torch.empty(M, dtype=torch.float64, device=dev)
    fl = _capi.FGT_DEVICE_PTRS
    h = [None]

    def plan():
        hh = ctypes.c_void_p()
        _capi.check(L.fgt_plan_create(ctypes.cast(x.data_ptr(), PD), M, ctypes.cast(y.data_ptr(), PD),
                                      N, delta, *sp, fl, 0, sh, ctypes.byref(hh)))
        return hh

    def apply(hh):
        _capi.check(L.fgt_apply_general(hh, ctypes.cast(a.data_ptr(), PD), N,
                                        ctypes.cast(u.data_ptr(), PD), 1, fl, sh))

    def step():
        hh = plan()
        apply(hh)
        L.fgt_plan_destroy(hh)

    ms = timed(step, steps, warmup)
    hh = plan()
    ms_apply = timed(lambda: apply(hh), steps, warmup)
    kms = kernel_ms(lambda: apply(hh))
    L.fgt_plan_destroy(hh)
    line = {"kernels_ms": kms, "config": name, "metric": "(M+N) points/s", "value": (M + N) / (ms / 1e3),
            "ms_per_step": ms, "apply_ms": ms_apply,
            "apply_value": (M + N) / (ms_apply / 1e3), "plan_ms": ms - ms_apply,
            "M": M, "N": N, "delta": delta, "tol": tol, "n_e": len(keep[0]), "steps": steps,
            "warmup": warmup, **extra}
    EMIT(json.dumps(line))


def cfg2(steps, warmup):
    n = 10_000_000
    x = torch.from_numpy(up(n, 0, 3)).to(dev)
    y = torch.from_numpy(up(n, 0, 0)).to(dev)
    a = torch.from_numpy(normal(n, 0, 1, 4)).to(dev)
    single_config("cfg2", x, y, a, 1e-4, 1e-6, steps, warmup,
                  {"data": "uniform unsorted, alpha Box-Muller normal (streams 1/4)"})


def cfg4(steps, warmup):
    M, N = 2 ** 25, 2 ** 27
    cen = up(16, 0, 5)

    def mixture(n, seed):
        comp = np.minimum(15, (16 * up(n, seed, 6)).astype(np.int64))
        return cen[comp] + 1e-3 * normal(n, seed, 7, 8)

    y = torch.from_numpy(mixture(N, 0)).to(dev)
    x = torch.from_numpy(mixture(M, 1)).to(dev)
    a = torch.from_numpy(up(N, 0, 1)).to(dev)
    single_config("cfg4 (1 GPU)", x, y, a, 1e-6, 1e-8, steps, warmup,
                  {"data": "16-component mixture sigma 1e-3, unsorted, alpha U[0,1)"})


class Ranks:
    """Process group of a multi-GPU cfg 5 run (torchrun): ranks take equal
    contiguous ranges of the B transforms (independent problems, no exchange),
    timed between a barrier and CUDA events, max over ranks."""

    def __init__(self):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.dist = None
        self.backend = os.environ.get("FGT_BENCH_BACKEND", "nccl")
        if self.world > 1:
            import torch.distributed as dist
            if not dist.is_initialized():
                if self.backend == "nccl":
                    dist.init_process_group("nccl", device_id=dev)
                else:
                    dist.init_process_group(self.backend)
            self.dist = dist

    def barrier(self):
        if self.dist is not None:
            if self.backend == "nccl":
                self.dist.barrier(device_ids=[dev.index])
            else:
                self.dist.barrier()

    def max(self, v):
        if self.dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64,
                         device=dev if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather(self, t):
        """all_gather of equal-size device tensors -> list on rank 0 (cpu)."""
        if self.dist is None:
            return [t.cpu()]
        src = t if self.backend == "nccl" else t.cpu()
        parts = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(parts, src)
        return [p.cpu() for p in parts]


def cfg5(steps, warmup, B=4096, n=65536, fixed_delta=None, tols=(1e-3, 1e-6, 1e-10),
         check=False):
    """BASELINE cfg 5: B transforms of N = M = n.  Under torchrun the
    transforms are split over the ranks (rank r: transforms
    [r B / G, (r + 1) B / G), the same data as on one GPU)."""
    rk = Ranks()
    b0, b1 = B * rk.rank // rk.world, B * (rk.rank + 1) // rk.world
    Bl = b1 - b0
    # per transform b: seed b, sorted uniform targets / sources, alpha = 2u-1
    x = torch.empty(Bl, n, dtype=torch.float64, device=dev)
    y = torch.empty(Bl, n, dtype=torch.float64, device=dev)
    a = torch.empty(Bl, n, dtype=torch.float64, device=dev)
    for i in range(Bl):
        b = b0 + i
        _capi.check(L.fgt_uniform_points_device(x[i].data_ptr(), n, b, 3, 0, sh))
        _capi.check(L.fgt_uniform_points_device(y[i].data_ptr(), n, b, 0, 0, sh))
        _capi.check(L.fgt_uniform_points_device(a[i].data_ptr(), n, b, 1, 0, sh))
    x = torch.sort(x, dim=1).values.contiguous()
    y = torch.sort(y, dim=1).values.contiguous()
    a.mul_(2.0).sub_(1.0)
    deltas_all = 10.0 ** (-6.0 + 5.0 * up(B, 0, 9))
    dlabel = "log-uniform [1e-6, 1e-1] (stream 9)"
    if fixed_delta is not None:
        deltas_all = np.full(B, fixed_delta)
        dlabel = "all %g" % fixed_delta
    deltas = np.ascontiguousarray(deltas_all[b0:b1])
    off = np.arange(Bl + 1, dtype=np.int64) * n
    u = torch.empty(Bl * n, dtype=torch.float64, device=dev)
    fl = _capi.FGT_DEVICE_PTRS | _capi.FGT_BORROW
    for tol in tols:
        keep, sp = soe_args(tol)

        def plan():
            hh = ctypes.c_void_p()
            _capi.check(L.fgt_batch_create(Bl, ctypes.cast(x.data_ptr(), PD), off.ctypes.data_as(PI64),
                                           ctypes.cast(y.data_ptr(), PD), off.ctypes.data_as(PI64),
                                           deltas.ctypes.data_as(PD), *sp, fl, dev.index, sh,
                                           ctypes.byref(hh)))
            return hh

        def apply(hh):
            _capi.check(L.fgt_apply_general(hh, ctypes.cast(a.data_ptr(), PD), Bl * n,
                                            ctypes.cast(u.data_ptr(), PD), 1, fl, sh))

        def step():
            hh = plan()
            apply(hh)
            L.fgt_plan_destroy(hh)

        def ranked(fn):
            for _ in range(warmup):
                fn()
            torch.cuda.synchronize()
            rk.barrier()
            ms = timed(fn, steps, 0)
            rk.barrier()
            return rk.max(ms)

        ms = ranked(step)
        hh = plan()
        ms_apply = ranked(lambda: apply(hh))
        kms = kernel_ms(lambda: apply(hh))
        L.fgt_plan_destroy(hh)
        extra = {}
        if check:
            # every rank's potentials vs one plan over all B transforms (rank 0)
            step()
            torch.cuda.synchronize()
            parts = rk.gather(u)
            if rk.rank == 0:
                xs = torch.empty(B, n, dtype=torch.float64, device=dev)
                ys = torch.empty(B, n, dtype=torch.float64, device=dev)
                al = torch.empty(B, n, dtype=torch.float64, device=dev)
                for b in range(B):
                    _capi.check(L.fgt_uniform_points_device(xs[b].data_ptr(), n, b, 3, 0, sh))
                    _capi.check(L.fgt_uniform_points_device(ys[b].data_ptr(), n, b, 0, 0, sh))
                    _capi.check(L.fgt_uniform_points_device(al[b].data_ptr(), n, b, 1, 0, sh))
                xs = torch.sort(xs, dim=1).values.contiguous()
                ys = torch.sort(ys, dim=1).values.contiguous()
                al.mul_(2.0).sub_(1.0)
                offa = np.arange(B + 1, dtype=np.int64) * n
                ua = torch.empty(B * n, dtype=torch.float64, device=dev)
                hh = ctypes.c_void_p()
                _capi.check(L.fgt_batch_create(B, ctypes.cast(xs.data_ptr(), PD),
                                               offa.ctypes.data_as(PI64),
                                               ctypes.cast(ys.data_ptr(), PD),
                                               offa.ctypes.data_as(PI64),
                                               deltas_all.ctypes.data_as(PD), *sp, fl, dev.index,
                                               sh, ctypes.byref(hh)))
                _capi.check(L.fgt_apply_general(hh, ctypes.cast(al.data_ptr(), PD), B * n,
                                                ctypes.cast(ua.data_ptr(), PD), 1, fl, sh))
                L.fgt_plan_destroy(hh)
                torch.cuda.synchronize()
                ur = torch.cat(parts)
                err = float((ur - ua.cpu()).abs().max() / al.abs().sum(dim=1).max().cpu())
                extra["multi_rank_check"] = {
                    "max_abs_diff_over_sum_abs_alpha_b": err, "pass": err <= 1e-12,
                    "reference": "one batched plan over all B transforms on rank 0's GPU"}
        pts = 2.0 * B * n
        if rk.rank == 0:
            EMIT(json.dumps({"config": "cfg5", "metric": "(M+N) points/s", "value": pts / (ms / 1e3),
                              "ms_per_step": ms, "apply_ms": ms_apply,
                              "apply_value": pts / (ms_apply / 1e3), "plan_ms": ms - ms_apply,
                              "transforms": B, "M_each": n, "N_each": n, "tol": tol,
                              "n_e": len(keep[0]), "kernels_ms": kms, "deltas": dlabel,
                              "n_gpus": rk.world,
                              "parallelism": (f"transforms split over {rk.world} GPUs"
                                              if rk.world > 1 else "1 GPU"),
                              "steps": steps, "warmup": warmup, **extra}))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,4,5")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--tols", default="1e-3,1e-6,1e-10", help="cfg5 tolerances")
    ap.add_argument("--cfg5-deltas", default="", help="comma list: run cfg5 with one fixed delta each")
    args = ap.parse_args()
    for d in [v for v in args.cfg5_deltas.split(",") if v]:
        cfg5(args.steps, args.warmup, fixed_delta=float(d), tols=(1e-10,))
    if args.cfg5_deltas:
        sys.exit(0)
    for c in args.configs.split(","):
        if c.strip() == "5":
            cfg5(args.steps, args.warmup, tols=tuple(float(t) for t in args.tols.split(",")))
        else:
            {"2": cfg2, "4": cfg4}[c.strip()](args.steps, args.warmup)
