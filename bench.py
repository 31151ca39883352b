#!/usr/bin/env python3
"""Benchmark of the SOE fast Gauss transform hot path (BASELINE.json metric).

Workload (BASELINE.json configs[2], the config the metric is quoted on, fits one
GPU): N = M = 1e8 targets/sources, i.i.d. uniform on [0,1] from the reference
counter RNG (seed 0; streams 3 targets / 0 sources / 1 strengths,
proj/include/fgt1d/rng.hpp:28-31), pre-sorted, alpha = 2u-1 index-aligned with
the sorted sources (proj/tools/fgt1d_cli.cpp:232-239), tol 1e-10 -> n_e = 6,
delta = 1e-3 (the middle of the {1e-1, 1e-3, 1e-5} sweep; the others are
reported in "delta_sweep").

One step = one complete transform through the C ABI on device-resident inputs:
fgt_plan_create (finite / sorted / same-points checks, merge-path tile
partition) + fgt_apply_general (K1 tile aggregates, K2 carry scan, K3 main
pass with fused weighted real-part combine) + plan destroy.  Metric:
(M+N) points/s over the whole job.  Under torchrun (N>1) the merged stream is
split into contiguous chunks of equal element count (merge path); each rank
runs the two-phase chunk API with one NCCL all_gather of the chunk aggregates
(3 n_e complex per rank) between the phases, all on the device
(FGT_DEVICE_AGGS, fgt_chunk_carries_device).

"e2e" is the same transform from pinned HOST buffers through the one-shot
fgt_transform_host (N=1: uploads / downloads overlapped with the device
work) or the chunk API with host buffers (N>1), copies inside the timed
region.  "roofline" is K3 (the dominant kernel) against HBM at 16 B per
merged point; "cpu_baseline" times the reference library (oracle/_ref) on a
bounded sample.

  python bench.py [--gpus N --steps K --warmup W]        # our arm
  python bench.py --impl reference [...]                  # reference CPU arm
  --check        (N>1) compare the ranks' potentials with one plan
  --chunk-path   (N=1) time the chunk path: the per-rank step of a multi-GPU run
"""
import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PD = ctypes.POINTER(ctypes.c_double)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", "--size", dest="n", type=float, default=1e8,
                    help="targets = sources per transform (--size under torchrun)")
    ap.add_argument("--delta", type=float, default=1e-3)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-sample", type=float, default=1e7,
                    help="N = M of the bounded CPU sample (reference / cpu_baseline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--chunk-path", action="store_true",
                    help="N=1: run the multi-GPU chunk path (plan_create_chunk, device "
                         "aggregate exchange, finish) instead of one plan: the per-rank "
                         "step of a multi-GPU run at this per-rank size")
    ap.add_argument("--config", type=int, default=3, choices=[2, 3, 4, 5],
                    help="BASELINE.json config: 3 (default, the headline line) or the "
                         "single-GPU runs of cfg 2 (unsorted: sort-bound), 4 (clustered, "
                         "unsorted) and 5 (4096 batched transforms, one line per tol)")
    ap.add_argument("--cfg5-transforms", type=int, default=4096,
                    help="--config 5: number of transforms B (BASELINE: 4096)")
    ap.add_argument("--cfg5-size", type=int, default=65536,
                    help="--config 5: targets = sources per transform (BASELINE: 65536)")
    ap.add_argument("--tols", default="1e-3,1e-6,1e-10", help="--config 5 tolerances")
    ap.add_argument("--check", action="store_true",
                    help="N>1 (or --chunk-path): rank 0 also runs the whole transform as one "
                         "plan and reports max|u_ranks - u_single| / sum|alpha| "
                         "(multi_rank_check)")
    return ap.parse_args()


METRIC = "(M+N) points/sec at tol 1e-10 fp64; % of HBM/FP64 roofline at 1/2/4/8 GPUs"
UNIT = "points/s"


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def cpu_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model


def ne_for_tolerance(tol):
    """SURVEY 8(a13) / README.md:184-189: the fewest preset modes whose
    documented transform error is <= tol (kept here so the reference arm
    never loads the product library)."""
    for ne, t in ((3, 1e-3), (4, 1e-6), (5, 1e-8), (6, 1e-10), (7, 1e-11)):
        if tol >= t:
            return ne
    raise ValueError("tolerance below the reach of the CF tables")


def workload_config(n, delta, tol):
    """The workload both arms report (identical dicts: same_config)."""
    ne = ne_for_tolerance(tol)
    return {"workload": f"cfg3: N=M={n:.0e} presorted uniform [0,1], alpha=2u-1, "
                        f"delta={delta:g}, tol={tol:g} (n_e={ne})",
            "n_e": ne, "delta": delta, "M": n, "N": n,
            "l2": "inputs (3.2 GB) >> 126 MB L2; no flush needed"}


def reference_inputs(n, seed):
    """cfg3 inputs from the reference library's own generator
    (rng::uniform_points, rng.cpp:24-29): sorted targets (stream 3), sorted
    sources (stream 0), alpha = 2u-1 index-aligned with the sorted sources
    (stream 1), as run_bench_once with --presort (fgt1d_cli.cpp:228-239)."""
    import oracle
    x = np.sort(oracle.ref_uniform_points(n, seed, 3))
    y = np.sort(oracle.ref_uniform_points(n, seed, 0))
    a = 2.0 * oracle.ref_uniform_points(n, seed, 1) - 1.0
    return x, y, a


def reference_sample(args, threads, n=None, data=None):
    """One run of the reference's own CPU path (oracle/_ref = the reference's
    transform.cpp compiled unmodified; the C restatement if it was not built):
    plan -> precompute_gap_table -> apply_general, phases timed like
    proj/tools/fgt1d_cli.cpp:240-251."""
    import oracle
    n = int(args.cpu_sample) if n is None else int(n)
    ne = ne_for_tolerance(args.tol)
    x, y, a = data if data is not None else reference_inputs(n, args.seed)
    if oracle.ref_available():
        t0 = time.perf_counter()
        _u, (t_sort, t_pre, t_rem) = oracle.ref_transform(x, y, a, args.delta, ne=ne, mode=0,
                                                           threads=threads, precompute=True)
        total = time.perf_counter() - t0
        kind = "reference"
    else:
        t0 = time.perf_counter()
        oracle.transform(x, y, a, args.delta, ne=ne, mode=0, threads=threads)
        total = time.perf_counter() - t0
        t_sort = t_pre = t_rem = float("nan")
        kind = "port"
    return dict(value=2.0 * n / total, t_total=total, t_sort=t_sort, t_pre=t_pre, t_rem=t_rem,
                kind=kind, n=n, ne=ne)


def run_reference(args):
    """--impl reference: the reference's CPU transform on the SAME workload as
    our arm (N = M = args.n, default 1e8), rank 0 only.  Its only parallelism
    is one thread per folded mode (transform.cpp:167-168), so threads =
    min(n_e, nproc).  Warm-up runs use a 1e6-point sample of the workload
    (they only page in code and allocator state; a full-size warm-up would
    add ~30 s each); every timed step is the full workload."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    ne = ne_for_tolerance(args.tol)
    threads = max(1, min(ne, os.cpu_count() or 1))
    n = int(args.n)
    warm_n = min(n, 1_000_000)
    warm = reference_inputs(warm_n, args.seed)
    for _ in range(args.warmup):
        reference_sample(args, threads, n=warm_n, data=warm)
    del warm
    data = reference_inputs(n, args.seed)
    res, totals = None, []
    phases = np.zeros(3)
    t_all = time.perf_counter()
    for _ in range(args.steps):
        res = reference_sample(args, threads, n=n, data=data)
        totals.append(res["t_total"])
        phases += np.array([res["t_sort"], res["t_pre"], res["t_rem"]])
    wall = time.perf_counter() - t_all
    ms = 1e3 * float(np.mean(totals))
    value = 2.0 * n / (ms / 1e3)
    ph = phases / max(args.steps, 1)
    sample = (f"the whole workload every step: N=M={n} presorted uniform (seed {args.seed}), "
              f"delta={args.delta}, n_e={ne}: plan + precompute_gap_table + apply_general, "
              f"threads={threads} (mode parallelism, transform.cpp:167-168); "
              f"warm-up runs on N=M={warm_n}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference counter RNG rng::uniform_points)",
        "config": workload_config(n, args.delta, args.tol),
        "parallelism": f"reference CPU path, {threads} threads",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": res["kind"],
                         "sample": sample, "cpu": cpu_info(), "nproc": os.cpu_count(),
                         "t_sort": ph[0], "t_pre": ph[1], "t_rem": ph[2]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    polled every 2 ms (pynvml), nvidia-smi -lms as the fallback."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index, pci_bus_id=None):
        self.index = index
        self.pci = pci_bus_id
        self.proc = None
        self.lines = []
        self.nv = None
        self.samples = []
        self.stop_flag = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        if self.pci:
            try:
                return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(self.pci)
            except Exception:
                pass
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def start(self):
        try:
            self.nv, self.h = self._nvml_handle()
            self.max_mhz = float(self.nv.nvmlDeviceGetMaxClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _poll(self):
        nv, h = self.nv, self.h
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_flag.is_set():
            try:
                self.samples.append((time.perf_counter(),
                                     float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                     int(get_reasons(h))))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self, window=None):
        """window: (t0, t1) perf_counter bounds of the timed region; NVML
        samples outside it are dropped."""
        if self.nv is not None:
            self.stop_flag.set()
            self.thread.join(timeout=2)
            smp = self.samples
            if window is not None:
                inside = [x for x in smp if window[0] <= x[0] <= window[1]]
                smp = inside or smp[-1:]
            reasons = set()
            for _, _, bits in smp:
                for b, nm in self.REASONS.items():
                    if bits & b:
                        reasons.add(nm)
            sm = [c for _, c, _ in smp]
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


def link_bandwidth(dev, stream, nbytes=512 << 20, reps=3):
    """Pinned host <-> device copy bandwidth (GB/s), best of reps, CUDA events."""
    import torch
    h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
    d = torch.empty(nbytes // 8, dtype=torch.float64, device=dev)
    out = {}
    for name, (dst, src) in (("h2d_gbs", (d, h)), ("d2h_gbs", (h, d))):
        best = None
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dst.copy_(src, non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out[name] = nbytes / (best / 1e3) / 1e9
    del h, d
    return out


# ------------------------------------------------------------------ main arm

def merge_split(x, y, diag):
    """Targets among the first `diag` merged elements (sources first on ties)."""
    lo, hi = max(0, diag - y.size), min(diag, x.size)
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if x[mid - 1] < y[diag - mid]:
            lo = mid
        else:
            hi = mid - 1
    return lo


def run_other_config(args):
    """--config 2 / 4 / 5: the other BASELINE configs on one GPU with the same
    timing rules (device-resident inputs > L2, W warm-ups, K timed steps
    between CUDA events on the launching stream).  One line per config (per
    tolerance for cfg 5) with the bench keys plus plan / apply breakdown:
    for the unsorted configs the plan time is the device sort."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bench_configs as bc

    def emit(txt):
        d = json.loads(txt)
        line = {"metric": METRIC, "value": d["value"], "unit": UNIT, "n_gpus": d.get("n_gpus", 1),
                "steps": d["steps"], "warmup": d["warmup"], "ms_per_step": d["ms_per_step"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (reference counter RNG)",
                "config": {k: d[k] for k in d if k not in ("value", "steps", "warmup",
                                                             "ms_per_step", "metric", "n_gpus",
                                                             "multi_rank_check")},
                "plan_ms": d["plan_ms"], "apply_ms": d["apply_ms"]}
        if "multi_rank_check" in d:
            line["multi_rank_check"] = d["multi_rank_check"]
        print(json.dumps(line), flush=True)
    bc.EMIT = emit
    if args.config == 2:
        bc.cfg2(args.steps, args.warmup)
    elif args.config == 4:
        bc.cfg4(args.steps, args.warmup)
    else:
        bc.cfg5(args.steps, args.warmup, B=args.cfg5_transforms, n=args.cfg5_size,
                tols=tuple(float(t) for t in args.tols.split(",")), check=args.check)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config != 3:
        run_other_config(args)
        return
    import torch
    import torch.distributed as dist

    from paper_1909_09825_b200 import _capi
    from paper_1909_09825_b200.soe import soe_for_tolerance

    rank, world, local = env_rank()
    # FGT_BENCH_BACKEND=gloo is a test hook: several ranks may then share one
    # GPU (the multi-rank code path runs; its timings mean nothing)
    backend = os.environ.get("FGT_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # a process group also at world 1 when FGT_BENCH_FORCE_PG is set (test hook:
    # the collectives of the multi-rank path then run over NCCL on one GPU)
    pg = world > 1 or bool(os.environ.get("FGT_BENCH_FORCE_PG"))
    if pg:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def gather_aggs(t):
        """all_gather of this rank's chunk aggregates (device tensor)."""
        if backend == "nccl":
            out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t)
            return out.cpu().numpy()
        parts = [torch.empty_like(t.cpu()) for _ in range(world)]
        dist.all_gather(parts, t.cpu())
        return torch.cat(parts).numpy()

    def reduce_max(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    L = _capi.lib()
    stream = torch.cuda.current_stream()
    sh = ctypes.c_void_p(stream.cuda_stream)

    n = int(args.n)
    ne_soe = soe_for_tolerance(args.tol)
    ne = len(ne_soe)
    tr, ti, wr, wi, sc = ne_soe.arrays()
    soe_ptrs = (tr.ctypes.data_as(PD), ti.ctypes.data_as(PD), wr.ctypes.data_as(PD),
                wi.ctypes.data_as(PD), sc.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), ne, 1)

    # ---- synthetic data on the device (untimed): RNG + our radix sort
    def gen_sorted(stream_id):
        raw = torch.empty(n, dtype=torch.float64, device=dev)
        _capi.check(L.fgt_uniform_points_device(raw.data_ptr(), n, args.seed, stream_id, 0, sh))
        out = torch.empty_like(raw)
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        _capi.check(L.fgt_sort_device(raw.data_ptr(), n, out.data_ptr(), perm.data_ptr(), sh))
        del raw, perm
        return out

    x = gen_sorted(3)
    y = gen_sorted(0)
    a = torch.empty(n, dtype=torch.float64, device=dev)
    _capi.check(L.fgt_uniform_points_device(a.data_ptr(), n, args.seed, 1, 0, sh))
    a.mul_(2.0).sub_(1.0)
    torch.cuda.synchronize()

    # ---- this rank's contiguous chunk of the merged stream
    if world > 1:
        xh, yh = x.cpu().numpy(), y.cpu().numpy()
        tot = 2 * n
        d0, d1 = tot * rank // world, tot * (rank + 1) // world
        i0, i1 = merge_split(xh, yh, d0), merge_split(xh, yh, d1)
        j0, j1 = d0 - i0, d1 - i1
        has_prev = d0 > 0
        z_prev = max(xh[i0 - 1] if i0 > 0 else -np.inf, yh[j0 - 1] if j0 > 0 else -np.inf) \
            if has_prev else 0.0
        del xh, yh
    else:
        i0, i1, j0, j1, has_prev, z_prev = 0, n, 0, n, False, 0.0
    xc, yc, ac = x[i0:i1], y[j0:j1], a[j0:j1]
    Mc, Nc = i1 - i0, j1 - j0
    u = torch.empty(max(Mc, 1), dtype=torch.float64, device=dev)
    flags = _capi.FGT_DEVICE_PTRS | _capi.FGT_BORROW
    # device buffers of the multi-rank exchange (6 n_e doubles per rank)
    agg_dev = torch.empty(6 * ne, dtype=torch.float64, device=dev)
    allagg_dev = torch.empty(world * 6 * ne, dtype=torch.float64, device=dev)
    car_dev = torch.empty(4 * ne, dtype=torch.float64, device=dev)

    def gather_dev(t, out):
        """all_gather of this rank's device aggregates into `out` (device)."""
        if not pg:
            out.copy_(t)
        elif backend == "nccl":
            dist.all_gather_into_tensor(out, t)
        else:
            parts = [torch.empty_like(t.cpu()) for _ in range(world)]
            dist.all_gather(parts, t.cpu())
            out.copy_(torch.cat(parts))

    def one_step(delta):
        h = ctypes.c_void_p()
        if world == 1 and not args.chunk_path:
            _capi.check(L.fgt_plan_create(ctypes.cast(xc.data_ptr(), PD), Mc,
                                          ctypes.cast(yc.data_ptr(), PD), Nc, delta, *soe_ptrs,
                                          flags, local, sh, ctypes.byref(h)))
            _capi.check(L.fgt_apply_general(h, ctypes.cast(ac.data_ptr(), PD), Nc,
                                            ctypes.cast(u.data_ptr(), PD), 1, flags, sh))
        else:
            _capi.check(L.fgt_plan_create_chunk(ctypes.cast(xc.data_ptr(), PD), Mc,
                                                ctypes.cast(yc.data_ptr(), PD), Nc, float(z_prev),
                                                int(has_prev), delta, *soe_ptrs, flags, local, sh,
                                                ctypes.byref(h)))
            # device-side exchange: aggregates -> all_gather -> this chunk's
            # carries, all stream-ordered (no host round trip in the step)
            fd = flags | _capi.FGT_DEVICE_AGGS
            _capi.check(L.fgt_apply_chunk_aggregate(h, ctypes.cast(ac.data_ptr(), PD),
                                                    ctypes.cast(agg_dev.data_ptr(), PD), fd, sh))
            gather_dev(agg_dev, allagg_dev)
            _capi.check(L.fgt_chunk_carries_device(ctypes.c_void_p(allagg_dev.data_ptr()), world,
                                                   ne, rank, ctypes.c_void_p(car_dev.data_ptr()),
                                                   sh))
            _capi.check(L.fgt_apply_chunk_finish(h, ctypes.cast(ac.data_ptr(), PD),
                                                 ctypes.cast(car_dev.data_ptr(), PD),
                                                 ctypes.cast(u.data_ptr(), PD), fd, sh))
        L.fgt_plan_destroy(h)

    def barrier():
        if pg:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    def timed(steps, delta):
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            one_step(delta)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1) / steps
        if pg:
            ms = reduce_max(ms)
        return ms

    for _ in range(max(args.warmup, 0)):
        one_step(args.delta)
    torch.cuda.synchronize()

    try:
        pr = torch.cuda.get_device_properties(dev)
        pci = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
    except Exception:
        pci = None
    clocks = ClockSampler(local, pci)
    clocks.start()
    time.sleep(0.3)
    launches0 = L.fgt_launch_counter()
    tw0 = time.perf_counter()
    ms = timed(args.steps, args.delta)
    tw1 = time.perf_counter()
    launches = L.fgt_launch_counter() - launches0
    clk = clocks.stop((tw0, tw1))
    value = 2.0 * n / (ms / 1e3)

    # ---- multi-rank correctness: the ranks' chunk potentials vs one plan
    mr_check = None
    if args.check and (world > 1 or args.chunk_path):
        def allgather_cpu(t):
            """all_gather of equal-size CPU tensors over either backend."""
            if not pg:
                return [t]
            src = t.to(dev) if backend == "nccl" else t
            parts = [torch.zeros_like(src) for _ in range(world)]
            dist.all_gather(parts, src)
            return [p_.cpu() for p_ in parts]
        one_step(args.delta)
        torch.cuda.synchronize()
        cnts = allgather_cpu(torch.tensor([Mc], dtype=torch.int64))
        mx = int(max(c.item() for c in cnts))
        buf = torch.zeros(mx, dtype=torch.float64)
        buf[:Mc] = u[:Mc].cpu()
        parts = allgather_cpu(buf)
        if rank == 0:
            u_ranks = torch.cat([parts[r][:int(cnts[r].item())] for r in range(world)])
            h = ctypes.c_void_p()
            u_one = torch.empty(n, dtype=torch.float64, device=dev)
            _capi.check(L.fgt_plan_create(ctypes.cast(x.data_ptr(), PD), n,
                                          ctypes.cast(y.data_ptr(), PD), n, args.delta, *soe_ptrs,
                                          flags, local, sh, ctypes.byref(h)))
            _capi.check(L.fgt_apply_general(h, ctypes.cast(a.data_ptr(), PD), n,
                                            ctypes.cast(u_one.data_ptr(), PD), 1, flags, sh))
            L.fgt_plan_destroy(h)
            torch.cuda.synchronize()
            err = float((u_ranks - u_one.cpu()).abs().max() / a.abs().sum().cpu())
            mr_check = {"max_abs_diff_over_sum_abs_alpha": err, "pass": err <= 1e-12,
                        "reference": "one plan over the whole stream on rank 0's GPU"}

    # ---- per-kernel durations (CUDA events on the launching stream)
    L.fgt_profile_enable(1)
    L.fgt_profile_read(None, None, 3)
    prof_steps = 3
    for _ in range(prof_steps):
        one_step(args.delta)
    torch.cuda.synchronize()
    kms = np.zeros(3)
    kcnt = (ctypes.c_longlong * 3)()
    L.fgt_profile_read(kms.ctypes.data_as(PD), kcnt, 3)
    L.fgt_profile_enable(0)
    kavg = [kms[i] / prof_steps for i in range(3)]  # per step (K2 runs twice with chunks)
    apply_ms = sum(kavg)

    # ---- FP64 peak (measured) and roofline
    peak = ctypes.c_double()
    pms = ctypes.c_double()
    _capi.check(L.fgt_fp64_peak(ctypes.byref(peak), ctypes.byref(pms)))
    Mt = Nt = float(n)
    pts_rank = float(Mc + Nc)
    # W = n_e (48 + 4 M/(M+N)) fp64-pipe instructions per point
    W = ne * (48.0 + 4.0 * Mt / (Mt + Nt))
    alg_tflop = 2.0 * W * pts_rank / 1e12  # every fp64-pipe instruction counted as FMA-2
    achieved_fp64 = alg_tflop / (apply_ms / 1e3) if apply_ms > 0 else None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
        hbm_peak, hbm_src = float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        hbm_peak, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    hbm_bytes = 16.0 * pts_rank
    achieved_hbm = hbm_bytes / (apply_ms / 1e3) / 1e9 if apply_ms > 0 else None
    achieved_k3 = hbm_bytes / (kavg[2] / 1e3) / 1e9 if kavg[2] > 0 else None

    # ---- delta sweep (cfg3 lists {1e-1, 1e-3, 1e-5})
    sweep = {}
    if not args.no_sweep:
        for d in (1e-1, 1e-3, 1e-5):
            one_step(d)
            sm = timed(max(2, args.steps // 3), d)
            sweep[f"{d:g}"] = {"ms_per_step": sm, "value": 2.0 * n / (sm / 1e3)}

    # ---- e2e through the public API with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        hx = xc.cpu().pin_memory()
        hy = yc.cpu().pin_memory()
        ha = ac.cpu().pin_memory()
        hu = torch.empty(max(Mc, 1), dtype=torch.float64).pin_memory()

        def e2e_step():
            h = ctypes.c_void_p()
            if world == 1:
                # one-shot host-buffer entry: uploads / downloads overlapped
                # with the device work (fgt_transform_host)
                _capi.check(L.fgt_transform_host(ctypes.cast(hx.data_ptr(), PD), Mc,
                                                 ctypes.cast(hy.data_ptr(), PD), Nc,
                                                 ctypes.cast(ha.data_ptr(), PD), args.delta,
                                                 *soe_ptrs[:-1], 1, ctypes.cast(hu.data_ptr(), PD),
                                                 local, sh))
                return
            else:
                _capi.check(L.fgt_plan_create_chunk(ctypes.cast(hx.data_ptr(), PD), Mc,
                                                    ctypes.cast(hy.data_ptr(), PD), Nc,
                                                    float(z_prev), int(has_prev), args.delta,
                                                    *soe_ptrs, 0, local, sh, ctypes.byref(h)))
                agg = np.empty(6 * ne)
                _capi.check(L.fgt_apply_chunk_aggregate(h, ctypes.cast(ha.data_ptr(), PD),
                                                        agg.ctypes.data_as(PD), 0, sh))
                allagg = gather_aggs(torch.from_numpy(agg).to(dev))
                carries = np.empty(world * 4 * ne)
                _capi.check(L.fgt_chunk_carries(allagg.ctypes.data_as(PD), world, ne,
                                                carries.ctypes.data_as(PD)))
                mine = np.ascontiguousarray(carries[rank * 4 * ne:(rank + 1) * 4 * ne])
                _capi.check(L.fgt_apply_chunk_finish(h, ctypes.cast(ha.data_ptr(), PD),
                                                     mine.ctypes.data_as(PD),
                                                     ctypes.cast(hu.data_ptr(), PD), 0, sh))
            L.fgt_plan_destroy(h)

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        barrier()
        es = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            es = reduce_max(es)
        # cross-check: e2e potentials equal the device-path potentials
        one_step(args.delta)
        torch.cuda.synchronize()
        diff = float((hu[:Mc] - u[:Mc].cpu()).abs().max() / ac.abs().sum().cpu()) if Mc > 0 else 0.0
        e2e = {"value": 2.0 * n / es, "unit": UNIT, "ms_per_step": es * 1e3,
               "h2d_bytes_per_step": int(8 * (Mc + 2 * Nc)) * world,
               "d2h_bytes_per_step": int(8 * Mc) * world,
               "api": "fgt_transform_host (pipelined host-buffer transform)" if world == 1
               else "fgt_plan_create_chunk + fgt_apply_chunk_aggregate/finish (host buffers)",
               "max_diff_vs_device_path": diff, "matches_device_path": diff <= 1e-12}
        # the host link bounds e2e: measured pinned copy bandwidth per direction,
        # floor = this rank's h2d / BW_h2d + d2h / BW_d2h (the API is synchronous)
        bw = link_bandwidth(dev, stream)
        floor_seq = 8 * (Mc + 2 * Nc) / bw["h2d_gbs"] / 1e9 + 8 * Mc / bw["d2h_gbs"] / 1e9
        # full duplex: the download can hide behind the upload; the upload
        # of every input byte is the floor of any host-buffer transform
        floor = 8 * (Mc + 2 * Nc) / bw["h2d_gbs"] / 1e9
        e2e["link"] = {**bw, "floor_ms": floor * 1e3, "frac": floor / es,
                       "sequential_floor_ms": floor_seq * 1e3,
                       "note": "e2e time vs the host-link floor: upload of x, y, alpha at the "
                               "measured pinned H2D bandwidth (the download overlaps it)"}

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = max(1, min(ne, os.cpu_count() or 1))
        r = reference_sample(args, threads)
        cpu = {"value": r["value"], "unit": UNIT, "cores": threads, "kind": r["kind"],
               "sample": (f"N=M={r['n']} presorted uniform, delta={args.delta}, n_e={ne}: "
                          f"reference plan + precompute_gap_table + apply_general, "
                          f"threads={threads}; t_sort/t_pre/t_rem = "
                          f"{r['t_sort']:.3f}/{r['t_pre']:.3f}/{r['t_rem']:.3f} s"),
               "cpu": cpu_info(), "nproc": os.cpu_count()}

    # DRAM traffic of one apply from the committed ncu --set full capture
    # (dram__bytes_read.sum + dram__bytes_write.sum over its launches)
    traffic = {}
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    if n == int(1e8) and world == 1 and os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference counter RNG, seed 0; sorted on device by our radix sort)",
            "config": workload_config(n, args.delta, args.tol),
            "parallelism": (f"merged-stream chunks x{world}" if world > 1 else
                            "1 GPU (chunk path)" if args.chunk_path else "1 GPU"),
            # dominant kernel: K3 (main pass) -- reads x, y, alpha and writes u,
            # 16 B per merged point, timed by CUDA events on the launching stream
            "roofline": {"bound": "hbm", "achieved": achieved_k3, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved_k3 / hbm_peak if achieved_k3 else None,
                         "traffic": traffic.get("k3_dram_bytes_per_launch"),
                         "traffic_source": "profiles/traffic.json (ncu --set full of K3: "
                                           "dram__bytes_read.sum + dram__bytes_write.sum)",
                         "kernel": "K3c k3c_kernel (collapsed narrow main pass, CTA-chunked): one launch per apply",
                         "bytes_per_launch": 16.0 * pts_rank, "bytes_per_point": 16,
                         "launch_ms": kavg[2], "peak_source": hbm_src},
            "roofline_apply": {"bound": "hbm", "achieved": achieved_hbm, "peak": hbm_peak,
                               "unit": "GB/s", "frac": achieved_hbm / hbm_peak if achieved_hbm else None,
                               "bytes_per_point": 16,
                               "kernel": "apply = K1c (moments) + K2 (top, down) + K3c",
                               "traffic": traffic.get("dram_bytes_per_apply"),
                               "peak_source": hbm_src},
            # the whole step (plan included): 16 B per point over the step time
            "roofline_step": {"bound": "hbm", "achieved": hbm_bytes / (ms / 1e3) / 1e9,
                              "peak": hbm_peak, "unit": "GB/s",
                              "frac": hbm_bytes / (ms / 1e3) / 1e9 / hbm_peak,
                              "bytes_per_point": 16, "kernel": "plan + apply (+ destroy)",
                              "traffic": traffic.get("dram_bytes_per_step"),
                              "peak_source": hbm_src},
            # SURVEY 8(d)'s FP64 model of the exp-per-gap algorithm (W = 300 fp64
            # instr/pt at n_e = 6); the collapsed moment form does far less
            # FP64 work, so frac > 1 here means "faster than that algorithm's
            # FP64 roofline", not a counter reading
            "roofline_fp64_survey": {"bound": "fp64", "achieved": achieved_fp64, "peak": peak.value,
                                     "unit": "TFLOP/s",
                                     "frac": (achieved_fp64 / peak.value) if achieved_fp64 else None,
                                     "work": f"SURVEY 8(d) W = n_e(48 + 4M/(M+N)) = {W:.0f} "
                                             "fp64-pipe instr/pt, counted as FMA-2 flops",
                                     "peak_source": "measured on this GPU (fgt_fp64_peak DFMA probe)"},
            # kind 0: wide-segment K1 (none on cfg 3); kind 1: K1c moments + block
            # aggregates, K2 top, K2m down-sweep; kind 2: K3c (+ wide K3)
            "kernels_ms": {"K1_wide": kavg[0], "K1b_K2_moment_scan": kavg[1], "K3_main": kavg[2],
                           "apply_total": apply_ms, "plan_and_other": ms - apply_ms},
            "apply_value": 2.0 * n / (apply_ms / 1e3) if apply_ms > 0 else None,
            "gpu_launches": int(launches),
            "clocks": clk,
            "delta_sweep": sweep,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if mr_check is not None:
            line["multi_rank_check"] = mr_check
        print(json.dumps(line), flush=True)
    if pg:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
