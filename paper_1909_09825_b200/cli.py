"""Command-line front end with the reference CLI's transform-path subcommands
and output schema (proj/tools/fgt1d_cli.cpp), running on the GPU library:

    python -m paper_1909_09825_b200.cli bench --N 100000 --ne 4 [--json]
    python -m paper_1909_09825_b200.cli delta-sweep --N 10000 --delta 1e-3 ...
    python -m paper_1909_09825_b200.cli transform sources.csv [targets.csv] --delta 1
    python -m paper_1909_09825_b200.cli soe --n 8 [--out table.txt]

Exit codes as the reference (fgt1d_cli.cpp:577-590): 2 for invalid input
(ValueError), 1 for numerical / device failures.  `soe` serves the CF tables
only (the contour / reduction constructions are outside the transform path).

Phase mapping: t_sort = plan() (upload, checks, device sort when
unsorted, segment metadata), t_pre = 0 (the device path has no gap table),
t_rem = apply, t_total = their sum.
"""
import argparse
import json
import sys
import time

import numpy as np

from . import _capi
from .soe import cf_soe, load_coefficient_table, max_error, save_coefficient_table
from .transform import (K_STREAM_SOURCES, K_STREAM_STRENGTHS, K_STREAM_TARGETS,
                        TransformRequest, apply_general, apply_same, delta_sweep, gen_points,
                        measure_error, plan, preset_for_ne, uniform_points_array)


def _g(x):
    """C++ ostream with precision(17)."""
    return format(float(x), ".17g")


def _open_out(path):
    if not path:
        return sys.stdout
    try:
        return open(path, "w")
    except OSError:
        raise ValueError(f"cannot open for writing: {path}")


# ------------------------------------------------------------------- bench

BENCH_HEADER = ("scenario,N,M,n_e,delta,seed,dist,threads,t_sort,t_pre,t_rem,t_total,"
                "max_rel_error,throughput_full,throughput_amortized")


def run_bench_once(s, soe, cached):
    """fgt1d_cli.cpp:220-269."""
    src = gen_points(s.dist, s.M, s.seed, K_STREAM_SOURCES)
    tgt = src if s.scenario == "same" else gen_points(s.dist, s.N, s.seed, K_STREAM_TARGETS)
    a = uniform_points_array(s.M, s.seed, K_STREAM_STRENGTHS)
    if s.presort:
        src = np.sort(src)
        tgt = src if s.scenario == "same" else np.sort(tgt)
    req = TransformRequest(tgt, src, a, s.delta)
    t0 = time.perf_counter()
    p = plan(req, soe, False)
    t_sort = time.perf_counter() - t0
    t_pre = 0.0
    t2 = time.perf_counter()
    res = apply_same(p, a, s.threads) if s.scenario == "same" else apply_general(p, a, s.threads)
    t_rem = time.perf_counter() - t2
    t_total = t_sort + t_pre + t_rem
    if cached[0] < 0.0:
        cached[0] = measure_error(req, res, s.seed)
    pts = float(s.N + s.M)
    return {"scenario": "SamePoints" if s.scenario == "same" else "DistinctPoints",
            "N": s.N, "M": s.M, "n_e": s.ne, "delta": s.delta, "seed": s.seed,
            "dist": s.dist, "threads": s.threads, "t_sort": t_sort, "t_pre": t_pre,
            "t_rem": t_rem, "t_total": t_total, "max_rel_error": cached[0],
            "throughput_full": pts / t_total if t_total > 0 else 0.0,
            "throughput_amortized": pts / t_rem if t_rem > 0 else 0.0}


def bench_csv_row(r):
    return ",".join([r["scenario"], str(r["N"]), str(r["M"]), str(r["n_e"]), _g(r["delta"]),
                     str(r["seed"]), r["dist"], str(r["threads"]), _g(r["t_sort"]),
                     _g(r["t_pre"]), _g(r["t_rem"]), _g(r["t_total"]), _g(r["max_rel_error"]),
                     _g(r["throughput_full"]), _g(r["throughput_amortized"])])


def cmd_bench(s, repeat, as_json, out):
    """fgt1d_cli.cpp:292-312."""
    if s.N < 1 or s.M < 1:
        raise ValueError("--N and --M must be at least 1")
    if repeat < 1:
        raise ValueError("--repeat must be at least 1")
    if s.scenario not in ("same", "distinct"):
        raise ValueError("--scenario must be same or distinct")
    if s.scenario == "same":
        s.M = s.N
    soe = preset_for_ne(s.ne)
    cached = [-1.0]
    rows = [run_bench_once(s, soe, cached) for _ in range(repeat)]
    os_ = _open_out(out)
    if as_json:
        os_.write(json.dumps(rows, indent=2) + "\n")
    else:
        os_.write(BENCH_HEADER + "\n")
        for r in rows:
            os_.write(bench_csv_row(r) + "\n")
    return 0


# ------------------------------------------------------------- delta sweep

def cmd_delta_sweep(N, ne, deltas, seed, dist, as_json, out):
    rows = delta_sweep(N, ne, deltas, seed, dist)
    os_ = _open_out(out)
    if as_json:
        os_.write(json.dumps(rows, indent=2) + "\n")
    else:
        os_.write("delta,error\n")
        for r in rows:
            os_.write(f"{_g(r['delta'])},{_g(r['error'])}\n")
    return 0


# --------------------------------------------------------------- transform

def read_point_file(path):
    """fgt1d_cli.cpp:360-400: coordinate[,strength] per line; '#' comments;
    ',', ';' or tabs as separators; one header line tolerated."""
    try:
        f = open(path)
    except OSError:
        raise ValueError(f"cannot open for reading: {path}")
    coords, strengths = [], []
    first = True
    with f:
        for lineno, line in enumerate(f, 1):
            body = line.split("#", 1)[0]
            for ch in ",;\t":
                body = body.replace(ch, " ")
            toks = body.split()
            if not toks:
                continue
            try:
                x = float(toks[0])
                a = float(toks[1]) if len(toks) >= 2 else None
            except ValueError:
                if first:
                    first = False
                    continue
                raise ValueError(f"{path}:{lineno}: cannot parse point row '{line.rstrip()}'")
            first = False
            coords.append(x)
            if a is not None:
                strengths.append(a)
    if strengths and len(strengths) != len(coords):
        raise ValueError(f"{path}: strength column present only on some rows")
    return coords, strengths


def cmd_transform(sources, targets, delta, ne, table, threads, out):
    """fgt1d_cli.cpp:402-433."""
    src, a = read_point_file(sources)
    if not src:
        raise ValueError(f"{sources}: no source points")
    if not a:
        a = [1.0] * len(src)
    tgt = src if not targets else read_point_file(targets)[0]
    soe = load_coefficient_table(table) if table else preset_for_ne(ne)
    req = TransformRequest(tgt, src, a, delta)
    p = plan(req, soe, False)
    res = apply_same(p, a, threads) if p.same_points else apply_general(p, a, threads)
    os_ = _open_out(out)
    os_.write("index,potential\n")
    for i, v in enumerate(res):
        os_.write(f"{i},{_g(v)}\n")
    return 0


# --------------------------------------------------------------------- soe

def cmd_soe(method, n, out):
    """fgt1d_cli.cpp:70-81 for the CF tables."""
    if method != "cf":
        raise ValueError(f"method '{method}' is not available here (CF tables only)")
    soe = cf_soe(n)
    rep = max_error(soe)
    if out:
        save_coefficient_table(out, soe, "cf")
    print(f"n={rep.n} max_error={_g(rep.max_abs_error)} argmax_x={_g(rep.argmax_x)}")
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="fgt1d", description=(
        "Sum-of-exponentials Gaussian kernel approximations and the fast Gauss transform"))
    sub = ap.add_subparsers(dest="cmd", required=True)
    so = sub.add_parser("soe", help="Build one SOE, print its grid error, optionally save a table")
    so.add_argument("--method", default="cf")
    so.add_argument("--n", type=int, default=8)
    so.add_argument("--out", default="")
    b = sub.add_parser("bench", help="Run the fast transform on generated data and time its phases")
    b.add_argument("--scenario", default="same")
    b.add_argument("--N", type=int, default=100000)
    b.add_argument("--M", type=int, default=-1)
    b.add_argument("--ne", type=int, default=4)
    b.add_argument("--delta", type=float, default=1.0)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--dist", default="uniform")
    b.add_argument("--presort", action="store_true")
    b.add_argument("--threads", type=int, default=1)
    b.add_argument("--repeat", type=int, default=1)
    b.add_argument("--json", action="store_true")
    b.add_argument("--out", default="")
    d = sub.add_parser("delta-sweep", help="Transform error as a function of delta")
    d.add_argument("--N", type=int, default=10000)
    d.add_argument("--ne", type=int, default=4)
    d.add_argument("--delta", type=float, action="append", default=[])
    d.add_argument("--seed", type=int, default=0)
    d.add_argument("--dist", default="uniform")
    d.add_argument("--json", action="store_true")
    d.add_argument("--out", default="")
    t = sub.add_parser("transform", help="Apply the fast transform to points from files")
    t.add_argument("sources")
    t.add_argument("targets", nargs="?", default="")
    t.add_argument("--delta", type=float, default=1.0)
    t.add_argument("--ne", type=int, default=4)
    t.add_argument("--table", default="")
    t.add_argument("--threads", type=int, default=1)
    t.add_argument("--out", default="")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        if a.cmd == "soe":
            return cmd_soe(a.method, a.n, a.out)
        if a.cmd == "bench":
            a.M = a.M if a.M > 0 else a.N
            return cmd_bench(a, a.repeat, a.json, a.out)
        if a.cmd == "delta-sweep":
            return cmd_delta_sweep(a.N, a.ne, a.delta, a.seed, a.dist, a.json, a.out)
        if a.cmd == "transform":
            return cmd_transform(a.sources, a.targets, a.delta, a.ne, a.table, a.threads, a.out)
    except _capi.NumericalError as e:
        print(f"numerical failure: {e}", file=sys.stderr)
        return 1
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # device failures and the like
        print(f"failure: {e}", file=sys.stderr)
        return 1
    return 2


if __name__ == "__main__":
    sys.exit(main())
