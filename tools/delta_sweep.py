#!/usr/bin/env python3
"""delta-sweep (the reference CLI's `fgt1d delta-sweep`, fgt1d_cli.cpp:317-352):
transform error of an N-point same-point transform as a function of delta,
measured against the sampled direct sum (100 targets).  CSV `delta,error` or
a JSON array of {"delta", "error"}, like the reference.

    python tools/delta_sweep.py --N 10000 --ne 4 --delta 1e-4 --delta 1e-2 [--json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09825_b200 import delta_sweep  # noqa: E402


def main():
    ap = argparse.ArgumentParser(description="Transform error as a function of delta")
    ap.add_argument("--N", type=int, default=10000, help="number of points (same-point set)")
    ap.add_argument("--ne", type=int, default=4, help="folded modes (precision preset 3..6)")
    ap.add_argument("--delta", type=float, action="append", default=[],
                    help="delta values (repeatable; empty emits header only)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dist", default="uniform", help="uniform|chebyshev")
    ap.add_argument("--json", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    try:
        rows = delta_sweep(a.N, a.ne, a.delta, a.seed, a.dist)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    out = open(a.out, "w") if a.out else sys.stdout
    if a.json:
        out.write(json.dumps(rows, indent=2) + "\n")
    else:
        out.write("delta,error\n")
        for r in rows:
            out.write(f"{r['delta']!r},{r['error']!r}\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
