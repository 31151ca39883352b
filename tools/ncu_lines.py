#!/usr/bin/env python3
"""Aggregate warp-stall samples of an ncu source page (cuda,sass interleaved
csv) per CUDA source line: python tools/ncu_lines.py page.csv [top]."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
SORTCOL = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
acc = defaultdict(lambda: [0, 0, ""])
fname = "?"
col = None
cur = None
total = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        col = r.index("Warp Stall Sampling (All Samples)")
        icol = r.index("Instructions Executed")
        continue
    if col is None or len(r) <= col:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        acc[cur][2] = r[1][:90]
    elif cur is not None and r[2].startswith("0x"):
        s = int(r[col] or 0)
        acc[cur][0] += s
        acc[cur][1] += int(float(r[icol] or 0))
        total += s
print("total samples", total)
for k, (s, n, src) in sorted(acc.items(), key=lambda kv: -kv[1][SORTCOL])[:top]:
    print(f"{100.0 * s / max(total, 1):5.1f}% {s:7d} {n:11d} {k[0]}:{k[1]:<5d} {src}")
