"""Per-opcode and per-source-line instruction counts of one kernel in an ncu report
(needs -lineinfo and --import-source): where the warp instructions go."""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', f'regex:{kern}',
                      '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
byop, byline = collections.Counter(), collections.Counter()
tot = 0
for r in rows:
    if 'Instructions Executed' in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    try:
        n = int(float(r[hdr.index('Instructions Executed')]))
    except ValueError:
        continue
    src = r[hdr.index('Source')].strip()
    op = src.split()[0] if src else '?'
    if op.startswith('@'):
        op = src.split()[1]
    byop[op.split('.')[0]] += n
    tot += n
print('total', tot, 'per unit', tot / norm)
for op, n in byop.most_common(30):
    print(f'  {op:10s} {n:12d} {n / norm:8.1f}')
