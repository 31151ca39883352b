"""SASS-level summary of one kernel in an ncu report (--set full, -lineinfo):
executed warp instructions and stall samples per opcode and per SASS range.
usage: ncu_sass.py REPORT KERNEL_REGEX [NORM] [--dump FILE]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
norm = float(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith('-') else 1.0
dump = sys.argv[sys.argv.index('--dump') + 1] if '--dump' in sys.argv else None
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', f'regex:{kern}',
                      '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if 'Address' in r)
ix = {k: hdr.index(k) for k in hdr}
recs, seen = [], set()
for r in rows:
    if len(r) != len(hdr) or r[0] == 'Address':
        continue
    try:
        n = int(float(r[ix['Instructions Executed']]))
        smp = int(float(r[ix['Warp Stall Sampling (All Samples)']]))
    except ValueError:
        continue
    if r[0] in seen:  # the csv lists each SASS line twice
        continue
    seen.add(r[0])
    recs.append((r[0], r[ix['Source']].strip(), n, smp))
tot = sum(n for _, _, n, _ in recs)
tots = sum(s for _, _, _, s in recs)
print(f'total warp instructions {tot} ({tot / norm:.3f} per unit), samples {tots}')
by = defaultdict(lambda: [0, 0])
for _, s, n, smp in recs:
    op = s.split()[0] if s else '?'
    if op.startswith('@'):
        op = s.split()[1]
    op = op.split('.')[0]
    by[op][0] += n
    by[op][1] += smp
for op, (n, smp) in sorted(by.items(), key=lambda t: -t[1][0])[:30]:
    print(f'{op:12s} {n:12d} {n / norm:7.3f}/unit {100 * n / tot:5.1f}%  samples {100 * smp / max(tots, 1):5.1f}%')
if dump:
    with open(dump, 'w') as f:
        for a, s, n, smp in recs:
            f.write(f'{a[-5:]} {n / norm:8.4f} {smp:6d}  {s}\n')
