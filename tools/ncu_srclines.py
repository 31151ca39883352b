"""Top CUDA source lines of one kernel by executed warp instructions (ncu report
with -lineinfo / --import-source)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', f'regex:{kern}',
                      '--print-source', 'cuda'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, res, fname = None, [], ''
for r in rows:
    if 'Instructions Executed' in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        if r and r[0].startswith('File'):
            fname = r[0]
        continue
    try:
        n = int(float(r[hdr.index('Instructions Executed')]))
    except ValueError:
        continue
    if n:
        res.append((n, r[hdr.index('#')] if '#' in hdr else '', r[hdr.index('Source')].strip()[:100]))
res.sort(reverse=True)
tot = sum(n for n, _, _ in res)
print('total', tot, tot / norm)
for n, ln, src in res[:top]:
    print(f'{n / norm:8.1f}  {ln:>5}  {src}')
