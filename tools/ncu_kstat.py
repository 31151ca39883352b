"""Key metrics + stall reasons of the kernels in an ncu report."""
import csv
import subprocess
import sys

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
keys = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'launch__registers_per_thread',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'launch__grid_size', 'launch__block_size']
for row in r[2:]:
    d = dict(zip(h, row))
    print(d['Kernel Name'][:70])
    for k in keys:
        print(f'  {k:60s} {d.get(k)}')
    st = {k.replace('smsp__pcsamp_warps_issue_stalled_', ''): float(v) for k, v in d.items()
          if k.startswith('smsp__pcsamp_warps_issue_stalled_') and 'not_issued' not in k and v.replace('.', '').isdigit()}
    tot = sum(st.values()) or 1
    print('  stalls:', ', '.join(f'{k} {100 * v / tot:.0f}%' for k, v in sorted(st.items(), key=lambda t: -t[1]) if v / tot > 0.02))
