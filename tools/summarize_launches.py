#!/usr/bin/env python3
"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel."""
import collections
import csv
import sys


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0].replace("fgt_b200::", "").replace("<unnamed>::", "")
            v = float(d["Metric Value"].replace(",", ""))
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1e-3)
            tot[name] += v * scale
            cnt[name] += 1
    s = sum(tot.values())
    lines = [f"{'kernel':45s} {'launches':>8s} {'total_us':>11s} {'avg_us':>10s} {'share':>6s}"]
    for k, v in tot.most_common():
        lines.append(f"{k[:45]:45s} {cnt[k]:8d} {v:11.1f} {v / cnt[k]:10.1f} {100 * v / s:5.1f}%")
    # bench.py's untimed setup (synthetic data: RNG + radix sort, FP64 peak
    # probe, torch elementwise) vs the kernels of the timed step
    setup = ("uniform_kernel", "make_keys_kernel", "tile_hist_kernel", "global_hist_kernel",
             "sort_scan_reduce_kernel", "sort_scan_apply_kernel", "scan_apply_kernel", "scatter_kernel",
             "identity_sort_kernel", "unkey_kernel", "fp64_probe_kernel", "at::",
             "void at::", "native::")
    step = {k: v for k, v in tot.items()
            if not (k[5:] if k.startswith("void ") else k).startswith(setup)}
    nstep = max((cnt[k] for k in step if "seg_main_kernel" in k), default=0)
    if step and nstep:
        ss = sum(step.values())
        lines.append("")
        lines.append(f"timed-step kernels only (setup excluded), {nstep} steps in the list; "
                     f"per step {ss / nstep:.1f} us")
        lines.append(f"{'kernel':45s} {'per_step_us':>11s} {'share':>6s}")
        for k, v in sorted(step.items(), key=lambda kv: -kv[1]):
            lines.append(f"{k[:45]:45s} {v / nstep:11.1f} {100 * v / ss:5.1f}%")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
