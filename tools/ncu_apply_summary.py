#!/usr/bin/env python3
"""Summarise an ncu --set full capture of one whole cfg3 step (plan + apply,
tools/profile_round.sh) into profiles/r02_step_ncu.json and
profiles/traffic.json (the DRAM traffic bench.py reports as roofline.traffic
and roofline_step.traffic)."""
import csv
import json
import subprocess
import sys

rep = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof/step_full.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__grid_size", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_selected",
        "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
        "smsp__pcsamp_warps_issue_stalled_no_instructions"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
kern, tot = [], 0.0
for r in rows[2:]:
    d = {"kernel": r[hdr.index("Kernel Name")][:80]}
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            d[k] = r[i] + (" " + units[i] if units[i] else "")
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    d["dram_bytes"] = float(r[ir]) * scale[units[ir]] + float(r[iw]) * scale[units[iw]]
    tot += d["dram_bytes"]
    kern.append(d)
apply = [k for k in kern if any(t in k["kernel"] for t in ("k1c", "k1agg", "k1b", "scan_top", "k2m_down", "k3c", "k3n"))]
json.dump({"source": "ncu --set full --clock-control none (tools/profile_round.sh) of one cfg3 step: "
                     "N=M=1e8 presorted, delta=1e-3, n_e=6; plan (partition, tile pass, mode table) "
                     "and apply (K1c moments + block aggregates, K2 top, K2m down-sweep with the "
                     "collapsed carries, K3c collapsed main pass)",
           "kernels": kern, "dram_bytes_per_step": tot,
           "dram_bytes_per_apply": sum(k["dram_bytes"] for k in apply),
           "algorithmic_bytes_per_apply": 16 * 2e8},
          open("profiles/r02_step_ncu.json", "w"), indent=1)
k3 = [k for k in kern if "k3c" in k["kernel"] or "k3n" in k["kernel"]]
json.dump({"kernel": "cfg3 step (N=M=1e8, n_e=6): plan + apply", "dram_bytes_per_step": tot,
           "dram_bytes_per_apply": sum(k["dram_bytes"] for k in apply),
           "k3_dram_bytes_per_launch": k3[0]["dram_bytes"] if k3 else None,
           "source": "profiles/r02_step_ncu.json (ncu --set full, dram__bytes_read.sum + "
                     "dram__bytes_write.sum over the step's launches)"},
          open("profiles/traffic.json", "w"), indent=1)
print("traffic GB", tot / 1e9)
for k in kern:
    print(k["kernel"][:40], k["gpu__time_duration.sum"],
          k.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"))
