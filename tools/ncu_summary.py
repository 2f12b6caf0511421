#!/usr/bin/env python
"""Summaries of one `ncu --set full` report for profiles/ (tracked files):

  <prefix>_details.csv   the --page details table (sections/metrics/rules)
  <prefix>_metrics.csv   selected raw metrics (DRAM bytes, pipes, stalls, occupancy)
  <prefix>_lines.txt     top source lines by warp-stall samples (tools/ncu_lines.py)

and prints the per-launch DRAM traffic (dram__bytes_read.sum + write.sum) that
bench.py reports as roofline.traffic (profiles/traffic.json).

usage: ncu_summary.py report.ncu-rep 'kernel regex' profiles/<prefix> [workload]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

rep, kre, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
workload = sys.argv[4] if len(sys.argv) > 4 else None
here = Path(__file__).resolve().parent
sel = ["--kernel-name-base", "demangled", "--kernel-name", f"regex:{kre}"]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args, *sel], capture_output=True, text=True, check=True).stdout


Path(prefix + "_details.csv").write_text(ncu("--page", "details", "--csv"))
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
keep = ("dram__bytes", "gpu__time_duration", "sm__pipe_fp64", "sm__warps_active", "smsp__average_warps_issue_stalled",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared", "l1tex__data_pipe_lsu_wavefronts_mem_shared",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate", "sm__throughput", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__occupancy_limit", "sm__maximum_warps_per_active_cycle_pct",
        "launch__grid_size", "launch__block_size", "dram__throughput", "smsp__issue_active")
with open(prefix + "_metrics.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["metric", "unit", "value"])
    w.writerow(["Kernel Name", "", vals[hdr.index("Kernel Name")]])
    for h, u, v in zip(hdr, units, vals):
        if any(h.startswith(k) for k in keep):
            w.writerow([h, u, v])
m = dict(zip(hdr, vals))
u = dict(zip(hdr, units))


def as_bytes(k):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(k, "byte"), 1)
    return float(str(m[k]).replace(",", "")) * scale


traffic = as_bytes("dram__bytes_read.sum") + as_bytes("dram__bytes_write.sum")
dur = m.get("gpu__time_duration.sum")
print(f"traffic {traffic:.0f} B per launch, duration {dur} {u.get('gpu__time_duration.sum')}")
lines = subprocess.run([sys.executable, str(here / "ncu_lines.py"), rep, kre, "40"], capture_output=True, text=True)
Path(prefix + "_lines.txt").write_text(lines.stdout)
if workload:
    tj = here.parent / "profiles" / "traffic.json"
    d = json.loads(tj.read_text()) if tj.exists() else {}
    d[workload] = int(traffic)
    d["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum of one launch of the workload's step kernel, "
                  "ncu --set full (cold caches); per-workload reports in profiles/*_metrics.csv")
    tj.write_text(json.dumps(d, indent=1) + "\n")
