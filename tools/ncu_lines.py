#!/usr/bin/env python
"""Top source lines of an ncu report (needs -lineinfo and --import-source):
by warp-stall samples (default) or by executed warp instructions (--inst).

usage: ncu_lines.py report.ncu-rep 'kernel regex' [N] [--inst]"""
import csv
import io
import subprocess
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
by_inst = "--inst" in sys.argv
rep, kre = args[0], args[1]
top = int(args[2]) if len(args) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name-base", "demangled", "--kernel-name", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, fname, agg, tot, tot_i = None, None, {}, 0, 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].strip().isdigit():
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        s = int(float(d.get("Warp Stall Sampling (All Samples)", "0") or 0))
        ni = int(float(d.get("Instructions Executed", "0") or 0))
        stalls = {k[6:]: int(float(v or 0)) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k}
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = agg.setdefault(key, [0, r[1].strip()[:60], {}, 0])
    a[0] += s
    a[3] += ni
    for k, v in stalls.items():
        a[2][k] = a[2].get(k, 0) + v
    tot += s
    tot_i += ni
print(f"total samples {tot}, executed warp instructions {tot_i}")
order = (lambda kv: -kv[1][3]) if by_inst else (lambda kv: -kv[1][0])
for (f, ln), (s, src, st, ni) in sorted(agg.items(), key=order)[:top]:
    big = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / max(tot, 1):5.1f}% inst {100 * ni / max(tot_i, 1):5.1f}% {f}:{ln:<4d} {src:60s} "
          + " ".join(f"{k}={v}" for k, v in big if v))
