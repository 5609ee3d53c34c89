#!/usr/bin/env python
"""Per-CUDA-source-line share of executed warp instructions and warp-stall samples of one
kernel in an ncu report (`--import-source on`, `-lineinfo` build).

    python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top-N]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "k_sweep"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, smp, text = collections.Counter(), collections.Counter(), {}
f, hdr = "?", None
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr) or not r[0].strip():
        continue
    ie, sm = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    key = (f, int(r[0]))
    text[key] = r[1].strip()[:100]
    try:
        agg[key] += int(r[ie] or 0)
        smp[key] += int(r[sm] or 0)
    except ValueError:
        pass
tot, ts = sum(agg.values()) or 1, sum(smp.values()) or 1
print(f"warp instructions {tot:.4e}, stall samples {ts}")
for k, v in agg.most_common(top):
    print(f"{v / tot * 100:5.1f}% {smp[k] / ts * 100:5.1f}%  {k[0]}:{k[1]}  {text[k]}")
