#!/usr/bin/env python
"""Aggregate an ncu source page (SASS view) into kernel regions: instructions executed,
thread instructions and warp-stall samples per region, the regions being the top-level
SASS loops (backward branches) of the kernel, plus stall samples at barriers.

    python tools/ncu_regions.py prof.ncu-rep [kernel-regex]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "k_sweep_v2"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
data = rows[rows.index(hdr) + 1:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex, ith = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
ismp = hdr.index("Warp Stall Sampling (All Samples)")
ins = []
for r in data:
    try:
        ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ith] or 0), int(r[ismp] or 0)))
    except (ValueError, IndexError):
        continue
base = ins[0][0]
addr = {a: i for i, (a, *_ ) in enumerate(ins)}
loops = []
for i, (a, t, *_) in enumerate(ins):
    m = re.search(r"BRA (?:\S+ )?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr:
            loops.append((addr[tgt], i))
T = sum(x[2] for x in ins)
TS = sum(x[4] for x in ins)
TT = sum(x[3] for x in ins)
print(f"total warp inst {T:.4g}, thread inst {TT:.4g} ({TT / max(T, 1):.2f}/warp inst), stall samples {TS}")
# innermost-first: report loops holding > 2% of instructions
seen = set()
for lo, hi in sorted(loops, key=lambda x: x[1] - x[0]):
    ex = sum(ins[j][2] for j in range(lo, hi + 1) if j not in seen)
    if ex < 0.02 * T:
        continue
    th = sum(ins[j][3] for j in range(lo, hi + 1) if j not in seen)
    sm = sum(ins[j][4] for j in range(lo, hi + 1) if j not in seen)
    print(f"loop [{ins[lo][0] - base:#07x},{ins[hi][0] - base:#07x}] {hi - lo + 1:4d} instr: "
          f"{100 * ex / T:5.1f}% inst, {th / max(ex, 1):5.2f} thr/inst, {100 * sm / TS:5.1f}% stall samples")
    seen.update(range(lo, hi + 1))
rest = [j for j in range(len(ins)) if j not in seen]
print(f"outside those loops: {100 * sum(ins[j][2] for j in rest) / T:5.1f}% inst, "
      f"{100 * sum(ins[j][4] for j in rest) / TS:5.1f}% stall samples")
bar = [x for x in ins if x[1].startswith("BAR") or " BAR." in x[1]]
print(f"barriers: {100 * sum(x[4] for x in bar) / TS:5.1f}% stall samples")
hot = sorted(ins, key=lambda x: -x[4])[:12]
for a, t, ex, th, sm in hot:
    print(f"  hot {a - base:#07x} {100 * sm / TS:5.2f}% {t[:60]}")
