#!/usr/bin/env python
"""List backward-branch loops in a cuobjdump -sass listing with instruction counts and
the number of spills / shared-base rematerialisations inside each (quick check of a
kernel's hot loops before spending GPU time).

    cuobjdump -sass -fun <mangled> lib.so > k.sass; python tools/sass_loops.py k.sass
"""
import re
import sys

ins = []
for line in open(sys.argv[1]):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
    if not m or not m.group(1):
        continue
    tgt = int(m.group(1), 16)
    if tgt < a and tgt in addr_idx:
        body = [x for _, x in ins[addr_idx[tgt]:i + 1]]
        def c(p):
            return sum(1 for x in body if re.search(p, x))
        print(f"loop {tgt:#06x}-{a:#06x}: {len(body)} instr, LDL/STL {c(r'LDL|STL')}, CgaCtaId {c('CgaCtaId')}, "
              f"ATOMS {c('ATOMS')}, MUFU {c('MUFU')}, LDS {c(r'LDS')}, LDG {c('LDG')}, D-ops {c(r'^\S*\s*D(ADD|MUL|FMA|SETP)')}")
