#!/usr/bin/env python
"""SIMT lane efficiency of the v2 work units for a config: per-track merged segment
counts from the device walk, units = bands of <= 256 consecutive stack members, warps
of 32 lanes.  Efficiency = sum(lane cost) / (32 * sum over warps of max lane cost) for
three lane->member assignments: strided (current: p = lane * nact + warp), contiguous,
and cost-sorted within the unit.   python tools/lane_eff.py 4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2503_17743_b200 as M  # noqa: E402
import problems as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
pr = M.Problem(P.config(cfg))
s = M.Solver(pr)
n3 = pr.stats()["n_tracks3d"]
cost = np.zeros(n3, np.int64)
B = 1 << 22
for f in range(0, n3, B):
    cost[f:f + B] = s.checksums(f, min(B, n3 - f))["nseg"]
st = pr.stacks()
tot = {"strided": 0, "contiguous": 0, "sorted": 0}
work = 0
for q in range(len(st["count"])):
    first, cnt = int(st["first"][q]), int(st["count"][q])
    for i0 in range(0, cnt, 256):
        n = min(256, cnt - i0)
        c = cost[first + i0:first + i0 + n]
        work += c.sum()
        nact = (n + 31) // 32
        pad = np.zeros(nact * 32, np.int64)
        pad[:n] = c
        # strided: lane l of warp w takes member l * nact + w
        tot["strided"] += pad.reshape(32, nact).max(axis=0).sum()
        tot["contiguous"] += pad.reshape(nact, 32).max(axis=1).sum()
        srt = np.zeros(nact * 32, np.int64)
        srt[:n] = np.sort(c)[::-1]
        tot["sorted"] += srt.reshape(nact, 32).max(axis=1).sum()
print({k: round(work / (32 * v), 4) for k, v in tot.items()}, "segments", int(work))
