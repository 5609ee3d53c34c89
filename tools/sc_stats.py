#!/usr/bin/env python
"""Work-decomposition statistics of the schedule-3 sweep (debug build with -DMOC_SC_STATS):

    python -m paper_2503_17743_b200.build paper_2503_17743_b200/libmoc3d_stats.so -DMOC_SC_STATS
    MOC3D_LIB=paper_2503_17743_b200/libmoc3d_stats.so python tools/sc_stats.py 5
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2503_17743_b200 as M  # noqa: E402
import problems as P  # noqa: E402

NAMES = ["unit_dirs", "columns", "active_cells", "full_pieces", "corner_pieces", "q_trips", "full_warp_trips",
         "corner_warp_trips", "full_warp_calls", "corner_warp_calls", "mat_warp_trips", "mat_warp_calls",
         "join_warp_trips", "join_warp_calls", "renorm_warp_trips", "renorm_warp_calls"]
kw = dict(a.split("=") for a in sys.argv[1:] if "=" in a)
for cfg in [int(x) for x in sys.argv[1:] if "=" not in x] or [4]:
    L = M.lib()
    s = M.Solver(M.Problem(P.config(cfg)), schedule=3, **{k: int(v) for k, v in kw.items()})
    st = (C.c_ulonglong * 16)()
    s.iterate(1)
    L.moc_debug_sc_stats(st, 1)
    s.iterate(1)
    L.moc_debug_sc_stats(st, 1)
    d = {n: int(st[i]) for i, n in enumerate(NAMES)}
    t = s.timings()
    d["cfg"] = cfg
    d["segs3d"] = t["n_segs3d"]
    d["cells_per_column"] = d["active_cells"] / d["columns"]
    d["pieces_per_cell"] = (d["full_pieces"] + d["corner_pieces"]) / d["active_cells"]
    d["corner_frac"] = d["corner_pieces"] / (d["full_pieces"] + d["corner_pieces"])
    d["q_per_column"] = d["q_trips"] / d["columns"]
    d["columns_per_unit_dir"] = d["columns"] / d["unit_dirs"]
    d["full_lane_eff"] = d["full_pieces"] / max(1, 32 * d["full_warp_trips"])  # one member per trip
    d["corner_lane_eff"] = d["corner_pieces"] / max(1, 2 * 32 * d["corner_warp_trips"])  # one member (two pieces) per trip
    print(json.dumps(d), flush=True)
    del s
