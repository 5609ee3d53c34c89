#!/usr/bin/env python
"""A/B timing of the sweep kernel for a library variant (MOC3D_LIB env var selects the
.so).  Prints one JSON line per config: median sweep ms and integrations/s.

    MOC3D_LIB=paper_2503_17743_b200/libmoc3d_c2.so python tools/ab_sweep.py 4 5 [--exp]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2503_17743_b200 as M  # noqa: E402
import problems as P  # noqa: E402

exp = "--exp" in sys.argv
sched = next((int(a.split("=")[1]) for a in sys.argv if a.startswith("--schedule=")), 0)
# extra solver options as key=value (e.g. sc_lanes_per_cell=1)
extra = {a.split("=")[0]: int(a.split("=")[1]) for a in sys.argv[1:] if "=" in a and not a.startswith("-")}
for cfg in [int(x) for x in sys.argv[1:] if not x.startswith("-") and "=" not in x] or [4]:
    torch.cuda.set_device(0)
    s = M.Solver(M.Problem(P.config(cfg)), exp_mode=1 if exp else 0, schedule=sched, **extra)
    s.iterate(2)
    ms = []
    for _ in range(5):
        s.iterate(1)
        ms.append(s.timings()["sweep_ms_last"])
    t = s.timings()
    med = float(np.median(ms))
    print(json.dumps({"lib": os.path.basename(M.SO_PATH), "cfg": cfg, "exp": exp, "schedule": sched, "opts": extra, "sweep_ms": med,
                      "integrations_per_s": t["n_integrations"] / (med * 1e-3),
                      "exp_fraction": t["exp_segments"] / max(1, t["n_segs3d"]),
                      "exp_gb": t["exp_bytes"] / 1e9, "setup_ms": t["setup_ms"]}), flush=True)
    del s
