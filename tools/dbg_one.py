"""Run N iterations of config C (optionally with coarser quadrature) — for
compute-sanitizer runs on the GPU box:  python tools/dbg_one.py 4 1 [coarse]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_17743_b200 as M  # noqa: E402
import problems as P  # noqa: E402

cfg, n = int(sys.argv[1]), int(sys.argv[2])
prob = P.config(cfg)
if "coarse" in sys.argv:
    prob = P.with_quadrature(prob, num_azim=8, num_polar=4, radial_spacing=0.5, axial_spacing=3.0)
s = M.Solver(M.Problem(prob))
print(s.iterate(n), flush=True)
