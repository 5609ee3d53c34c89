#!/usr/bin/env python
"""Small product-path run for compute-sanitizer (memcheck / racecheck / synccheck):
configs 1 and 2 and a small heterogeneous lattice, schedules 3 (product) and 0, two power
iterations each plus one checksum-mode sweep (schedule 3).  Prints k per case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2503_17743_b200 as M  # noqa: E402
import problems as P  # noqa: E402

for name, prob in (("cfg1", P.config(1)), ("cfg2", P.config(2)), ("lattice", P.small_lattice(3, 3, 4))):
    for sched in (3, 0):
        s = M.Solver(M.Problem(prob), schedule=sched, no_graph=True)
        k, _ = s.iterate(2)
        if sched == 3:
            s.sweep_checksums()
        print(name, sched, k, flush=True)
        del s
