#!/usr/bin/env python
"""Small product-path run for compute-sanitizer (memcheck / racecheck / synccheck):
configs 1 and 2 and a small heterogeneous lattice, schedules 3 (product; its 5 CTAs per SM
instance, which small stacks get, and the forced 3 CTAs per SM instance with the dynamic
plane copies and shuffled cell data) and 0, two power iterations each plus one
checksum-mode sweep (schedule 3).  Prints k per case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2503_17743_b200 as M  # noqa: E402
import problems as P  # noqa: E402

for name, prob in (("cfg1", P.config(1)), ("cfg2", P.config(2)), ("lattice", P.small_lattice(3, 3, 4))):
    for sched, opt in ((3, {}), (3, dict(sc_ctas_per_sm=3)), (0, {})):
        s = M.Solver(M.Problem(prob), schedule=sched, no_graph=True, **opt)
        k, _ = s.iterate(2)
        if sched == 3 and not opt:
            s.sweep_checksums()
        print(name, sched, opt, k, flush=True)
        del s
