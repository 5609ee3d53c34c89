#!/usr/bin/env python
"""fp64 oracle goldens for the GPU parity tests (test infrastructure: calls only oracle/
and the input generators in problems/; no value here comes from the CUDA path).

    python tools/oracle_golden.py cfg3_reduced     # converged, full phi
    OMP_NUM_THREADS=6 python tools/oracle_golden.py cfg4_it5   # fixed N, sampled phi

Converged cases stop at the SURVEY §8(c) Q11 parity setting (|dk| < tol_k and RMS
fission-source residual < tol_src; §5.1 compares converged k-eff).  Fixed-N
cases run N power iterations from phi = 1, k = 1, psi = 0 (Q11).  phi is the oracle's
normalised scalar flux (sum V F = 1, reading Q12).  Large cases store phi at a seeded
uniform sample of (FSR, group) elements plus the global max (for the normalised L-inf and
the 1e-6 max mask of the per-element criterion, SURVEY §8(c) 'Parity checks')."""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import problems as P  # noqa: E402

# name -> (problem factory, fixed iterations (0 = converge), sampled elements (0 = all))
CASES = {
    "cfg3_reduced": (lambda: P.with_quadrature(P.config(3), num_azim=8, num_polar=4, radial_spacing=0.5,
                                               axial_spacing=3.0), 0, 0),
    # cfg3 assembly at full BASELINE tracking, longer fixed N than the in-test 3 iterations
    "cfg3_it12": (lambda: P.config(3), 12, 60000),
    # cfg3 assembly at cfg5's tracking (dr 0.05 / dz 0.1: the benched lane strides)
    "cfg3_fine_it2": (lambda: P.with_quadrature(P.config(3), radial_spacing=0.05, axial_spacing=0.1), 2, 60000),
    # BASELINE configs[1] (C5G7 Rodded B), SURVEY §8(c) fixed-N = 5
    "cfg4_it5": (lambda: P.config(4), 5, 60000),
    # BASELINE configs[4] (the benched config): SURVEY §8(c) fixed-N = 2 (the oracle
    # re-traces every sweep: ~32 GB of fp64 boundary psi, ~20 min per iteration on 6 cores)
    "cfg5_it2": (lambda: P.config(5), 2, 60000),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", choices=sorted(CASES))
    ap.add_argument("--tol-k", type=float, default=1e-7)
    ap.add_argument("--tol-src", type=float, default=1e-6)
    ap.add_argument("--max-iter", type=int, default=20000)
    args = ap.parse_args()
    import oracle
    oracle.build()
    make, fixed, nsamp = CASES[args.case]
    prob = make()
    t0 = time.time()
    o = oracle.Oracle(prob)
    r = o.solve(fixed_iters=fixed, max_iter=args.max_iter, tol_k=args.tol_k, tol_src=args.tol_src)
    phi = r["phi"]
    extra = {}
    if nsamp and nsamp < phi.size:
        idx = np.sort(np.random.default_rng(17743).choice(phi.size, nsamp, replace=False))
        extra = dict(sample_idx=idx.astype(np.int64), phi_sample=phi.reshape(-1)[idx], phi_shape=np.array(phi.shape),
                     phi_max=phi.max())
    else:
        extra = dict(phi=phi)
    out = os.path.join(ROOT, "tests", "golden", f"{args.case}.npz")
    np.savez_compressed(out, k=r["k"], iterations=r["iterations"], fixed_iters=fixed, k_hist=r["k_hist"],
                        res_hist=r["res_hist"], tol_k=args.tol_k, tol_src=args.tol_src, leakage=r["leakage"],
                        production=r["production"], absorption=r["absorption"],
                        counts=np.array(list(o.counts.values())), threads=oracle.num_threads(),
                        seconds=time.time() - t0, **extra)
    print(f"{args.case}: k={r['k']:.10f} iterations={r['iterations']} seconds={time.time() - t0:.0f} -> {out}")


if __name__ == "__main__":
    main()
