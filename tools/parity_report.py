#!/usr/bin/env python
"""Parity report: k and FSR flux of the CUDA path against the fp64 oracle on the
parity-test cases, with BOTH flux criteria of SURVEY §8(c):

  linf = max |phi_gpu - phi_or| / max phi_or                  (normalised L-inf)
  rel  = max |phi_gpu - phi_or| / phi_or  over phi_or >= 1e-6 max phi_or

Writes one JSON object per case (and where the worst element sits) to the path given
by --out (default gpurun_out/parity_report.jsonl).  Test infrastructure: calls oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import problems as P  # noqa: E402


def flux_errors(phi, ref, mat=None):
    linf = float(np.abs(phi - ref).max() / np.abs(ref).max())
    mask = ref >= 1e-6 * ref.max()
    rel_all = np.where(mask, np.abs(phi - ref) / np.where(mask, ref, 1.0), 0.0)
    w = np.unravel_index(int(np.argmax(rel_all)), rel_all.shape)
    out = dict(linf=linf, rel=float(rel_all[w]), worst_fsr=int(w[0]), worst_group=int(w[1]),
               worst_phi_over_max=float(ref[w] / ref.max()))
    if mat is not None:
        out["worst_material"] = int(mat[w[0]])
    # distribution of per-element relative error by flux band
    for lo, hi in ((1e-6, 1e-4), (1e-4, 1e-2), (1e-2, 1.01)):
        b = mask & (ref >= lo * ref.max()) & (ref < hi * ref.max())
        out[f"rel_band_{lo:g}_{hi:g}"] = float(rel_all[b].max()) if b.any() else None
    return out


def run_case(M, oracle, name, prob, iters=None, converge=None, **solver_kw):
    t0 = time.time()
    pr = M.Problem(prob)
    s = M.Solver(pr, **solver_kw)
    if converge:
        r = s.solve(**converge)
        k = r["k"]
        ref = oracle.Oracle(prob).solve(max_iter=20000, tol_k=1e-10, tol_src=1e-9)
    else:
        k, _ = s.iterate(iters)
        ref = oracle.Oracle(prob).solve(fixed_iters=iters)
    phi = s.scalar_flux()
    mat = oracle.Oracle(prob).fsr_material()
    d = dict(case=name, iters=iters, converged=bool(converge), k_gpu=k, k_oracle=ref["k"],
             k_abs_err=abs(k - ref["k"]), emitted=s.timings()["emitted_last"],
             n_segs3d=s.timings()["n_segs3d"], opts={k: v for k, v in solver_kw.items()},
             seconds=round(time.time() - t0, 1))
    d.update(flux_errors(phi, ref["phi"], mat))
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_report.jsonl"))
    ap.add_argument("--cases", default="all")
    ap.add_argument("--schedule", type=int, default=None)
    args = ap.parse_args()
    import oracle
    import paper_2503_17743_b200 as M
    oracle.build()
    kw = {} if args.schedule is None else {"schedule": args.schedule}
    cases = [
        ("small_lattice_3x3x4_it8", P.small_lattice(3, 3, 4), dict(iters=8)),
        ("small_lattice_G2_it6", P.small_lattice(3, 3, 4, xs=P.xs_synthetic(2)), dict(iters=6)),
        ("cfg2_converged", P.config(2), dict(converge=dict(tol_k=1e-8, tol_src=1e-7, max_iter=5000))),
        ("cfg3_reduced_it3", P.with_quadrature(P.config(3), num_azim=8, num_polar=4, radial_spacing=0.5,
                                               axial_spacing=3.0), dict(iters=3)),
        ("cfg3_it3", P.config(3), dict(iters=3)),
        ("cfg4_it2", P.config(4), dict(iters=2)),
    ]
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "a") as f:
        for name, prob, how in cases:
            if args.cases != "all" and name not in args.cases.split(","):
                continue
            d = run_case(M, oracle, name, prob, **how, **kw)
            print(json.dumps(d), flush=True)
            f.write(json.dumps(d) + "\n")


if __name__ == "__main__":
    main()
