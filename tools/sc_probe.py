#!/usr/bin/env python
"""Schedule-3 (stack-collective sweep) probe: parity against the oracle, the kernel's own
emitted FSR-id hashes against the oracle's per-track checksums (forward and reversed), and
sweep timings against schedule 0.  Writes JSON lines to --out.  Test infrastructure."""
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
from tools.parity_report import flux_errors  # noqa: E402


def out(f, d):
    print(json.dumps(d), flush=True)
    f.write(json.dumps(d) + "\n")
    f.flush()


def hash_check(M, oracle, prob, name, sample=None, **kw):
    pr = M.Problem(prob)
    s = M.Solver(pr, schedule=3, **kw)
    s.iterate(1)
    nseg, h = s.sweep_checksums()
    o = oracle.Oracle(prob)
    n3 = pr.stats()["n_tracks3d"]
    if sample is None:
        ids = [(0, n3)]
    else:
        rng = np.random.default_rng(7)
        ids = [(int(a), sample) for a in rng.integers(0, max(1, n3 - sample), 5)]
    bad_f = bad_b = badn = tot = 0
    first_bad = None
    for a, n in ids:
        c = o.checksums(a, n)
        fw, bw = slice(2 * a, 2 * (a + n), 2), slice(2 * a + 1, 2 * (a + n), 2)
        bf = np.nonzero(h[fw] != c["hash"])[0]
        bb = np.nonzero(h[bw] != c["rhash"])[0]
        bn = np.nonzero((nseg[fw] != c["nseg"]) | (nseg[bw] != c["nseg"]))[0]
        bad_f += len(bf)
        bad_b += len(bb)
        badn += len(bn)
        tot += n
        if first_bad is None and (len(bf) or len(bb)):
            t = int(a + (bf[0] if len(bf) else bb[0]))
            fs, ls = o.trace3d(t)
            first_bad = dict(track=t, oracle_n=int(len(fs)), gpu_nf=int(nseg[2 * t]), gpu_nb=int(nseg[2 * t + 1]),
                             oracle_ids=fs[:12].tolist(), oracle_len=ls[:12].tolist())
    return dict(case=name, kind="hash", tracks=tot, bad_fwd=bad_f, bad_bwd=bad_b, bad_nseg=badn, first_bad=first_bad,
                opts=kw)


def parity(M, oracle, prob, name, iters, **kw):
    s = M.Solver(M.Problem(prob), schedule=3, **kw)
    t0 = time.time()
    k, _ = s.iterate(iters)
    t = s.timings()
    ref = oracle.Oracle(prob).solve(fixed_iters=iters)
    d = dict(case=name, kind="parity", iters=iters, k_gpu=k, k_oracle=ref["k"], k_abs_err=abs(k - ref["k"]),
             emitted=t["emitted_last"], two_nseg=2 * t["n_segs3d"], opts=kw, seconds=round(time.time() - t0, 1))
    d.update(flux_errors(s.scalar_flux(), ref["phi"]))
    return d


def timing(M, prob, name, iters=4, scheds=(0, 3), **kw):
    res = {}
    for sched in scheds:
        s = M.Solver(M.Problem(prob), schedule=sched, **(kw if sched == 3 else {}))
        s.iterate(1)
        ms = []
        for _ in range(iters):
            s.iterate(1)
            ms.append(s.timings()["sweep_ms_last"])
        t = s.timings()
        res[f"sched{sched}_sweep_ms"] = float(np.median(ms))
        res[f"sched{sched}_k"] = s.iterate(0)[0]
        res[f"sched{sched}_emitted"] = t["emitted_last"]
        res["integrations"] = t["n_integrations"]
        del s
    for sched in scheds:
        res[f"sched{sched}_integ_per_s"] = res["integrations"] / (res[f"sched{sched}_sweep_ms"] * 1e-3)
    return dict(case=name, kind="timing", opts=kw, **res)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sc_probe.jsonl"))
    ap.add_argument("--what", default="hash,parity,timing")
    ap.add_argument("--scheds", default="0,3")
    ap.add_argument("--cfgs", default="4,5")
    args = ap.parse_args()
    import oracle
    import paper_2503_17743_b200 as M
    oracle.build()
    what = args.what.split(",")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "a") as f:
        if "hash" in what:
            out(f, hash_check(M, oracle, P.small_lattice(3, 3, 4), "small_lattice"))
            out(f, hash_check(M, oracle, P.config(2), "cfg2"))
            out(f, hash_check(M, oracle, P.config(1), "cfg1"))
            out(f, hash_check(M, oracle, P.small_lattice(3, 3, 4), "small_lattice_R4", sc_lanes_per_cell=4))
            out(f, hash_check(M, oracle, P.config(3), "cfg3", sample=2000))
        if "parity" in what:
            out(f, parity(M, oracle, P.small_lattice(3, 3, 4), "small_lattice_it8", 8))
            out(f, parity(M, oracle, P.small_lattice(3, 3, 4), "small_lattice_it8_R2", 8, sc_lanes_per_cell=2))
            out(f, parity(M, oracle, P.small_lattice(3, 3, 4, xs=P.xs_synthetic(2)), "small_lattice_G2_it6", 6))
            out(f, parity(M, oracle, P.with_quadrature(P.config(3), num_azim=8, num_polar=4, radial_spacing=0.5,
                                                       axial_spacing=3.0), "cfg3_reduced_it3", 3))
            out(f, parity(M, oracle, P.config(3), "cfg3_it3", 3))
        if "timing" in what:
            for c in args.cfgs.split(","):
                out(f, timing(M, P.config(int(c)), f"cfg{c}", scheds=tuple(int(x) for x in args.scheds.split(","))))


if __name__ == "__main__":
    main()
