#!/usr/bin/env python
"""bench.py — OTF 3D-MOC power iteration on B200 (BASELINE.json metric).

One step = one full power iteration of the hot path (source,
OTF sweep with attenuation + tally + boundary hand-off, finalize, k-eff,
normalisation, residual) over the whole synthetic C5G7-shaped problem, with all
inputs resident in HBM.  `value` = 3D-MOC segment-group integrations per second
(2 x N_seg3D x G per iteration) over the whole job.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]
                    [--backend nccl|gloo] [--schedule 3]

N > 1: one rank per GPU.  Under torchrun (RANK/WORLD_SIZE set) each process is a rank; run
directly with --gpus N > 1, bench.py re-launches itself through torch.distributed.run
(127.0.0.1).  Backend nccl (default): the library owns an NCCL communicator and the whole
iteration (sweep, tally all-reduce, boundary-psi halo, finalize) is one CUDA-graph replay;
gloo (e.g. several ranks sharing one GPU for testing): the exchange is staged through host
memory.  Rank 0 prints the line; `value` = all ranks' integrations / max-over-ranks time.
`--impl reference` times the fp64 CPU oracle (oracle/) on the host cores on a
bounded sample of the same workload (the oracle is a deliberately slow checker:
the ratio is context, parity and roofline fraction are the headline).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import problems as P  # noqa: E402

METRIC = "3D-MOC segment-group integrations/s"
UNIT = "integrations/s"
WORKLOADS = {
    3: "cfg3: single C5G7 UO2 assembly 21.42x21.42x214.2 cm, 7G, 16 azim x 6 polar, 0.1/0.5 cm",
    4: "cfg4: C5G7 3D Rodded B 64.26x64.26x214.2 cm, 7G, 16 azim x 6 polar, 0.1/0.5 cm",
    5: "cfg5: C5G7 3D Rodded B 64.26x64.26x214.2 cm, 7G, 16 azim x 6 polar, fine 0.05/0.1 cm",
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def r_alu(G: int, mhz: float, n_sm: int = 148) -> float:
    """ALU roofline: N_SM f 128 / (5 + 5/G) integrations/s."""
    return n_sm * mhz * 1e6 * 128.0 / (5.0 + 5.0 / G)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical CPUs visible)"
    except OSError:
        pass
    return None


def _host_info():
    """CPU record for the oracle leg: model, sockets, physical cores,
    logical CPUs, RAM, OMP_NUM_THREADS."""
    info = {"cpu_model": _cpu_model(), "logical_cpus": os.cpu_count(),
            "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}
    try:
        phys, sockets = set(), set()
        cur = {}
        for line in open("/proc/cpuinfo"):
            if ":" in line:
                k, v = [x.strip() for x in line.split(":", 1)]
                cur[k] = v
            elif cur:
                sockets.add(cur.get("physical id"))
                phys.add((cur.get("physical id"), cur.get("core id")))
                cur = {}
        info["sockets"] = len(sockets - {None}) or None
        info["physical_cores"] = len({p for p in phys if p[1] is not None}) or None
    except OSError:
        pass
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                info["ram_gb"] = round(int(line.split()[1]) / 1048576, 1)
    except OSError:
        pass
    return info


PAPER_CONTEXT = ("PAPER.md:4 reports a 300-400x speedup of its GPU OTF/EXP MOC over 'traditional methods', "
                 "and P:301 30-100x over OpenMOC, on a 12700KF / 32-core AMD host with 1080Ti, 2080Ti, 3060, "
                 "4090 and MI60 GPUs (Table 1, P:250-260), precision unstated: context only, different "
                 "hardware, problems and baselines")


def oracle_sample(prob, target_s: float = 15.0):
    """Time the oracle as it stands on a bounded sample of the workload's tracks:
    every `stride`-th 3D track, swept once in both directions (re-traced explicitly)."""
    import oracle
    o = oracle.Oracle(prob)
    n3 = o.counts["n_tracks3d"]
    stride = max(1, n3 // 2000)
    sec, nint = o.time_sample_sweep(stride)
    # scale the stride so the measured sample takes ~target_s
    if sec > 0:
        stride = max(1, int(stride * sec / target_s))
    sec, nint = o.time_sample_sweep(stride)
    threads = oracle.num_threads()
    return dict(value=nint / sec, unit=UNIT, cores=threads, kind="oracle", cpu_model=_cpu_model(), host=_host_info(),
                sample=f"every {stride}th of {n3} 3D tracks ({(n3 + stride - 1) // stride} tracks, "
                       f"{nint:.3e} integrations, fp64, explicit re-trace + sweep, {sec:.1f} s on {threads} threads)",
                seconds=sec, integrations=nint)


def k_eff_errors(M, dev):
    """BASELINE metric's 'k-eff err' on problems with a closed-form answer (the oracle
    parity at full size lives in tests/test_gpu_parity.py): converged k of the 1-group
    reflective cube vs nuSf/Sa = 1.5 and of the 7-group cube vs the dominant
    eigenvalue of the dense G x G matrix."""
    out = {}
    for variant in ("1g", "7g"):
        prob = P.config1(variant)
        s = M.Solver(M.Problem(prob), device=dev)
        r = s.solve(tol_k=1e-10, tol_src=1e-8, max_iter=20000, check_every=20)
        m = prob["materials"][0]
        A = np.diag(m["sigma_t"]) - np.array(m["sigma_s"]).T
        kd = float(max(abs(np.linalg.eigvals(np.linalg.solve(A, np.outer(m["chi"], m["nu_sigma_f"]))))))
        out[f"cfg1_{variant}"] = {"k_gpu": r["k"], "k_exact": kd, "abs_err": abs(r["k"] - kd),
                                  "iterations": r["iterations"]}
        del s
    return out


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    prob = P.config(args.config)
    per_step = []
    base = None
    for it in range(args.warmup + args.steps):
        cb = oracle_sample(prob, target_s=args.ref_seconds)
        if it >= args.warmup:
            per_step.append(cb)
        base = cb
    val = float(np.median([c["value"] for c in per_step]))
    ms = float(np.median([c["seconds"] for c in per_step])) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded C5G7-shaped XS, problems/)",
        "config": {"workload": WORKLOADS.get(args.config, f"cfg{args.config}"), "sample": base["sample"]},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": base["cores"], "kind": "oracle",
                         "sample": base["sample"], "cpu_model": base.get("cpu_model"), "host": base.get("host")},
        "paper_context": PAPER_CONTEXT,
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def relaunch(args) -> int:
    """--gpus N > 1 without torchrun: run this script under torch.distributed.run."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_ours(args):
    import torch

    import paper_2503_17743_b200 as M

    rank, world, local = _dist_env()
    ndev = torch.cuda.device_count()
    backend = args.backend or ("nccl" if world <= ndev else "gloo")
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(backend)
    dev = local % max(1, ndev)  # gloo testing: several ranks may share one GPU
    torch.cuda.set_device(dev)
    prob = P.config(args.config)
    if args.xs:  # real NEA C5G7 tables from a user file (k context only; not the benched data)
        prob = P.with_xs(prob, P.load_xs_table(args.xs))
    t0 = time.time()
    pr = M.Problem(prob)
    t_lay = time.time() - t0
    st = pr.stats()
    t0 = time.time()
    s = M.Solver(pr, device=dev, schedule=args.schedule, rank=rank, world=world, exp_mode=1 if args.exp else 0,
                 backend=backend if world > 1 else None)
    t_setup = time.time() - t0
    tm = s.timings()
    G = pr.G
    nint = tm["n_integrations"]
    stream = torch.cuda.current_stream(dev)
    # warm-up
    for _ in range(args.warmup):
        s.iterate(1)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    # timed region: K full iterations in one library call (each a CUDA-graph replay, no
    # host synchronisation in between), CUDA events on the solver's stream
    with ClockSampler(dev) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        e0.record(stream)
        s.iterate(args.steps)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
    rank_ms = [ms]
    if world > 1:
        import torch.distributed as dist
        out = [None] * world
        dist.all_gather_object(out, ms)
        rank_ms = [float(x) for x in out]
        ms = max(rank_ms)
    # per-iteration sweep-kernel times (events around the sweep inside each replay)
    sweep_ms = []
    for _ in range(args.steps):
        s.iterate(1)
        sweep_ms.append(s.timings()["sweep_ms_last"])
    ms_step = ms / args.steps
    value = nint * args.steps / (ms * 1e-3)  # whole job (single problem, strong scaling)
    k, res = s.iterate(0)
    # e2e through the public API with host buffers: H2D of the step's input (cross
    # sections from pinned host memory), one iteration, D2H of the step's result (phi)
    mats = prob["materials"]
    xs = [torch.tensor(np.array([m[key] for m in mats], np.float64)).pin_memory().numpy()
          for key in ("sigma_t", "sigma_s", "nu_sigma_f", "chi")]
    h2d = sum(x.nbytes for x in xs)
    phi_host = torch.empty((s.J, G), dtype=torch.float64).pin_memory().numpy()
    import ctypes
    torch.cuda.synchronize(dev)
    e_steps = max(2, args.steps // 2)
    # one untimed warm-up step of the e2e path (first-use staging buffers, as for the device leg)
    s.update_materials(*xs)
    s.iterate(1)
    M.lib().moc_get_scalar_flux(s._h, phi_host.ctypes.data_as(ctypes.c_void_p))
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    e_marks = []
    for _ in range(e_steps):
        s.update_materials(*xs)
        s.iterate(1)
        M.lib().moc_get_scalar_flux(s._h, phi_host.ctypes.data_as(ctypes.c_void_p))
        e_marks.append(time.perf_counter())
    torch.cuda.synchronize(dev)
    e2e_s = (time.perf_counter() - t0) / e_steps
    print("e2e step ms:", [round(1e3 * (b - a), 2) for a, b in zip([t0] + e_marks[:-1], e_marks)], file=sys.stderr)
    d2h = s.J * G * 8  # phi [J][G] fp64 into the pinned host buffer
    e2e_val = nint / e2e_s
    clocks = clk.summary()
    peaks, kind = _peaks()
    mhz_max = float(peaks.get("sm_max_mhz", 1965.0))
    sweep_med = float(np.median(sweep_ms))
    # the roofline is per GPU: this rank's integrations (its emitted segment-directions x G,
    # = nint on one GPU) over its own sweep time
    emitted = s.timings().get("emitted_last", -1)
    nint_rank = emitted * G if emitted and emitted > 0 else nint / world
    achieved = nint_rank / (sweep_med * 1e-3)
    peak = r_alu(G, mhz_max)
    kerr = k_eff_errors(M, dev) if rank == 0 and not args.no_parity else None
    # |k_gpu - k_oracle| on the benched configuration itself: the fp64 oracle's fixed-N
    # golden (tools/oracle_golden.py, SURVEY §8(c) fixed-N parity), every rank iterating
    gold = os.path.join(ROOT, "tests", "golden", f"cfg{args.config}_it{ {4: 5, 5: 2}.get(args.config, 0)}.npz")
    bench_parity = None
    if not args.no_parity and os.path.exists(gold):
        g = np.load(gold)
        s.reset()
        kg, _ = s.iterate(int(g["fixed_iters"]))
        phi = s.scalar_flux().reshape(-1)[g["sample_idx"]]
        ref = g["phi_sample"]
        pm = float(g["phi_max"])
        mask = ref >= 1e-6 * pm
        bench_parity = {"iterations": int(g["fixed_iters"]), "k_gpu": kg, "k_oracle": float(g["k"]),
                        "abs_err": abs(kg - float(g["k"])),
                        "flux_rel_max": float(np.max(np.abs(phi[mask] - ref[mask]) / ref[mask])),
                        "flux_linf": float(np.max(np.abs(phi - ref)) / pm), "flux_elements_sampled": int(ref.size),
                        "source": os.path.relpath(gold, ROOT)}
    if kerr is not None:
        kerr["benched_config_vs_oracle"] = bench_parity
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = oracle_sample(prob, target_s=args.ref_seconds)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "host")}
    # the unit that binds in practice (from the committed ncu --set full capture of this
    # kernel and config): the L1 LSU data pipe and the issue rate, next to R_ALU
    binding = None
    np_ = os.path.join(ROOT, "profiles", f"ncu_sweep_cfg{args.config}_s{args.schedule}.json")
    if os.path.exists(np_):
        try:  # one sweep = one launch per occupancy group: duration-weighted over its launches
            ks = [k["metrics"] for k in json.load(open(np_)) if "k_sweep" in k["kernel"]]
            w = [float(m["gpu__time_duration.sum"][0]) for m in ks]

            def avg(key):
                return sum(wi * float(m[key][0]) for wi, m in zip(w, ks)) / sum(w) / 100

            binding = {"lsu_data_pipe_busy": avg("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                       "issue_active": avg("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                       "launches_per_sweep": len(ks), "source": os.path.relpath(np_, ROOT)}
        except Exception:
            binding = None
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_cfg{args.config}_s{args.schedule}.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_sweep")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": ("synthetic (seeded C5G7-shaped 7G XS, problems/; deterministic laydown)" if not args.xs
                                 else f"C5G7 geometry with user cross sections {os.path.basename(args.xs)}"),
        "config": {"workload": WORKLOADS.get(args.config, f"cfg{args.config}"), "fsr": st["n_fsr"],
                   "tracks3d": st["n_tracks3d"], "segments3d": tm["n_segs3d"], "groups": G,
                   "integrations_per_step": nint, "parallelism": f"tracks partitioned over {world} GPU(s)",
                   "schedule": args.schedule, "k_eff_after": k, "residual_after": res,
                   "l2": "inputs larger than L2 (boundary psi %.1f GB)" % (2 * 2 * st["n_tracks3d"] * 8 * 4 / 1e9),
                   "host_laydown_s": round(t_lay, 2), "device_setup_s": round(t_setup, 2),
                   "sweep_ms_median": sweep_med, "device_gb": round(tm["device_bytes"] / 1e9, 2),
                   "emitted_last": emitted, "emitted_expected": 2 * tm["n_segs3d"] if world == 1 else None,
                   "sc_units_by_ctas_per_sm": dict(zip(("3", "4", "5"), tm.get("sc_units", [0, 0, 0]))),
                   "backend": backend if world > 1 else None, "per_rank_ms": rank_ms,
                   "cuda_graph": True},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": UNIT, "frac": achieved / peak,
                     "traffic": traffic, "kernel": "k_sweep_sc (one sweep = one launch per occupancy group, timed together)",
                     "peak_basis":
                         f"R_ALU = 148 SM x {mhz_max:.0f} MHz ({kind} sm_max) x 128 / (5 + 5/G), SURVEY 8(d)",
                     "frac_at_measured_clock": (achieved / r_alu(G, clocks["sm_mhz"]))
                     if clocks.get("sm_mhz") else None,
                     "measured_binding": binding},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "moc_solver_update_materials + moc_iterate(1) + moc_get_scalar_flux"},
        "gpu_launches": tm["launches_per_iter"] * args.steps,  # kernels in the K timed graph replays
        "clocks": clocks,
        "cpu_baseline": cpu,
        "k_eff_err": kerr,
        "paper_context": PAPER_CONTEXT,
        "sweep_s_per_iter": sweep_med * 1e-3,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)  # median over >= 20 iterations
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--schedule", type=int, default=3)
    ap.add_argument("--backend", default=None, choices=[None, "nccl", "gloo"],
                    help="multi-rank exchange (default nccl when every rank has its own GPU, else gloo)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the closed-form k-eff error legs")
    ap.add_argument("--exp", action="store_true", help="EXP/OTF hybrid of §4.2 instead of pure OTF (--schedule 0)")
    ap.add_argument("--ref-seconds", type=float, default=15.0)
    ap.add_argument("--xs", default=None, help="C5G7 cross-section table (problems.load_xs_table JSON)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
