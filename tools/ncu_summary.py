#!/usr/bin/env python
"""Summarise an ncu report (`--set full`) or launch list (`--metrics gpu__time_duration.sum --csv`)
into the small JSON files committed under profiles/.

    python tools/ncu_summary.py report.ncu-rep  > profiles/<name>.json
    python tools/ncu_summary.py launches.csv     > profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum.pct_of_peak_sustained_elapsed",
    "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg", "sm__cycles_elapsed.avg",
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "sm__maximum_warps_per_active_cycle_pct", "sm__cycles_elapsed.avg.per_second",
]


def _raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        m = {k: (d.get(k), u.get(k)) for k in KEYS if k in d}
        stalls = {}
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(
                        d[k].replace(",", ""))
                except ValueError:
                    pass
        top = dict(sorted(stalls.items(), key=lambda x: -x[1])[:8])
        res.append({"kernel": d.get("Kernel Name"), "metrics": m, "top_stalls_per_issue": top})
    return res


def _launches(path):
    rows = list(csv.reader(open(path)))
    i0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[i0]
    agg = defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows[i0 + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        if unit == "ms":
            v *= 1e3
        elif unit in ("nsecond", "ns"):
            v *= 1e-3
        elif unit in ("msecond",):
            v *= 1e3
        elif unit in ("usecond", "us"):
            pass
        agg[name][0] += 1
        agg[name][1] += v
        order.append((name, v))
    tot = sum(v for _, v in order)
    return {"launches": len(order), "total_us": tot,
            "by_kernel": {k: {"count": c, "total_us": t, "share": t / tot if tot else None} for k, (c, t) in
                          sorted(agg.items(), key=lambda x: -x[1][1])}}


if __name__ == "__main__":
    p = sys.argv[1]
    out = _raw(p) if p.endswith(".ncu-rep") else _launches(p)
    json.dump(out, sys.stdout, indent=1)
    print()
