# M0 microbenchmarks with the SM clock sampled by nvidia-smi during the run: the JSON lines of
# micro.cu, then one {"clocks": ...} line (median / min / max SM MHz, throttle reasons seen).
out=${1:-gpurun_out/micro.jsonl}
d=$(dirname "$0")
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o $d/micro $d/micro.cu || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.active --format=csv,noheader,nounits -lms 50 > /tmp/micro_clk.txt &
smi=$!
$d/micro > $out
kill $smi
python - "$out" <<'PY'
import json, sys, statistics
rows = [l.split(",") for l in open("/tmp/micro_clk.txt") if l.strip()]
mhz = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
rs = sorted({r[1].strip() for r in rows if len(r) > 1})
busy = [m for m in mhz if m > 1500] or mhz  # samples while a kernel ran (idle gaps drop the clock)
med = statistics.median(busy) if busy else None
lines = [json.loads(l) for l in open(sys.argv[1])]
with open(sys.argv[1], "w") as f:
    for d in lines:
        if "ops_per_s" in d and med:
            # per-SM rate per clock at the SM clock sampled during the run (the kernel's own
            # clock64 spans undercount when blocks are not all co-resident)
            d["ops_per_sm_clk_at_sampled_clock"] = round(d["ops_per_s"] / (148 * med * 1e6), 3)
        f.write(json.dumps(d) + "\n")
    f.write(json.dumps({"clocks": {"sm_mhz_median_busy": med, "sm_mhz_min": min(mhz) if mhz else None,
                                   "sm_mhz_max": max(mhz) if mhz else None, "samples": len(mhz),
                                   "event_reasons_bitmasks": rs}}) + "\n")
PY
cat $out
