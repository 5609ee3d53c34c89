# quick schedule-3 check: hashes, small parity, cfg4/cfg5 timing (tag in $1)
timeout 900 python tools/sc_probe.py --out gpurun_out/sc_probe_$1.jsonl --scheds 3 > gpurun_out/sc_probe_$1.log 2>&1
tail -4 gpurun_out/sc_probe_$1.log
