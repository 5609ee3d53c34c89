# full GPU test suite with durations (tag $1); parity record -> gpurun_out/parity_r2.json
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gputest_$1.txt 2>&1
tail -25 gpurun_out/gputest_$1.txt
