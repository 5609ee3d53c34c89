# round bench evidence (tag $1): bench line cfg5 (+cfg4), reference arm, ncu launch list and one
# ncu --set full capture of the sweep kernel; summaries written under gpurun_out/
tag=$1
python bench.py > gpurun_out/bench_cfg5_$tag.json 2> gpurun_out/bench_cfg5_$tag.err
python bench.py --config 4 --no-cpu > gpurun_out/bench_cfg4_$tag.json 2> gpurun_out/bench_cfg4_$tag.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg5_$tag.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-parity > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_sc -s 3 -c 1 -o gpurun_out/ncu_sweep_cfg5_$tag python bench.py --steps 1 --warmup 3 --no-cpu --no-parity > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_sc -s 3 -c 1 -o gpurun_out/ncu_sweep_cfg4_$tag python bench.py --config 4 --steps 1 --warmup 3 --no-cpu --no-parity > /dev/null 2>&1
cat gpurun_out/bench_cfg5_$tag.json gpurun_out/bench_cfg4_$tag.json gpurun_out/bench_ref_$tag.json | cut -c1-400
