# sanitizer runs, M0 microbenchmarks with clock sampling, EXP re-measure (tag $1)
tag=$1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitizer_${tool}_$tag.txt 2>&1
  tail -3 gpurun_out/sanitizer_${tool}_$tag.txt
done
if [ -f tools/micro/run_micro.sh ]; then bash tools/micro/run_micro.sh gpurun_out/micro_$tag.jsonl; fi
timeout 900 python tools/ab_sweep.py 4 5 --schedule=0 > gpurun_out/exp_$tag.jsonl 2>&1
timeout 900 python tools/ab_sweep.py 4 5 --schedule=0 --exp >> gpurun_out/exp_$tag.jsonl 2>&1
cat gpurun_out/exp_$tag.jsonl | cut -c1-200
