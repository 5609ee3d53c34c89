# multi-rank at full size on one GPU (gloo host exchange): 1 vs 2 ranks, same iteration count
for n in 1 2; do
  timeout 1500 python bench.py --gpus $n --backend gloo --config ${1:-5} --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/scale_gloo_n$n.json 2> gpurun_out/scale_gloo_n$n.err
  tail -1 gpurun_out/scale_gloo_n$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['config']['k_eff_after'], d['config']['per_rank_ms'], d['config']['device_gb'])"
done
