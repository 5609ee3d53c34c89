set -x
for c in 5 4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_sc -s 2 -c 1 -o gpurun_out/ncu_sc_cfg${c}_r2a python tools/ab_sweep.py $c --schedule=3 > gpurun_out/ncu_sc_cfg${c}_r2a.log 2>&1
done
