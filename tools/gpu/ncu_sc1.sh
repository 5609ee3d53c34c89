# one ncu --set full capture of the schedule-3 sweep at config $2 (tag $1), plus work statistics
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_sc -s 2 -c 1 -o gpurun_out/ncu_sc_cfg$2_$1 python tools/ab_sweep.py $2 --schedule=3 > gpurun_out/ncu_sc_cfg$2_$1.log 2>&1
MOC3D_LIB=paper_2503_17743_b200/libmoc3d_stats.so timeout 300 python tools/sc_stats.py $2 > gpurun_out/sc_stats_$1.jsonl 2>&1
cat gpurun_out/sc_stats_$1.jsonl
