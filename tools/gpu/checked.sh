# bounds-checked build (-DMOC_SC_CHECK: shared-memory psi/hash, plane, FSR and link indices
# of the sweep trap when out of range) under the GPU test suite and a full-size cfg4/cfg5
# sweep (tag $1); stands in for compute-sanitizer where that is unavailable
tag=$1
MOC3D_LIB=paper_2503_17743_b200/libmoc3d_check.so timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/checked_tests_$tag.txt 2>&1
tail -3 gpurun_out/checked_tests_$tag.txt
MOC3D_LIB=paper_2503_17743_b200/libmoc3d_check.so timeout 600 python tools/ab_sweep.py 5 4 --schedule=3 > gpurun_out/checked_sweep_$tag.jsonl 2>&1
cut -c1-160 gpurun_out/checked_sweep_$tag.jsonl
