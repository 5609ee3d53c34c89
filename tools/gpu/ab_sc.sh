# A/B timing of schedule-3 variants: product build + libmoc3d_<v>.so for each v in $2.. (tag $1)
tag=$1; shift
timeout 300 python tools/ab_sweep.py 5 4 --schedule=3 >> gpurun_out/ab_$tag.jsonl 2>&1
for v in "$@"; do MOC3D_LIB=paper_2503_17743_b200/libmoc3d_$v.so timeout 300 python tools/ab_sweep.py 5 4 --schedule=3 >> gpurun_out/ab_$tag.jsonl 2>&1; done
cat gpurun_out/ab_$tag.jsonl
