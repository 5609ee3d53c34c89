# A/B of solver options on schedule 3: each arg "lib:opt=v,opt=v" (lib '' = product build) (tag $1)
tag=$1; shift
for spec in "$@"; do
  lib=${spec%%:*}; opts=${spec#*:}; opts=${opts//,/ }
  if [ -n "$lib" ]; then export MOC3D_LIB=paper_2503_17743_b200/libmoc3d_$lib.so; else unset MOC3D_LIB; fi
  timeout 300 python tools/ab_sweep.py 5 4 --schedule=3 $opts >> gpurun_out/ab_$tag.jsonl 2>&1
done
cut -c1-160 gpurun_out/ab_$tag.jsonl
