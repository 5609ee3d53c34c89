# interleaved A/B of schedule-3 builds (tag $1, configs $2, variants $3..): each variant
# twice in alternating order, so a first-run or thermal drift shows up as a pair spread
tag=$1; cfgs=$2; shift 2
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = cur ]; then lib=paper_2503_17743_b200/libmoc3d.so; else lib=paper_2503_17743_b200/libmoc3d_$v.so; fi
    MOC3D_LIB=$lib timeout 300 python tools/ab_sweep.py $cfgs --schedule=3 >> gpurun_out/ab_$tag.jsonl 2>&1
  done
done
python - "$tag" <<'PY'
import json,sys,collections
r=collections.defaultdict(list)
for l in open(f"gpurun_out/ab_{sys.argv[1]}.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    r[(d["lib"],d["cfg"])].append(round(d["sweep_ms"],2))
for k,v in sorted(r.items()): print(k, v)
PY
