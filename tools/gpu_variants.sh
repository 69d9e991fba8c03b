#!/bin/bash
# usage: tools/gpu_variants.sh OUTDIR CONFIG "ENV1" "ENV2" ...   (run on the GPU box)
# one bench.py line per env-var setting (device-timed, --no-cpu --no-fine)
O=$1; C=$2; shift 2; mkdir -p $O
i=0
for e in "$@"; do
  env $e timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu --no-fine > $O/c${C}_v$i.json 2>$O/c${C}_v$i.err
  python - "$O/c${C}_v$i.json" "$e" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:40s} ms={d['ms_per_step']:.3f} levels={ {k: round(v*1000,1) for k,v in d.get('detail', d['config']).get('level_sweep_ms',{}).items()} }")
except Exception as ex:
    print(sys.argv[2], "FAILED", ex)
PY
  i=$((i+1))
done
