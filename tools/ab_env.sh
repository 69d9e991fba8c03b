#!/bin/bash
# A/B timing of config 3 under environment settings: tools/ab_env.sh <out> "<ENV=..>" "<ENV=..>" ...
# (bench.py --no-cpu --no-fine per setting; prints ms per solve for fp64 exact / fp64 fast / fp32 fast)
O=gpurun_out/$1; shift; mkdir -p $O
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 300 python bench.py --no-cpu --no-fine > $O/b_$i.json 2>$O/b_$i.err
  python -c "
import json;d=json.load(open('$O/b_$i.json'));print('$e', round(d['ms_per_step'],3), {k:round(v*1000,1) for k,v in d['detail']['level_sweep_ms'].items()})" || tail -3 $O/b_$i.err
done
