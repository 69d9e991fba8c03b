cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "float64 exact" "float32 fast"; do set -- $v
 for fc in "0 0 1" "1 1 7" "2 2 7" "3 3 7" "1 3 7" "3 1 7"; do set -- $1 $2 $fc
  CMG_FCFG2=$3 CMG_FCFG3=$4 CMG_FUSE_MASK=$5 timeout 300 python bench.py --steps 3 --warmup 3 --dtype $1 --precision $2 --no-cpu > gpurun_out/b.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/b.json')); print('$1 $2 cfg=$3,$4 mask=$5', round(d['ms_per_step'],3), {k: round(v*1000,1) for k,v in d['config']['level_sweep_ms'].items()})" || tail -3 gpurun_out/b.json
 done
done
for fc in "0 0 1" "1 1 7" "2 2 7" "3 3 7"; do set -- $fc
 CMG_FCFG2=$1 CMG_FCFG3=$2 CMG_FUSE_MASK=$3 timeout 600 python tools/probe_big.py 16384 float32 fast 2>&1 | tail -3 | sed "s/^/cfg=$1,$2 /"
done
