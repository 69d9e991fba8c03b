cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/micro/launch_sync > gpurun_out/micro.txt 2>&1; cat gpurun_out/micro.txt
for prec in exact fast; do
 for cfg in "1 4 16" "1 16 32" "1 8 32" "0 4 16" "7 4 8" "3 4 32"; do
  set -- $cfg
  if [ "$1" = "0" ]; then export CMG_FUSED=0; else export CMG_FUSED=1; fi
  CMG_FUSE_MASK=$1 CMG_TS2=$2 CMG_TS3=$3 timeout 300 python bench.py --steps 3 --warmup 3 --precision $prec --no-cpu > gpurun_out/b.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/b.json')); print('$prec mask=$1 ts=$2,$3', round(d['ms_per_step'],3), {k: round(v*1000,1) for k,v in d['config']['level_sweep_ms'].items()})" || tail -3 gpurun_out/b.json
 done
done
