cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMG_COOP=1 CMG_FUSE_MASK=1 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for v in "float64 exact" "float64 fast" "float32 fast"; do set -- $v
 for cfg in "0 1 4" "1 1 4" "1 1 2" "1 1 8"; do set -- $1 $2 $cfg
  CMG_COOP=$3 CMG_FUSE_MASK=$4 CMG_COOP_OCC=$5 timeout 300 python bench.py --steps 3 --warmup 3 --dtype $1 --precision $2 --no-cpu > gpurun_out/b.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/b.json')); print('$1 $2 coop=$3 mask=$4 occ=$5', round(d['ms_per_step'],3))" || tail -3 gpurun_out/b.json
 done
done
