cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for prec in exact fast; do
 for ts in "4 8" "8 16" "4 16"; do
  set -- $ts
  CMG_TS2=$1 CMG_TS3=$2 timeout 300 python bench.py --steps 3 --warmup 3 --precision $prec --no-cpu > gpurun_out/b_${prec}_$1_$2.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/b_${prec}_$1_$2.json')); print('$prec ts=$1,$2', round(d['ms_per_step'],3), d['config']['level_sweep_ms'], round(d['e2e']['ms_per_step'],3))"
 done
done
timeout 300 python bench.py --steps 3 --warmup 3 --dtype float32 --precision fast --no-cpu > gpurun_out/b_f32.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/b_f32.json')); print('f32', round(d['ms_per_step'],3), d['config']['level_sweep_ms'], d['config']['cycles_to_tolerance'])"
