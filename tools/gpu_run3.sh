cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for prec in exact fast; do
 for occ in 1 2; do
  CMG_OCC=$occ timeout 300 python bench.py --steps 3 --warmup 3 --precision $prec --no-cpu > gpurun_out/b_${prec}_$occ.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/b_${prec}_$occ.json')); print('$prec occ=$occ', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['gpu_launches'])" || tail -5 gpurun_out/b_${prec}_$occ.json
 done
done
CMG_OCC=2 timeout 300 python bench.py --steps 3 --warmup 3 --dtype float32 --precision fast --no-cpu > gpurun_out/b_f32.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/b_f32.json')); print('f32', round(d['ms_per_step'],3), d['config']['cycles_to_tolerance'])" || tail -5 gpurun_out/b_f32.json
