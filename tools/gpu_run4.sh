cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -12 gpurun_out/pytest_gpu.log
for prec in exact fast; do
  timeout 300 python bench.py --steps 3 --warmup 3 --precision $prec --no-cpu > gpurun_out/b_${prec}.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/b_${prec}.json')); print('$prec', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['gpu_launches'], d['config']['level_sweep_ms'])" || tail -5 gpurun_out/b_${prec}.json
done
timeout 300 python bench.py --steps 3 --warmup 3 --dtype float32 --precision fast --no-cpu > gpurun_out/b_f32.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/b_f32.json')); print('f32', round(d['ms_per_step'],3), d['config']['cycles_to_tolerance'], d['config']['level_sweep_ms'])" || tail -5 gpurun_out/b_f32.json
