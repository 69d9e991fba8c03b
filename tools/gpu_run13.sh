cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for x in 1 0; do
  CMG_L1X2=$x timeout 300 python bench.py --steps 3 --warmup 3 --dtype float32 --precision fast --no-cpu > gpurun_out/b.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/b.json')); print('f32 x2=$x', round(d['ms_per_step'],3), {k: round(v*1000,1) for k,v in d['config']['level_sweep_ms'].items()}, d['config']['cycles'])" || tail -3 gpurun_out/b.json
  CMG_L1X2=$x timeout 600 python tools/probe_big.py 16384 float32 fast 2>&1 | tail -4
done
