cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in "float64 exact" "float64 fast" "float32 fast"; do set -- $v
  timeout 300 python bench.py --steps 3 --warmup 3 --dtype $1 --precision $2 --no-cpu > gpurun_out/b.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/b.json')); print('$1 $2', round(d['ms_per_step'],3))" || tail -3 gpurun_out/b.json
done
for mask in 1 3 7; do
CMG_FUSE_MASK=$mask timeout 300 python bench.py --steps 3 --warmup 3 --config 4 --no-cpu > gpurun_out/b.json 2>&1
python -c "import json,sys; d=json.load(open('gpurun_out/b.json')); print('cfg4 mask=$mask', round(d['ms_per_step'],3))" || tail -3 gpurun_out/b.json
done
timeout 900 python bench.py --steps 2 --warmup 3 --config 5 --no-cpu > gpurun_out/b5.json 2>&1
python -c "import json,sys; d=json.load(open('gpurun_out/b5.json')); print('cfg5', round(d['ms_per_step'],3), d['roofline']['frac'])" || tail -3 gpurun_out/b5.json
