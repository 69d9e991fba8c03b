cd $GRAFT_REPO_ROOT
export CMG_FUSE_MASK=1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
CMG_NO_WHILE=1 timeout 900 python -m pytest tests -m gpu -q -x -k "small or c2_J3" 2>&1 | tail -1
timeout 300 python tools/stamps_report.py exact float64
timeout 300 python tools/stamps_report.py fast float32
for v in "float64 exact" "float32 fast"; do set -- $v
  timeout 300 python bench.py --steps 3 --warmup 3 --dtype $1 --precision $2 --no-cpu > gpurun_out/b.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/b.json')); print('$1 $2', round(d['ms_per_step'],3))" || tail -3 gpurun_out/b.json
done
