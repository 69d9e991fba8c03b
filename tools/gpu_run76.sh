cd $GRAFT_REPO_ROOT
timeout 1100 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -n 1
python tools/stamps_report.py exact float64 | grep -E "energy|per cycle"
for p in "float64 exact" "float32 fast"; do set -- $p; python bench.py --steps 5 --warmup 3 --no-cpu --no-fine --dtype $1 --precision $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['ms_per_step'],3))"; done
