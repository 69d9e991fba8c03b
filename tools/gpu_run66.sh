cd $GRAFT_REPO_ROOT
timeout 1100 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 2
for p in "float64 exact" "float64 fast" "float32 fast"; do set -- $p; python bench.py --steps 5 --warmup 3 --no-cpu --no-fine --dtype $1 --precision $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['ms_per_step'],3), d['config']['level_sweep_ms'])"; done
python tools/stamps_report.py exact float64
for c in 1 2; do python bench.py --steps 3 --warmup 3 --no-cpu --no-fine --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', round(d['ms_per_step'],3))"; done
