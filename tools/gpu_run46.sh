cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 5
for p in "float64 exact" "float64 fast" "float32 fast"; do set -- $p; python bench.py --steps 5 --warmup 3 --no-cpu --no-fine --dtype $1 --precision $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][-30:], round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['config']['cycles'], d['config']['level_sweep_ms'])"; done
python tools/stamps_report.py exact float64
