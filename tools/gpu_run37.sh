cd $GRAFT_REPO_ROOT
python tools/stamps_report.py exact float64
python tools/stamps_report.py fast float64
python tools/stamps_report.py fast float32
python tools/time_levels.py exact
python tools/time_levels.py fast
for p in "float64 fast" "float32 fast"; do set -- $p; python bench.py --steps 5 --warmup 3 --no-cpu --no-fine --dtype $1 --precision $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['config']['cycles'], d['gpu_launches'], d['config']['level_sweep_ms'])"; done
