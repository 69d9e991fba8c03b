cd $GRAFT_REPO_ROOT
timeout 1100 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 2
for p in "float64 exact" "float64 fast" "float32 fast"; do set -- $p; for e in '' 'CMG_FSUM=0'; do env $e python bench.py --steps 5 --warmup 3 --no-cpu --no-fine --dtype $1 --precision $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 $e', round(d['ms_per_step'],3), d['config']['level_sweep_ms'])"; done; done
