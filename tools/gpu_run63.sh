cd $GRAFT_REPO_ROOT
timeout 1100 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 3
for e in '' 'CMG_FSUM=0'; do env $e python bench.py --steps 3 --warmup 3 --no-cpu --config 5 --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 $e', round(d['ms_per_step'],3), d['config']['level_sweep_ms'])"; done
python tools/time_big.py 16384 float32 fast 1 '[{}, {"CMG_TMA": "0"}]'
