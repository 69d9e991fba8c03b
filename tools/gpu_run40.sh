cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 3
python tools/time_big.py 16384 float32 fast 1 '[{}, {"CMG_L1X2": "1"}, {"CMG_L1X2": "7"}, {"CMG_L1X2": "8"}]'
python tools/time_big.py 512 float32 fast 64 '[{}, {"CMG_L1X2": "4"}]'
python bench.py --steps 3 --warmup 3 --no-cpu --config 5 --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['ms_per_step'],3), d['roofline']['frac'], d['config']['level_sweep_ms'])"
python bench.py --steps 5 --warmup 3 --no-cpu --config 4 --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['ms_per_step'],3), d['roofline']['frac'], d['config']['level_sweep_ms'])"
