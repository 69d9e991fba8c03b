cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 3
python tools/time_big.py 16384 float32 fast 1 '[{}, {"CMG_L1X2": "3"}]'
python tools/time_big.py 512 float32 fast 64 '[{}, {"CMG_L1X2": "3"}]'
python bench.py --steps 5 --warmup 3 --no-cpu --config 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
