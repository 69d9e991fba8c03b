cd $GRAFT_REPO_ROOT
timeout 1100 python -m pytest tests/test_gpu_variants.py -m gpu -q -x -k "fp32" 2>&1 | tail -n 2
python tools/time_big.py 16384 float32 fast 1 '[{}]'
python bench.py --steps 3 --warmup 3 --no-cpu --config 5 --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['ms_per_step'],3), d['roofline']['frac'], d['config']['level_sweep_ms'])"
python bench.py --steps 3 --warmup 3 --no-cpu --config 4 --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['ms_per_step'],3), d['config']['level_sweep_ms'])"
