cd $GRAFT_REPO_ROOT
timeout 1100 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -n 2
python tools/time_big.py 1024 float64 exact 1 '[{}, {"CMG_L1_WIDE": "0"}]'
python tools/time_big.py 1024 float64 fast 1 '[{}]'
python tools/time_big.py 512 float64 exact 1 '[{}]'
python tools/time_big.py 4096 float64 exact 1 '[{}]'
for p in "float64 exact" "float64 fast"; do set -- $p; python bench.py --steps 5 --warmup 3 --no-cpu --no-fine --dtype $1 --precision $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['ms_per_step'],3), d['config']['level_sweep_ms'])"; done
