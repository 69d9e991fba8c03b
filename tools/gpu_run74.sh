cd $GRAFT_REPO_ROOT
CMG_L1_SPLIT=1 timeout 1100 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -n 1
python tools/time_big.py 1024 float64 exact 1 '[{}, {"CMG_L1_SPLIT": "1"}, {"CMG_L1_SPLIT": "1", "CMG_L1_WIDE": "0"}]'
python tools/time_big.py 4096 float64 exact 1 '[{}, {"CMG_L1_SPLIT": "1"}]'
for e in '' 'CMG_L1_SPLIT=1'; do env $e python bench.py --steps 5 --warmup 3 --no-cpu --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['ms_per_step'],3), d['config']['level_sweep_ms'])"; done
