cd $GRAFT_REPO_ROOT
timeout 1100 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 3
for p in "float64 exact" "float64 fast" "float32 fast"; do set -- $p; for e in '' 'CMG_RP_TS2=8' 'CMG_RP_TS2=4'; do env $e python bench.py --steps 5 --warmup 3 --no-cpu --no-fine --dtype $1 --precision $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2 $e', round(d['ms_per_step'],3))"; done; done
python bench.py --steps 3 --warmup 3 --no-cpu --no-fine --config 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['ms_per_step'],3), d['config']['cycles'])"
CMG_ROWPAIR=0 python bench.py --steps 3 --warmup 3 --no-cpu --no-fine --config 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 rp0', round(d['ms_per_step'],3), d['config']['cycles'])"
python bench.py --steps 3 --warmup 3 --no-cpu --no-fine --config 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['ms_per_step'],3), d['config']['cycles'])"
CMG_ROWPAIR=0 python bench.py --steps 3 --warmup 3 --no-cpu --no-fine --config 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 rp0', round(d['ms_per_step'],3), d['config']['cycles'])"
