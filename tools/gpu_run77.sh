cd $GRAFT_REPO_ROOT
for e in '' 'CMG_TS3=16' 'CMG_TS3=32'; do env $e python bench.py --steps 3 --warmup 3 --no-cpu --config 5 --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 $e', round(d['ms_per_step'],3), d['config']['level_sweep_ms'])"; done
for e in '' 'CMG_TS2=8' 'CMG_TS3=16' 'CMG_TS2=8 CMG_TS3=16'; do env $e python bench.py --steps 3 --warmup 3 --no-cpu --config 4 --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $e', round(d['ms_per_step'],3), d['config']['level_sweep_ms'])"; done
