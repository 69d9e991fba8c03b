cd $GRAFT_REPO_ROOT
for e in '' 'CMG_FUSE_MASK=3' 'CMG_FUSE_MASK=3 CMG_TMA=0'; do env $e python bench.py --steps 3 --warmup 3 --no-cpu --config 4 --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $e', round(d['ms_per_step'],3), d['config']['level_sweep_ms'])"; done
