cd $GRAFT_REPO_ROOT
python tools/time_big.py 512 float32 fast 64 '[{}, {"CMG_FUSE_MASK": "3"}, {"CMG_FUSE_MASK": "7"}]'
python tools/time_big.py 4096 float32 fast 1 '[{}, {"CMG_FUSE_MASK": "1"}, {"CMG_FUSE_MASK": "7"}]'
python tools/time_big.py 2048 float64 exact 1 '[{}, {"CMG_FUSE_MASK": "1"}, {"CMG_FUSE_MASK": "3"}, {"CMG_FUSE_MASK": "7"}]'
for c in 5 4; do python bench.py --steps 5 --warmup 3 --no-cpu --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['e2e']['ms_per_step'], d['config']['cycles'], d['gpu_launches'], d['config']['level_sweep_ms'])"; done
