cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 3
for c in 3 5 4; do python bench.py --steps 5 --warmup 3 --no-cpu --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['e2e']['ms_per_step'], d['config']['cycles'])"; done
