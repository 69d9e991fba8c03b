cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -n 3
for c in 5 4 3; do python bench.py --steps 5 --warmup 3 --no-cpu --no-fine --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['config']['cycles'], d['gpu_launches'], {k: round(v,4) for k,v in d['config']['level_sweep_ms'].items()}, round(d['roofline']['frac'],3))"; done
