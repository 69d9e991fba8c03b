cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 3
for pdl in 1 0; do for p in "float64 exact" "float64 fast" "float32 fast"; do set -- $p; CMG_PDL=$pdl python bench.py --steps 5 --warmup 3 --no-cpu --no-fine --dtype $1 --precision $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl', d['config']['workload'][-30:], round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['config']['cycles'])"; done; done
for pdl in 1 0; do CMG_PDL=$pdl python bench.py --steps 3 --warmup 3 --no-cpu --config 4 --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl c4', round(d['ms_per_step'],3))"; done
for pdl in 1 0; do CMG_PDL=$pdl python bench.py --steps 3 --warmup 3 --no-cpu --config 5 --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl c5', round(d['ms_per_step'],3))"; done
