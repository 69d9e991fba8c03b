cd $GRAFT_REPO_ROOT
for e in '' 'CMG_ENERGY_NT=512'; do env $e python tools/stamps_report.py exact float64 | grep -E "energy|per cycle" | tr '\n' ' '; echo " <- $e"; done
for e in '' 'CMG_ENERGY_NT=512'; do env $e python bench.py --steps 5 --warmup 3 --no-cpu --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['ms_per_step'],3))"; done
for e in '' 'CMG_ENERGY_NT=512'; do env $e python bench.py --steps 5 --warmup 3 --no-cpu --no-fine --dtype float32 --precision fast | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('f32 $e', round(d['ms_per_step'],3))"; done
