cd $GRAFT_REPO_ROOT
for e in 'CMG_ENERGY_CTAS=64' 'CMG_ENERGY_CTAS=128' 'CMG_ENERGY_CTAS=148' '' 'CMG_ENERGY_CTAS=512' 'CMG_FUSED_FINALIZE=0'; do env $e python tools/stamps_report.py exact float64 | grep -E "energy|finalize|per cycle" | tr '\n' ' '; echo " <- $e"; done
for e in 'CMG_ENERGY_CTAS=128' 'CMG_ENERGY_CTAS=148' ''; do env $e python bench.py --steps 5 --warmup 3 --no-cpu --no-fine | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['ms_per_step'],3))"; done
