cd $GRAFT_REPO_ROOT
for v in "float64 exact" "float32 fast"; do set -- $v
 for coop in 0 1; do
  CMG_COOP=$coop timeout 300 python bench.py --steps 3 --warmup 3 --dtype $1 --precision $2 --no-cpu > gpurun_out/b.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/b.json')); print('$1 $2 coop=$coop', round(d['ms_per_step'],3))" || tail -3 gpurun_out/b.json
 done
done
CMG_COOP=1 timeout 300 python tools/stamps_report.py fast float32
