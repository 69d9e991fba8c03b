cd $GRAFT_REPO_ROOT
O=gpurun_out/r01b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q 2>&1 | tail -n 3
python bench.py --steps 5 --warmup 3 --no-cpu > $O/bench_c3.json 2>&1; echo "bench rc=$?"
CMG_NO_GRAPH=1 python bench.py --steps 2 --warmup 3 --no-cpu > $O/plain_c3ng.log 2>&1 && \
CMG_NO_GRAPH=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_c3.log 2>&1
echo "launch list rc=$?"
CMG_NO_GRAPH=1 python tools/prof_both.py > $O/plain_both.log 2>&1 && \
CMG_NO_GRAPH=1 timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -o $O/full_both python tools/prof_both.py > $O/ncu_full_both.log 2>&1
echo "full rc=$?"
tail -n 3 $O/ncu_full_both.log; cat $O/plain_both.log
ls -la $O
