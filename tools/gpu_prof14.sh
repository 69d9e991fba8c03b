cd $GRAFT_REPO_ROOT
O=gpurun_out/r01b; mkdir -p $O
python bench.py --steps 5 --warmup 3 --no-cpu > $O/bench_c3.json 2>&1; echo "bench rc=$?"
CMG_NO_GRAPH=1 python bench.py --steps 2 --warmup 3 --no-cpu > $O/plain_c3ng.log 2>&1 && \
CMG_NO_GRAPH=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_c3.log 2>&1
echo "launch list rc=$?"
R=/tmp/full_both
CMG_NO_GRAPH=1 python tools/prof_both.py > $O/plain_both.log 2>&1 && \
CMG_NO_GRAPH=1 timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -f -o $R python tools/prof_both.py > $O/ncu_full_both.log 2>&1
echo "full rc=$?"
ncu -i $R.ncu-rep --page raw --csv > $O/full_both_raw.csv 2> $O/imp.err
ncu -i $R.ncu-rep --page details --csv > $O/full_both_details.csv 2>> $O/imp.err
ncu -i $R.ncu-rep --page source --csv -k regex:k_l1_x2 > $O/src_l1_x2.csv 2>> $O/imp.err
ncu -i $R.ncu-rep --page source --csv -k regex:k_l1_tile > $O/src_l1_tile.csv 2>> $O/imp.err
ncu -i $R.ncu-rep --page source --csv -k regex:k_coarse_tile > $O/src_coarse.csv 2>> $O/imp.err
ncu -i $R.ncu-rep --page source --csv -k regex:k_sweep_team > $O/src_team.csv 2>> $O/imp.err
ncu -i $R.ncu-rep --page source --csv -k regex:k_energy > $O/src_energy.csv 2>> $O/imp.err
gzip -9 $O/*.csv
ls -la $O; cat $O/imp.err | head
