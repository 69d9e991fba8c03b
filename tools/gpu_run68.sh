cd $GRAFT_REPO_ROOT
O=gpurun_out/r01g; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -n 5
python bench.py --steps 5 --warmup 3 > $O/bench_c3.json 2>$O/bench_c3.err; echo "bench c3 rc=$?"
python bench.py --steps 5 --warmup 3 --config 4 --no-fine > $O/bench_c4.json 2>$O/bench_c4.err; echo "bench c4 rc=$?"
python bench.py --steps 3 --warmup 3 --config 5 --no-fine > $O/bench_c5.json 2>$O/bench_c5.err; echo "bench c5 rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2>$O/bench_ref.err; echo "bench ref rc=$?"
CMG_NO_GRAPH=1 python bench.py --steps 2 --warmup 3 --no-cpu --no-fine > $O/plain_c3ng.log 2>&1 && \
CMG_NO_GRAPH=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-fine > $O/ncu_launch_c3.log 2>&1
echo "launch list rc=$?"
R=/tmp/full_both
CMG_NO_GRAPH=1 python tools/prof_both.py > $O/plain_both.log 2>&1 && \
CMG_NO_GRAPH=1 timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -f -o $R python tools/prof_both.py > $O/ncu_full_both.log 2>&1
echo "full rc=$?"
ncu -i $R.ncu-rep --page raw --csv > $O/full_both_raw.csv 2> $O/imp.err
ncu -i $R.ncu-rep --page source --csv -k regex:k_l1_x2 > $O/src_l1_x2.csv 2>> $O/imp.err
ncu -i $R.ncu-rep --page source --csv -k regex:k_l1_tile > $O/src_l1_tile.csv 2>> $O/imp.err
gzip -9 $O/*.csv
python tools/ncu_summary.py $O/full_both_raw.csv.gz > $O/full_summary.md
for f in $O/bench_*.json; do echo $f; cat $f; done
cat $O/full_summary.md
ncu -i /tmp/full_both.ncu-rep --page source --csv -k regex:k_rowpair > $O/src_rowpair.csv 2>> $O/imp.err; gzip -9 $O/src_rowpair.csv
