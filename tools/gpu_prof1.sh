cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/prof_solve.py --reps 1 --cycles 3 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_exact.csv python tools/prof_solve.py --reps 1 --cycles 3 > gpurun_out/ncu1.log 2>&1
python tools/prof_solve.py --reps 1 --cycles 3 --precision fast > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fast.csv python tools/prof_solve.py --reps 1 --cycles 3 --precision fast > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log
wc -l gpurun_out/launches_*.csv
