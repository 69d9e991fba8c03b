cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CMG_NO_WHILE=1 CMG_TS2=4 CMG_TS3=16
python tools/prof_solve.py --reps 1 --cycles 3 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/launches_exact.csv python tools/prof_solve.py --reps 1 --cycles 3 > gpurun_out/ncu1.log 2>&1
python tools/prof_solve.py --reps 1 --cycles 3 --precision fast > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fast.csv python tools/prof_solve.py --reps 1 --cycles 3 --precision fast > gpurun_out/ncu2.log 2>&1
wc -l gpurun_out/launches_*.csv
