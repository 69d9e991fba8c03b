cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CMG_PERSIST=0 CMG_NO_WHILE=1
python tools/prof_solve.py --reps 1 --cycles 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 12 -o gpurun_out/prof_exact python tools/prof_solve.py --reps 1 --cycles 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
