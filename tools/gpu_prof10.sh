cd $GRAFT_REPO_ROOT
export CMG_NO_WHILE=1 CMG_FUSE_MASK=1
python tools/prof_solve.py --reps 1 --cycles 2 --dtype float32 --precision fast > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --cache-control none -k regex:"k_energy|k_sweep_team" -c 6 -o gpurun_out/prof_en python tools/prof_solve.py --reps 1 --cycles 2 --dtype float32 --precision fast > gpurun_out/ncu.log 2>&1
tail -1 gpurun_out/ncu.log
