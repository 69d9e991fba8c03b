cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CMG_NO_WHILE=1
python tools/prof_solve.py --config 4 --dtype float32 --precision fast --reps 1 --cycles 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_level_fused|k_sweep_team|k_energy" -c 6 -o gpurun_out/prof_c4 python tools/prof_solve.py --config 4 --dtype float32 --precision fast --reps 1 --cycles 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
