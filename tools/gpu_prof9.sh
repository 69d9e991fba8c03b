cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export CMG_NO_WHILE=1
python tools/prof_big.py 8192 float32 fast > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_coarse_tile" -c 2 -o gpurun_out/prof_coarse2 python tools/prof_big.py 8192 float32 fast > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
