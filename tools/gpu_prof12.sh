# round-1 evidence: bench lines (configs 3/4/5 + reference arm), launch list of the
# default bench command, ncu --set full of the top kernels (config 3 and config 5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r01
O=gpurun_out/r01
python bench.py --steps 5 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
python bench.py --steps 5 --warmup 3 --config 4 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
python bench.py --steps 3 --warmup 3 --config 5 > $O/bench_c5.json 2> $O/bench_c5.err; echo "c5 rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_c3.json 2> $O/ref_c3.err; echo "ref rc=$?"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
# launch list of the default bench command (CPU leg skipped: it launches nothing)
python bench.py --steps 2 --warmup 3 --no-cpu > $O/plain_c3.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_c3.log 2>&1
echo "launch list rc=$?"
CMG_NO_WHILE=1 python bench.py --steps 2 --warmup 3 --no-cpu > $O/plain_c3nw.log 2>&1 && \
CMG_NO_WHILE=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_nowhile.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch_c3nw.log 2>&1
echo "launch list (host-chunked graph) rc=$?"
# full capture: top kernels of config 3 (level-1 tile, level-2/3 team, energy)
python tools/prof_solve.py --reps 1 --cycles 2 > $O/plain_solve.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_l1_tile|k_sweep_team|k_energy" -s 0 -c 3 -o $O/full_c3 python tools/prof_solve.py --reps 1 --cycles 2 > $O/ncu_full_c3.log 2>&1
echo "full c3 rc=$?"
# full capture: config-5-size kernels (fp32 fast: packed level-1, TMA coarse tiles)
python tools/prof_big.py 16384 float32 fast > $O/plain_big.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_l1_x2|k_coarse_tile" -s 0 -c 2 -o $O/full_c5 python tools/prof_big.py 16384 float32 fast > $O/ncu_full_c5.log 2>&1
echo "full c5 rc=$?"
tail -n 2 $O/ncu_launch_c3.log $O/ncu_full_c3.log $O/ncu_full_c5.log
wc -l $O/launches_c3.csv
ls -la $O
