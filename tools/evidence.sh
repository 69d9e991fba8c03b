#!/bin/bash
# Round evidence on the GPU box: bench lines (configs 1-5, reference arm),
# the ncu launch list of the default bench command, and one ncu --set full
# capture of a config-3 V-cycle + a 16384^2 fp32 V-cycle.  -> gpurun_out/$1/
O=gpurun_out/${1:-evidence}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 rc=$?"
for c in 1 2 4 5; do
  timeout 600 python bench.py --config $c --no-fine > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "bench c$c rc=$?"
done
timeout 600 python bench.py --impl reference > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err; echo "ref rc=$?"
export CMG_NO_GRAPH=1
python bench.py --steps 2 --warmup 3 --no-cpu --no-fine > $O/plain_launch.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-fine > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/prof_both.py > $O/plain_both.log 2>&1 && \
timeout 1800 ncu --profile-from-start off --set full --clock-control none --import-source on -f -o /tmp/full_both \
  python tools/prof_both.py > $O/ncu_full.log 2>&1; echo "full rc=$?"
ncu -i /tmp/full_both.ncu-rep --page raw --csv > $O/full_both_raw.csv 2> $O/imp.err
for k in k_l1_tile k_l1_x2 k_rowpair k_energy_bulk k_coarse_tile k_sweep_team; do
  ncu -i /tmp/full_both.ncu-rep --page source --csv -k regex:$k > $O/src_$k.csv 2>> $O/imp.err
done
gzip -9 -f $O/*.csv
ls -la $O
