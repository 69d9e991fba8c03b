#!/bin/bash
# usage: tools/ncu_one.sh <outname> <kernel-regex> <count> <command...>
# plain run, then ncu --set full of the first <count> matching launches;
# exports raw + SASS source pages (gzipped CSV) into gpurun_out/<outname>/
cd $GRAFT_REPO_ROOT
name=$1; kre=$2; cnt=$3; shift 3
O=gpurun_out/$name; mkdir -p $O
"$@" > $O/plain.log 2>&1 || { echo "plain run failed"; tail -5 $O/plain.log; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$kre" -c $cnt -f -o /tmp/$name "$@" > $O/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/$name.ncu-rep --page raw --csv | gzip -9 > $O/raw.csv.gz
ncu -i /tmp/$name.ncu-rep --page source --csv | gzip -9 > $O/src.csv.gz
ncu -i /tmp/$name.ncu-rep --page details --csv | gzip -9 > $O/details.csv.gz
ls -la $O
