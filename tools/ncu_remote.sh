#!/bin/bash
# usage: tools/ncu_remote.sh <name> <kernel-regex> <cmd...>
# Runs ncu --set full on NCU_COUNT (default 1) launches of the kernel (after NCU_SKIP launches), then keeps
# only CSV exports (raw + source) in gpurun_out/<name>.* (full reports exceed the 64 MiB copy-back limit).
name=$1; shift; kre=$1; shift
tmp=/tmp/ncu_$(echo $name | tr '/' '_')
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-1} -o $tmp "$@" > gpurun_out/$name.ncu.log 2>&1
ncu -i $tmp.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
ncu -i $tmp.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.src.csv 2>/dev/null
gzip -f gpurun_out/$name.src.csv
rm -f $tmp.ncu-rep
