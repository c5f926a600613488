#!/bin/bash
# usage: tools/ncu_remote.sh <name> <kernel-regex> <cmd...>
# Runs ncu --set full on NCU_COUNT (default 1) launches of the kernel, then keeps only CSV exports (raw + source)
# in gpurun_out/ (full reports exceed the 64 MiB copy-back limit).
name=$1; shift; kre=$1; shift
ncu --set full --clock-control none --import-source on -k regex:"$kre" -c ${NCU_COUNT:-1} -o /tmp/$name "$@" > gpurun_out/$name.ncu.log 2>&1
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.src.csv 2>/dev/null
gzip -f gpurun_out/$name.src.csv
rm -f /tmp/$name.ncu-rep
