#!/bin/bash
# usage: tools/gpu_iter.sh <out-subdir> "<pytest -k expr>" "<rate specs separated by ;>" [ncu-kernel-regex ncu-rate-spec]
# One GPU iteration: a parity subset, per-X-string rates, and optionally one ncu --set full capture.
cd $GRAFT_REPO_ROOT
O=gpurun_out/$1; mkdir -p $O
if [ -n "$2" ]; then timeout 1200 python -m pytest tests -x -q -m gpu -k "$2" > $O/tests.txt 2>&1; tail -3 $O/tests.txt; fi
IFS=';' read -ra SPECS <<< "$3"
for spec in "${SPECS[@]}"; do eval "timeout 300 $spec" >> $O/rates.txt 2>&1; done
cat $O/rates.txt
if [ -n "$4" ]; then
  timeout 300 python tools/rate.py $5 > $O/plain_ncu.log 2>&1 && \
  NCU_COUNT=${NCU_COUNT:-1} bash tools/ncu_remote.sh $1/ncu "$4" python tools/rate.py $5
fi
ls $O
