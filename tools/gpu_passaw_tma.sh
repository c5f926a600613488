#!/bin/bash
O=gpurun_out/aw; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "streamed_production or chi_elementwise or config5 or n24 or rowmajor or streamed" > $O/tests.txt 2>&1; tail -3 $O/tests.txt
for v in 1 0; do
  echo "== SRE_PAW_TMA=$v" >> $O/rates.txt
  SRE_PAW_TMA=$v timeout 300 python tools/rate.py 24 4096 512 2 >> $O/rates.txt 2>&1
  SRE_PAW_TMA=$v timeout 300 python tools/rate.py 22 4096 1024 2 >> $O/rates.txt 2>&1
done
SRE_PAW_TMA=1 timeout 600 python tools/full_sweep.py 24 scrambled 19 4 > $O/slice_tma.json 2> $O/slice_tma.err
SRE_PAW_TMA=0 timeout 600 python tools/full_sweep.py 24 scrambled 19 4 > $O/slice_stg.json 2> $O/slice_stg.err
NCU_COUNT=1 NCU_SKIP=2 timeout 600 bash tools/ncu_remote.sh aw/ncu_passAw 'k_passAw' python tools/rate.py 24 4096 128 1
cat $O/rates.txt
