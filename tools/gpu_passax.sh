#!/bin/bash
# k_passAx (TMEM row transposes, SRE_PAW_TX=1) vs k_passAw: parity N = 21..24 (sums and chi), rates, slice, ncu
O=gpurun_out/ax; mkdir -p $O
SRE_PAW_TX=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "streamed_production or chi_elementwise or config5 or two_pass_ranges" > $O/tests.txt 2>&1; tail -2 $O/tests.txt
for v in 1 0; do
  echo "== SRE_PAW_TX=$v" >> $O/rates.txt
  SRE_PAW_TX=$v timeout 300 python tools/rate.py 24 4096 512 2 >> $O/rates.txt 2>&1
  SRE_PAW_TX=$v timeout 300 python tools/rate.py 22 4096 1024 2 >> $O/rates.txt 2>&1
done
cat $O/rates.txt
SRE_PAW_TX=1 timeout 600 python tools/full_sweep.py 24 scrambled 19 4 > $O/slice_tx.json 2> $O/slice_tx.err
SRE_PAW_TX=1 NCU_COUNT=1 NCU_SKIP=2 timeout 600 bash tools/ncu_remote.sh ax/ncu_passAx 'k_passAx' python tools/rate.py 24 4096 128 1
cat $O/slice_tx.json
