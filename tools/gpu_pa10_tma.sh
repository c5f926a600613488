#!/bin/bash
# k_passA10s<ROWM> bulk-store exit vs STG: N = 17..20 parity, rates, c4 bench, one ncu capture
O=gpurun_out/pa10; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_sums or two_pass or chi_elementwise or scrambled_pair_n20 or config1 or fp32" > $O/tests.txt 2>&1; tail -2 $O/tests.txt
for v in 1 0 1 0; do
  echo "== SRE_PA10_TMA=$v" >> $O/rates.txt
  SRE_PA10_TMA=$v timeout 300 python tools/rate.py 20 4096 8192 2 >> $O/rates.txt 2>&1
  SRE_PA10_TMA=$v timeout 300 python tools/rate.py 18 4096 16384 2 >> $O/rates.txt 2>&1
done
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
NCU_COUNT=1 NCU_SKIP=4 timeout 600 bash tools/ncu_remote.sh pa10/ncu_passA10s 'k_passA10s' python tools/rate.py 20 4096 1024 1
cat $O/rates.txt
