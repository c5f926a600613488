#!/bin/bash
# k_midr (ring-fed N = 14 generation) vs k_mid: parity, c3 bench, rates, ncu
O=gpurun_out/midr; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spectrum.py -x -q -m gpu > $O/tests.txt 2>&1; tail -2 $O/tests.txt
for v in 1 0; do
  echo "== SRE_MIDR=$v" >> $O/rates.txt
  SRE_MIDR=$v timeout 300 python tools/rate.py 14 0 16384 3 >> $O/rates.txt 2>&1
  SRE_MIDR=$v timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3_$v.json 2> $O/bench_c3_$v.err
done
NCU_COUNT=1 NCU_SKIP=1 timeout 600 bash tools/ncu_remote.sh midr/ncu_midr 'k_midr' python tools/rate.py 14 0 16384 1
cat $O/rates.txt
