#!/bin/bash
# 6-deep psi ring in k_passA10s (FP64): N = 15..20 parity, rates, c4 bench
O=gpurun_out/pa10ns; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spectrum.py -x -q -m gpu -k "full_sums or two_pass or chi_elementwise or scrambled_pair_n20 or config1 or fp32 or spectrum or t_state" > $O/tests.txt 2>&1; tail -2 $O/tests.txt
timeout 300 python tools/rate.py 20 4096 8192 2 > $O/rates.txt 2>&1
timeout 300 python tools/rate.py 18 4096 16384 2 >> $O/rates.txt 2>&1
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
cat $O/rates.txt
python -c "import json; d=json.loads([l for l in open('$O/bench_c4.json') if l.startswith('{')][0]); print('c4', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
