#!/bin/bash
# k_midr grid: fewer, longer CTAs (pick_gx slack) -- parity subset and c3 bench
O=gpurun_out/gx; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spectrum.py tests/test_gpu_bench.py -x -q -m gpu > $O/tests.txt 2>&1; tail -2 $O/tests.txt
for i in 1 2; do timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3_$i.json 2> $O/bench_c3_$i.err; done
timeout 300 python tools/rate.py 14 0 16384 3 > $O/rates.txt 2>&1
for f in $O/bench_c3_*.json; do python -c "import json; d=json.loads([l for l in open('$f') if l.startswith('{')][0]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
cat $O/rates.txt
