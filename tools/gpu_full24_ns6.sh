#!/bin/bash
# 6-deep psi ring in k_passAw: N = 21..24 parity, then the full pinned N = 24 sweep
O=gpurun_out/full24b; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "streamed_production or chi_elementwise or config5 or two_pass_ranges or variants" > $O/tests.txt 2>&1; tail -2 $O/tests.txt
timeout 2400 python tools/full_sweep.py 24 scrambled 19 > $O/full_n24_scrambled.json 2> $O/full_n24_scrambled.log
cat $O/full_n24_scrambled.json
