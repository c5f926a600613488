#!/bin/bash
# Full N = 24 sweep with the exact additivity pin (tools/full_sweep.py), current default kernels
mkdir -p gpurun_out/full24
timeout 2400 python tools/full_sweep.py 24 scrambled 19 > gpurun_out/full24/full_n24_scrambled.json 2> gpurun_out/full24/full_n24_scrambled.log
