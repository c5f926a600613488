#!/bin/bash
O=gpurun_out/ns; mkdir -p $O
timeout 300 python tools/rate.py 24 4096 512 2 > $O/rates.txt 2>&1
timeout 300 python tools/rate.py 22 4096 1024 2 >> $O/rates.txt 2>&1
timeout 600 python tools/full_sweep.py 24 scrambled 19 4 > $O/slice.json 2> $O/slice.err
cat $O/rates.txt $O/slice.json
