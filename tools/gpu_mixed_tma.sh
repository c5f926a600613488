#!/bin/bash
# NEXT-4 tile passes on TMA tiles: parity, bench lines, launch list and one --set full capture (x8)
mkdir -p gpurun_out/mx
timeout 600 python -m pytest tests/test_gpu_mana_mixed.py tests/test_gpu_bench.py -x -q > gpurun_out/mx/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/mx/tests.log
for cfg in x8 x10; do
  timeout 900 python bench.py --config $cfg > gpurun_out/mx/bench_$cfg.json 2> gpurun_out/mx/bench_$cfg.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/mx/launches_x8.csv python bench.py --config x8 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mx/l8.log 2>&1
NCU_COUNT=3 timeout 600 bash tools/ncu_remote.sh mx/ncu_x8_tma 'k_legs_tma' python bench.py --config x8 --steps 1 --warmup 0 --no-cpu-baseline
