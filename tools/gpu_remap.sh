#!/bin/bash
# NEXT-3 lane remap: mana parity, m12 bench with the remap on/off, one ncu capture of pass A
O=gpurun_out/remap; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_mana.py -x -q > $O/tests.txt 2>&1; tail -2 $O/tests.txt
for v in 1 0 1 0; do
  SRE_MANA_REMAP=$v timeout 600 python bench.py --config m12 --no-cpu-baseline > $O/bench_m12_$v.json 2> $O/bench_m12_$v.err
  python -c "import json; d=json.loads([l for l in open('$O/bench_m12_$v.json') if l.startswith('{')][0]); print('remap=$v', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline'].get('avg_launch_ms'), d['clocks']['sm_mhz'])" >> $O/summary.txt
done
for v in 1 0; do
  SRE_MANA_REMAP=$v NCU_COUNT=1 NCU_SKIP=2 timeout 600 bash tools/ncu_remote.sh remap/ncu_rowS_$v 'k_mana_rowS' python bench.py --config m12 --steps 1 --warmup 0 --no-cpu-baseline
done
cat $O/summary.txt
